"""paper_1802_00166_b200 — B200-native executor for the PCOT stencil / fp64-GEMM hot path.

Python mirror of the reference's run API (reference proj/core/include/pcot/
exec.hpp:62-82, kernel_io.hpp:11-22) over the C ABI in include/pcotgpu.h.
The compute path is libpcotgpu.so (hand-written sm_100a CUDA); there is no
CPU fallback: if the library is missing this module raises on first use.
"""
import ctypes
import json
import os

import numpy as np

__all__ = [
    "lib", "PcotError", "KernelInfo", "ExecResult", "GpuExecutor", "recognize",
    "find_kernel_file", "load_kernel_text", "fnv1a", "FAMILIES", "SCHEMES", "check_maps", "generic_source",
]

PKG = os.path.dirname(os.path.abspath(__file__))
REPO = os.path.dirname(PKG)
LIB_PATH = os.path.join(PKG, "libpcotgpu.so")
KERNELS_DIR = os.path.join(REPO, "kernels")

FAMILIES = {1: "stencil2d5", 2: "stencil3d7", 3: "gs2d9", 4: "gemm", 5: "generic"}
SCHEMES = {"untiled": 0, "slt": 1, "cot": 2}
# status -> reference pcot::ErrorKind name (error.hpp:8-16)
ERROR_KINDS = {1: "Overflow", 2: "DimMismatch", 3: "Unbounded", 4: "Parse", 5: "Validation",
               6: "Io", 7: "Unsupported", 8: "Cuda"}
SKIP_CHECKSUM = 1
SPACE_TIME = 2  # COT on 2-D stencils: recursive (depth block x row band) order across launches


class PcotError(RuntimeError):
    """Mirror of pcot::Error: carries the ErrorKind name in .kind."""

    def __init__(self, kind, msg):
        super().__init__("%s: %s" % (kind, msg))
        self.kind = kind


class KernelInfo(ctypes.Structure):
    _fields_ = [("family", ctypes.c_int32), ("rule", ctypes.c_int32),
                ("ring_hold", ctypes.c_int32), ("ndim", ctypes.c_int32),
                ("T", ctypes.c_int64), ("N", ctypes.c_int64),
                ("points", ctypes.c_uint64), ("reads", ctypes.c_uint64),
                ("writes", ctypes.c_uint64), ("name", ctypes.c_char * 64)]

    @property
    def family_name(self):
        return FAMILIES.get(self.family, "?")


class MapC(ctypes.Structure):
    """pcotgpu_map: reference MemoryMap (memalloc.hpp:14-33)."""
    _fields_ = [("array", ctypes.c_char_p), ("rank", ctypes.c_int32), ("storage_rank", ctypes.c_int32),
                ("linear", ctypes.POINTER(ctypes.c_int64)), ("constant", ctypes.POINTER(ctypes.c_int64)),
                ("moduli", ctypes.POINTER(ctypes.c_int64)), ("extents", ctypes.POINTER(ctypes.c_int64)),
                ("single_assignment", ctypes.c_int32), ("reserved", ctypes.c_int32)]


class Schedule(ctypes.Structure):
    _fields_ = [("scheme", ctypes.c_int32), ("ndim", ctypes.c_int32),
                ("leaf", ctypes.c_int64 * 8), ("flags", ctypes.c_int32),
                ("reserved", ctypes.c_int32)]


class ExecResult(ctypes.Structure):
    """Mirror of pcot::ExecResult (exec.hpp:45-52) + device time."""
    _fields_ = [("points", ctypes.c_uint64), ("reads", ctypes.c_uint64),
                ("writes", ctypes.c_uint64), ("violation", ctypes.c_int32),
                ("bt", ctypes.c_int32), ("checksum", ctypes.c_uint64),
                ("device_ms", ctypes.c_double), ("launches", ctypes.c_uint64)]

    @property
    def checksum_hex(self):
        return "%016x" % self.checksum


_lib = None
_I64P = ctypes.POINTER(ctypes.c_int64)
_DP = ctypes.POINTER(ctypes.c_double)

# (name, restype, argtypes) for every symbol include/pcotgpu.h declares
_SIGS = [
    ("pcotgpu_recognize", ctypes.c_int, [ctypes.c_char_p, _I64P, ctypes.c_size_t, ctypes.POINTER(KernelInfo)]),
    ("pcotgpu_find_kernel_file", ctypes.c_int, [ctypes.c_char_p, ctypes.c_char_p, ctypes.c_size_t]),
    ("pcotgpu_create", ctypes.c_int, [ctypes.c_char_p, _I64P, ctypes.c_size_t, ctypes.c_int, ctypes.POINTER(ctypes.c_void_p)]),
    ("pcotgpu_create_mapped", ctypes.c_int, [ctypes.c_char_p, _I64P, ctypes.c_size_t, ctypes.POINTER(MapC),
                                             ctypes.c_size_t, ctypes.c_int, ctypes.POINTER(ctypes.c_void_p)]),
    ("pcotgpu_check_maps", ctypes.c_int, [ctypes.c_char_p, _I64P, ctypes.c_size_t, ctypes.POINTER(MapC),
                                          ctypes.c_size_t, ctypes.POINTER(ctypes.c_int), ctypes.c_char_p,
                                          ctypes.c_size_t]),
    ("pcotgpu_generic_source", ctypes.c_int, [ctypes.c_char_p, _I64P, ctypes.c_size_t, ctypes.c_int,
                                              ctypes.c_char_p, ctypes.c_size_t, ctypes.POINTER(ctypes.c_size_t)]),
    ("pcotgpu_generic_info", ctypes.c_int, [ctypes.c_void_p, ctypes.POINTER(ctypes.c_int),
                                            ctypes.POINTER(ctypes.c_int), ctypes.c_char_p, ctypes.c_size_t]),
    ("pcotgpu_run", ctypes.c_int, [ctypes.c_void_p, ctypes.POINTER(Schedule), ctypes.POINTER(ExecResult)]),
    ("pcotgpu_run_untiled", ctypes.c_int, [ctypes.c_void_p, ctypes.POINTER(ExecResult)]),
    ("pcotgpu_run_batch", ctypes.c_int, [ctypes.c_void_p, ctypes.POINTER(Schedule), ctypes.c_size_t,
                                         ctypes.POINTER(_DP), ctypes.POINTER(_DP), ctypes.POINTER(ExecResult)]),
    ("pcotgpu_reset", ctypes.c_int, [ctypes.c_void_p]),
    ("pcotgpu_read_array", ctypes.c_int, [ctypes.c_void_p, ctypes.c_char_p, _DP, ctypes.c_size_t]),
    ("pcotgpu_write_array", ctypes.c_int, [ctypes.c_void_p, ctypes.c_char_p, _DP, ctypes.c_size_t]),
    ("pcotgpu_array_base", ctypes.c_int, [ctypes.c_void_p, ctypes.c_char_p, ctypes.POINTER(ctypes.c_uint64)]),
    ("pcotgpu_array_words", ctypes.c_int, [ctypes.c_void_p, ctypes.c_char_p, ctypes.POINTER(ctypes.c_uint64)]),
    ("pcotgpu_info", ctypes.c_int, [ctypes.c_void_p, ctypes.POINTER(KernelInfo)]),
    ("pcotgpu_device_view", ctypes.c_int, [ctypes.c_void_p, ctypes.c_char_p, ctypes.POINTER(ctypes.c_void_p), _I64P]),
    ("pcotgpu_set_stream", ctypes.c_int, [ctypes.c_void_p, ctypes.c_void_p]),
    ("pcotgpu_destroy", None, [ctypes.c_void_p]),
    ("pcotgpu_s2d5_layout", ctypes.c_int, [ctypes.c_int64, ctypes.c_int64, _I64P, _I64P, _I64P, _I64P]),
    ("pcotgpu_s2d5_advance", ctypes.c_int, [ctypes.c_void_p, ctypes.c_void_p, ctypes.c_int64, ctypes.c_int64,
                                            ctypes.c_int64, ctypes.c_int64, ctypes.c_int, ctypes.c_int,
                                            ctypes.c_int, ctypes.c_int64, ctypes.c_int64, ctypes.c_void_p]),
    ("pcotgpu_s2d5_advance_p2p", ctypes.c_int, [ctypes.c_void_p, ctypes.c_void_p, ctypes.c_int64, ctypes.c_int64,
                                                ctypes.c_int64, ctypes.c_int64, ctypes.c_int, ctypes.c_int,
                                                ctypes.c_int, ctypes.c_int64, ctypes.c_int64, ctypes.c_void_p,
                                                ctypes.c_void_p, ctypes.c_int64, ctypes.c_void_p]),
    ("pcotgpu_fill_init_value", ctypes.c_int, [ctypes.c_void_p, ctypes.c_int64, ctypes.c_int64, ctypes.c_int64,
                                               ctypes.c_char_p, ctypes.c_uint64, ctypes.c_void_p]),
    ("pcotgpu_s2d5_prepare", ctypes.c_int, [ctypes.c_void_p, ctypes.c_int64, ctypes.c_int64, ctypes.c_int64,
                                            ctypes.c_int64, ctypes.c_int, ctypes.c_void_p]),
    ("pcotgpu_test_div9", ctypes.c_int, [ctypes.c_void_p, ctypes.c_void_p, ctypes.c_void_p, ctypes.c_int64,
                                         ctypes.c_void_p]),
    ("pcotgpu_last_error", ctypes.c_char_p, []),
    ("pcotgpu_launch_count", ctypes.c_uint64, []),
    ("pcotgpu_abi_version", ctypes.c_int, []),
    ("pcotgpu_device_count", ctypes.c_int, [ctypes.POINTER(ctypes.c_int)]),
    ("pcotgpu_fnv1a", ctypes.c_uint64, [ctypes.c_void_p, ctypes.c_size_t, ctypes.c_uint64]),
]


def lib():
    """Load libpcotgpu.so (raises if it has not been built: no fallback)."""
    global _lib
    if _lib is None:
        if not os.path.exists(LIB_PATH):
            raise ImportError("libpcotgpu.so not built (run __graft_entry__.build()); "
                              "the CUDA path is the only implementation")
        L = ctypes.CDLL(LIB_PATH)
        for name, res, args in _SIGS:
            fn = getattr(L, name)
            fn.restype = res
            fn.argtypes = args
        _lib = L
    return _lib


def _check(status):
    if status != 0:
        msg = lib().pcotgpu_last_error().decode(errors="replace")
        raise PcotError(ERROR_KINDS.get(status, "status %d" % status), msg)


def fnv1a(buf, h=0xcbf29ce484222325):
    """reference exec.cpp:12-19 over the raw bytes of a numpy array / bytes."""
    if isinstance(buf, (bytes, bytearray)):
        buf = np.frombuffer(bytes(buf), dtype=np.uint8)
    a = np.ascontiguousarray(buf)
    return lib().pcotgpu_fnv1a(a.ctypes.data, a.nbytes, h)


def find_kernel_file(name):
    """reference kernel_io.cpp:250-276 (path, $PCOT_KERNEL_PATH, ./kernels)."""
    out = ctypes.create_string_buffer(4096)
    _check(lib().pcotgpu_find_kernel_file(name.encode(), out, 4096))
    return out.value.decode()


def load_kernel_text(kernel):
    """Accept JSON text, a path, or a kernel name (searched like the reference,
    then in this repo's kernels/)."""
    if kernel.lstrip().startswith("{"):
        return kernel
    path = find_kernel_file(kernel)
    if not path:
        for cand in (os.path.join(KERNELS_DIR, kernel), os.path.join(KERNELS_DIR, kernel + ".kernel")):
            if os.path.exists(cand):
                path = cand
                break
    if not path:
        raise PcotError("Io", "kernel not found: " + kernel)
    with open(path) as f:
        return f.read()


def _params_array(text, params):
    if isinstance(params, dict):
        try:
            names = json.loads(text)["params"]
        except (ValueError, KeyError) as e:
            raise PcotError("Parse", "kernel JSON: %s" % e)
        missing = [n for n in names if n not in params]
        if missing:
            raise PcotError("DimMismatch", "missing params %s" % missing)
        vals = [int(params[n]) for n in names]
    else:
        vals = [int(v) for v in params]
    return (ctypes.c_int64 * max(1, len(vals)))(*vals), len(vals)


def _maps_array(maps):
    """maps: [{"array", "linear" (rows), "constant", "moduli", "extents"}] ->
    (ctypes array of MapC, keep-alive list)."""
    keep = []
    arr = (MapC * max(1, len(maps)))()
    for i, m in enumerate(maps):
        lin = [v for row in m["linear"] for v in row]
        rank = len(m["linear"][0]) if m["linear"] else 0
        bufs = [(ctypes.c_int64 * max(1, len(x)))(*x) for x in (lin, m["constant"], m["moduli"], m["extents"])]
        name = m["array"].encode()
        keep += bufs + [name]
        arr[i] = MapC(name, rank, len(m["extents"]), bufs[0], bufs[1], bufs[2], bufs[3],
                      int(bool(m.get("single_assignment", False))), 0)
    return arr, keep


def check_maps(kernel, params, maps):
    """Host only: (hot_path, why) for a map set (pcotgpu_check_maps)."""
    text = load_kernel_text(kernel)
    arr, n = _params_array(text, params)
    marr, keep = _maps_array(maps)
    hot = ctypes.c_int()
    why = ctypes.create_string_buffer(512)
    _check(lib().pcotgpu_check_maps(text.encode(), arr, n, marr, len(maps), ctypes.byref(hot), why, 512))
    return bool(hot.value), why.value.decode()


def generic_source(kernel, params, compile=False):
    """Host only: the PRDG -> CUDA emitter's source for a kernel; compile=True
    also compiles it with NVRTC for sm_100a (PcotError Unsupported with the
    compiler log on failure)."""
    text = load_kernel_text(kernel)
    arr, n = _params_array(text, params)
    need = ctypes.c_size_t()
    lib().pcotgpu_generic_source(text.encode(), arr, n, 0, None, 0, ctypes.byref(need))
    buf = ctypes.create_string_buffer(max(need.value, 1) + 65536)
    st = lib().pcotgpu_generic_source(text.encode(), arr, n, int(bool(compile)), buf, len(buf), ctypes.byref(need))
    if st != 0:
        raise PcotError(ERROR_KINDS.get(st, "status %d" % st),
                        lib().pcotgpu_last_error().decode(errors="replace") + "\n" + buf.value.decode(errors="replace"))
    return buf.value.decode()


def recognize(kernel, params):
    """parse_kernel + recognizer (host only): returns KernelInfo."""
    text = load_kernel_text(kernel)
    arr, n = _params_array(text, params)
    info = KernelInfo()
    _check(lib().pcotgpu_recognize(text.encode(), arr, n, ctypes.byref(info)))
    return info


class GpuExecutor:
    """Drop-in for pcot::Executor (exec.hpp:62-82) on one B200.

    GpuExecutor(kernel, params, device=0); run(scheme, tile) / run_untiled();
    reset(); array_data(name); array_base(name).  `tile` is the reference
    TileSpec leaf vector: leaf[0] (time) is the temporal block depth.
    """

    def __init__(self, kernel, params, device=0, maps=None):
        self._h = None
        text = load_kernel_text(kernel)
        self.spec = json.loads(text)
        arr, n = _params_array(text, params)
        h = ctypes.c_void_p()
        if maps is None:
            _check(lib().pcotgpu_create(text.encode(), arr, n, int(device), ctypes.byref(h)))
        else:  # Executor(p, params, maps): the reference's MemoryMaps
            marr, keep = _maps_array(maps)
            _check(lib().pcotgpu_create_mapped(text.encode(), arr, n, marr, len(maps), int(device),
                                               ctypes.byref(h)))
        self._h = h
        self.info = KernelInfo()
        _check(lib().pcotgpu_info(self._h, ctypes.byref(self.info)))

    def close(self):
        if self._h is not None:
            lib().pcotgpu_destroy(self._h)
            self._h = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass

    def __enter__(self):
        return self

    def __exit__(self, *a):
        self.close()

    @staticmethod
    def _schedule(scheme, tile, skip_checksum, space_time=False):
        s = Schedule()
        if scheme == "cot-st":  # the space-time recursive order (TileOrder.space_time)
            scheme, space_time = "cot", True
        s.scheme = SCHEMES[scheme] if isinstance(scheme, str) else int(scheme)
        tile = list(tile or [])
        s.ndim = len(tile)
        for i, v in enumerate(tile[:8]):
            s.leaf[i] = int(v)
        s.flags = (SKIP_CHECKSUM if skip_checksum else 0) | (SPACE_TIME if space_time else 0)
        return s

    @property
    def input_names(self):
        return [a["name"] for a in self.spec["arrays"] if a.get("kind") == "input"]

    @property
    def output_name(self):
        return [a["name"] for a in self.spec["arrays"] if a.get("kind") == "output"][0]

    def run(self, scheme="untiled", tile=None, skip_checksum=False):
        s = self._schedule(scheme, tile, skip_checksum)
        r = ExecResult()
        _check(lib().pcotgpu_run(self._h, ctypes.byref(s), ctypes.byref(r)))
        return r

    def run_batch(self, inputs, outputs, scheme="untiled", tile=None, skip_checksum=False):
        """`len(outputs)` independent runs from host memory, copies overlapped
        with the compute (pcotgpu_run_batch).  inputs[k] is instance k's input
        array, or a sequence of them in `input_names` order; outputs[k] receives
        instance k's output.  All float64, C-contiguous, array_words long
        (pinned memory, e.g. torch's pin_memory, keeps the copies async)."""
        names = self.input_names
        count = len(outputs)
        if len(inputs) != count:
            raise PcotError("DimMismatch", "run_batch: %d input sets for %d outputs" % (len(inputs), count))
        keep = []
        ins = (_DP * max(1, count * len(names)))()
        outs = (_DP * max(1, count))()
        for k in range(count):
            per = [inputs[k]] if len(names) == 1 and not isinstance(inputs[k], (list, tuple)) else list(inputs[k])
            if len(per) != len(names):
                raise PcotError("DimMismatch", "run_batch: instance %d needs inputs %s" % (k, names))
            for q, a in enumerate(per):
                if a.dtype != np.float64 or not a.flags.c_contiguous or a.size != self.array_words(names[q]):
                    raise PcotError("DimMismatch", "run_batch: input %s of instance %d" % (names[q], k))
                keep.append(a)
                ins[k * len(names) + q] = a.ctypes.data_as(_DP)
            o = outputs[k]
            if (o.dtype != np.float64 or not o.flags.c_contiguous
                    or o.size != self.array_words(self.output_name)):
                raise PcotError("DimMismatch", "run_batch: output of instance %d" % k)
            outs[k] = o.ctypes.data_as(_DP)
        s = self._schedule(scheme, tile, skip_checksum)
        r = ExecResult()
        _check(lib().pcotgpu_run_batch(self._h, ctypes.byref(s), count, ins, outs, ctypes.byref(r)))
        return r

    def run_untiled(self, skip_checksum=False):
        return self.run("untiled", None, skip_checksum)

    def reset(self):
        _check(lib().pcotgpu_reset(self._h))

    def array_words(self, name):
        w = ctypes.c_uint64()
        _check(lib().pcotgpu_array_words(self._h, name.encode(), ctypes.byref(w)))
        return w.value

    def array_data(self, name, out=None):
        w = self.array_words(name)
        if out is None:
            out = np.empty(w, dtype=np.float64)
        assert out.dtype == np.float64 and out.size == w and out.flags.c_contiguous
        _check(lib().pcotgpu_read_array(self._h, name.encode(), out.ctypes.data_as(_DP), w))
        return out

    def write_array(self, name, values):
        a = np.ascontiguousarray(values, dtype=np.float64).reshape(-1)
        _check(lib().pcotgpu_write_array(self._h, name.encode(), a.ctypes.data_as(_DP), a.size))

    def array_base(self, name):
        b = ctypes.c_uint64()
        _check(lib().pcotgpu_array_base(self._h, name.encode(), ctypes.byref(b)))
        return b.value

    def device_view(self, name):
        p = ctypes.c_void_p()
        ld = ctypes.c_int64()
        _check(lib().pcotgpu_device_view(self._h, name.encode(), ctypes.byref(p), ctypes.byref(ld)))
        return p.value, ld.value

    def generic_info(self):
        """Device interpreter only: (schedule mode, compiled by the emitter, status)."""
        mode, comp = ctypes.c_int(), ctypes.c_int()
        why = ctypes.create_string_buffer(4096)
        _check(lib().pcotgpu_generic_info(self._h, ctypes.byref(mode), ctypes.byref(comp), why, 4096))
        return mode.value, bool(comp.value), why.value.decode(errors="replace")

    def set_stream(self, stream_ptr):
        _check(lib().pcotgpu_set_stream(self._h, ctypes.c_void_p(stream_ptr)))
