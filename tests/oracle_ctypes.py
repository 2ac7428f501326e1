"""TEST INFRASTRUCTURE: ctypes binding of oracle/liboracle.so (the CPU
restatement) + golden-fixture access.  Only tests/, smoke() and bench.py's
cpu_baseline leg use this module, and only as the checker."""
import ctypes
import json
import os
import subprocess

import numpy as np

REPO = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
ORACLE_DIR = os.path.join(REPO, "oracle")
LIB = os.path.join(ORACLE_DIR, "liboracle.so")
GOLDEN = os.path.join(REPO, "tests", "golden", "golden.json")

_lib = None
_DP = ctypes.POINTER(ctypes.c_double)
_I64 = ctypes.c_int64


def lib():
    global _lib
    if _lib is None:
        if not os.path.exists(LIB):
            subprocess.run(["make", "-s", "-C", ORACLE_DIR, "liboracle.so"], check=True)
        L = ctypes.CDLL(LIB)
        L.oracle_fnv1a.restype = ctypes.c_uint64
        L.oracle_fnv1a.argtypes = [ctypes.c_void_p, ctypes.c_size_t, ctypes.c_uint64]
        L.oracle_init_value.restype = ctypes.c_double
        L.oracle_init_value.argtypes = [ctypes.c_char_p, ctypes.c_uint64]
        L.oracle_init_array.argtypes = [ctypes.c_char_p, _DP, ctypes.c_uint64]
        L.oracle_init_window.argtypes = [ctypes.c_char_p] + [ctypes.c_uint64] * 5 + [_DP]
        L.oracle_stencil2d5.argtypes = [_I64, _I64, ctypes.c_int, _DP, _DP]
        L.oracle_stencil3d7.argtypes = [_I64, _I64, ctypes.c_int, ctypes.c_int, _DP, _DP]
        L.oracle_gs2d9.argtypes = [_I64, _I64, _DP, _DP]
        L.oracle_gemm.argtypes = [_I64, _DP, _DP, _DP]
        L.oracle_gemm_rows.argtypes = [_I64, _I64, _I64, _DP, _DP, _DP]
        L.oracle_set_threads.argtypes = [ctypes.c_int]
        L.oracle_get_threads.restype = ctypes.c_int
        _lib = L
    return _lib


def _p(a):
    return a.ctypes.data_as(_DP)


def fnv1a(a, h=0xcbf29ce484222325):
    a = np.ascontiguousarray(a)
    return lib().oracle_fnv1a(a.ctypes.data, a.nbytes, h)


def init_array(name, n):
    out = np.empty(n, dtype=np.float64)
    lib().oracle_init_array(name.encode(), _p(out), n)
    return out


def init_window(name, ncols, r0, c0, h, w):
    out = np.empty(h * w, dtype=np.float64)
    lib().oracle_init_window(name.encode(), ncols, r0, c0, h, w, _p(out))
    return out.reshape(h, w)


def stencil2d5(N, T, ring_hold, F):
    F = np.ascontiguousarray(F, dtype=np.float64).reshape(-1)
    out = np.empty(N * N, dtype=np.float64)
    lib().oracle_stencil2d5(N, T, ring_hold, _p(F), _p(out))
    return out


def stencil3d7(N, T, rule, ring_hold, F):
    F = np.ascontiguousarray(F, dtype=np.float64).reshape(-1)
    out = np.empty(N ** 3, dtype=np.float64)
    lib().oracle_stencil3d7(N, T, rule, ring_hold, _p(F), _p(out))
    return out


def gs2d9(N, T, F):
    F = np.ascontiguousarray(F, dtype=np.float64).reshape(-1)
    out = np.empty(N * N, dtype=np.float64)
    lib().oracle_gs2d9(N, T, _p(F), _p(out))
    return out


def gemm(N, A, B, rows=None):
    out = np.zeros(N * N, dtype=np.float64)
    if rows is None:
        lib().oracle_gemm(N, _p(A), _p(B), _p(out))
    else:
        lib().oracle_gemm_rows(N, rows[0], rows[1], _p(A), _p(B), _p(out))
    return out


# kernel name -> (family, rule, ring_hold); heat2d/heat3d are the reference corpus
KERNELS = {
    "jacobi2d": ("s2d", 0, 0), "heat2d": ("s2d", 0, 1), "heat2d_hold": ("s2d", 0, 1),
    "heat3d_b": ("s3d", 0, 0), "heat3d": ("s3d", 1, 1), "heat3d_hold": ("s3d", 1, 1),
    "gs2d": ("gs", 0, 0), "gemm": ("gemm", 0, 0),
}


def reference_output(name, params):
    """The oracle's Out array for a kernel spec at a binding."""
    fam, rule, hold = KERNELS[name]
    N = int(params["N"])
    if fam == "s2d":
        return stencil2d5(N, int(params["T"]), hold, init_array("F", N * N))
    if fam == "s3d":
        return stencil3d7(N, int(params["T"]), rule, hold, init_array("F", N ** 3))
    if fam == "gs":
        return gs2d9(N, int(params["T"]), init_array("F", N * N))
    return gemm(N, init_array("A", N * N), init_array("B", N * N))


def goldens():
    with open(GOLDEN) as f:
        return json.load(f)["entries"]


# The reference corpus kernels heat2d/heat3d are re-stated in this repo as
# heat2d_hold/heat3d_hold (kernels/gen_kernels.py); make_golden.py asserts the
# reference interpreter gives both the same checksum.
CORPUS_EQUIV = {"heat2d": "heat2d_hold", "heat3d": "heat3d_hold"}


def kernel_path(name):
    return os.path.join(REPO, "kernels", CORPUS_EQUIV.get(name, name) + ".kernel")
