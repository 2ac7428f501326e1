"""The boundary from the reference's side, and MemoryMap handling (SURVEY
§8a MemoryMap row, §8b, §8f.3).

`integration/pcot/gpu_executor.hpp` — the pcot::GpuExecutor a maintainer adds
to the reference tree — is compiled against the UNMODIFIED reference headers
and library into oracle/_ref/ref_adapter_demo (oracle/Makefile; test
infrastructure).  On the GPU the demo runs the reference's own sequence
parse_kernel_file -> allocate / single_assignment_maps -> slt_order / cot_order
-> run -> array_data through the adapter AND through the reference Executor,
and the two must agree: checksum, ExecResult counters, array_base, words
(reference tests/acceptance.cpp:154-165 run_order; exec.hpp:62-82).

Maps (reference memalloc.hpp:14-33): allocate()'s maps keep the hand-written
kernels; single-assignment maps too; any other legal map set runs on the
device interpreter with storage laid out by the maps themselves.
"""
import os
import subprocess

import numpy as np
import pytest

import paper_1802_00166_b200 as P
from tests import oracle_ctypes as O

DEMO = os.path.join(O.REPO, "oracle", "_ref", "ref_adapter_demo")
KDIR = os.path.join(O.REPO, "kernels")
need_demo = pytest.mark.skipif(not os.path.exists(DEMO), reason="adapter demo not built (needs /root/reference)")


def _demo(args, timeout=600):
    env = dict(os.environ, PCOT_KERNEL_PATH=KDIR)
    p = subprocess.run([DEMO] + args, capture_output=True, text=True, timeout=timeout, env=env)
    out = {}
    for line in p.stdout.splitlines():
        k, _, v = line.partition(" ")
        out.setdefault(k, []).append(v)
    return p.returncode, out, p.stdout + p.stderr


def _jacobi_maps(N, T, fold=2, x_ext=None):
    """allocate()'s maps for jacobi2d (printed by the demo: F/Out identity,
    X = (t mod 2, x - t, y - t)), with the fold modulus as a knob."""
    ident = {"linear": [[1, 0], [0, 1]], "constant": [0, 0], "moduli": [0, 0], "extents": [N, N]}
    X = {"array": "X", "linear": [[1, 0, 0], [-1, 1, 0], [-1, 0, 1]], "constant": [0, 0, 0],
         "moduli": [fold, 0, 0], "extents": [fold, x_ext or N, N]}
    return [dict(ident, array="F"), X, dict(ident, array="Out")]


# ---------------------------------------------------------------- CPU
@need_demo
def test_adapter_compiles_against_reference_and_prints_allocate_maps():
    rc, out, txt = _demo([os.path.join(KDIR, "jacobi2d.kernel"), "T=4,N=12", "--maps-only"])
    assert rc == 0, txt
    maps = {v.split()[0]: v for v in out["MAP"]}
    assert maps["X"].startswith("X moduli 2 0 0 extents 2 12 12 linear [ 1 0 0 ] [ -1 1 0 ] [ -1 0 1 ]")
    rc, out, txt = _demo([os.path.join(KDIR, "gs2d.kernel"), "T=4,N=12", "--maps-only"])
    assert {v.split()[0]: v for v in out["MAP"]}["X"].startswith("X moduli 1 0 0 extents 1 12 23")


def test_allocate_maps_keep_the_hot_path():
    hot, why = P.check_maps("jacobi2d", {"T": 16, "N": 64}, _jacobi_maps(64, 16))
    assert hot, why
    hot, why = P.check_maps("jacobi2d", {"T": 16, "N": 64}, _jacobi_maps(64, 16, fold=4))
    assert hot, why  # a multiple of the occupancy vector (2,2,2): also legal storage


def test_single_assignment_maps_keep_the_hot_path():
    N, T = 64, 16
    maps = _jacobi_maps(N, T)
    maps[1] = {"array": "X", "linear": [[1, 0, 0], [0, 1, 0], [0, 0, 1]], "constant": [0, 0, 0],
               "moduli": [0, 0, 0], "extents": [T + 1, N + T, N + T]}
    hot, why = P.check_maps("jacobi2d", {"T": T, "N": N}, maps)
    assert hot, why


def test_other_folds_go_to_the_interpreter():
    hot, why = P.check_maps("jacobi2d", {"T": 16, "N": 64}, _jacobi_maps(64, 16, fold=3))
    assert not hot and "vector" in why
    maps = _jacobi_maps(64, 16)
    maps[0] = dict(maps[0], extents=[64, 72])  # padded input storage: a different layout
    hot, why = P.check_maps("jacobi2d", {"T": 16, "N": 64}, maps)
    assert not hot and "identity" in why


def test_map_errors_are_the_references():
    with pytest.raises(P.PcotError) as e:  # reference map_of: no memory map for array X
        P.check_maps("jacobi2d", {"T": 16, "N": 64}, [m for m in _jacobi_maps(64, 16) if m["array"] != "X"])
    assert e.value.kind == "Validation"
    bad = _jacobi_maps(64, 16)
    bad[1] = dict(bad[1], linear=[[1, 0], [0, 1], [0, 0]])
    with pytest.raises(P.PcotError) as e:
        P.check_maps("jacobi2d", {"T": 16, "N": 64}, bad)
    assert e.value.kind == "DimMismatch"
    with pytest.raises(P.PcotError) as e:  # storage too small for the cells the run writes
        P.check_maps("jacobi2d", {"T": 16, "N": 64}, _jacobi_maps(64, 16, x_ext=40))
    assert e.value.kind == "Validation" and "out-of-extent" in str(e.value)


# ---------------------------------------------------------------- GPU
ADAPTER_CASES = [
    ("jacobi2d", "T=16,N=64", []), ("jacobi2d", "T=13,N=37", ["--scheme", "slt", "--tile", "4,8,16"]),
    ("jacobi2d", "T=16,N=64", ["--scheme", "cot", "--tile", "8,32,32"]),
    ("heat3d_b", "T=5,N=19", []), ("gs2d", "T=8,N=33", ["--scheme", "slt", "--tile", "4,8,16"]),
    ("gs2d", "T=6,N=40", []), ("gemm", "N=33", ["--scheme", "cot", "--tile", "8,8,8"]),
    ("triangle", "N=100", []), ("lud", "N=40", []), ("osp", "N=30", []),
    ("heat1d-fig7", "T=50,N=200", []), ("heat2d_hold", "T=9,N=23", []),
]


@pytest.mark.gpu
@need_demo
@pytest.mark.parametrize("single", [False, True], ids=["allocate", "single"])
@pytest.mark.parametrize("kernel,params,extra", ADAPTER_CASES,
                         ids=["%s-%s-%s" % (k, p, "-".join(e)) for k, p, e in ADAPTER_CASES])
def test_reference_sequence_through_the_adapter(kernel, params, extra, single):
    args = [os.path.join(KDIR, kernel + ".kernel"), params] + extra + (["--single"] if single else [])
    rc, out, txt = _demo(args)
    assert rc == 0, txt
    if kernel == "gemm":  # reordered sums: checked to 1e-12 elsewhere; counters and layout here
        assert out["GPU_COUNTS"] == out["REF_COUNTS"]
    else:
        assert out["GPU_CHECKSUM"] == out["REF_CHECKSUM"], txt
        assert out["GPU_RERUN_CHECKSUM"] == out["REF_CHECKSUM"]
        assert out["GPU_COUNTS"] == out["REF_COUNTS"], txt
    assert out["GPU_ARRAY"] == out["REF_ARRAY"], txt  # array_base + words under the maps
    fam = int(out["GPU_FAMILY"][0])
    if kernel in ("jacobi2d", "heat3d_b", "gs2d", "gemm", "heat2d_hold"):
        assert fam != 5  # the hand-written kernel kept the run under these maps
    else:
        assert fam == 5


@pytest.mark.gpu
@pytest.mark.parametrize("fold", [3, 5])
def test_interpreter_honours_a_folded_map(fold):
    """A fold the hand-written kernel does not reproduce (u = (3,3,3), still a
    universal occupancy vector for the 5-point stencil) runs on the
    interpreter with storage laid out by the map (2-plane... fold-plane ring):
    same bits as the reference golden, storage words = the map's."""
    N, T = 37, 13
    want = [e["checksum"] for e in O.goldens() if e["kernel"] == "jacobi2d" and e["params"] == {"T": T, "N": N}][0]
    with P.GpuExecutor("jacobi2d", {"T": T, "N": N}, maps=_jacobi_maps(N, T, fold=fold)) as ex:
        assert ex.info.family == 5
        r = ex.run_untiled()
        assert r.checksum_hex == want
        assert ex.array_words("X") == fold * N * N
        assert ex.array_base("Out") == 64 + (N * N * 8 + 63) // 64 * 64 + (fold * N * N * 8 + 63) // 64 * 64


def _mapped_cases():
    import json

    with open(os.path.join(O.REPO, "tests", "golden", "corpus.json")) as f:
        return json.load(f).get("mapped", [])


MAPPED = _mapped_cases()


@pytest.mark.gpu
@need_demo
@pytest.mark.parametrize("e", MAPPED, ids=["%s-%s" % (e["kernel"], "-".join("%s%d" % kv for kv in e["params"].items()))
                                           for e in MAPPED])
def test_large_corpus_kernels_from_allocate_mapped_storage(e):
    """lud / osp / triangle / heat1d-fig7 at sizes whose
    single-assignment storage would not be the point (lud N=512: A folded from
    N^3 to ~2N^2 words), run on the device from allocate()'s maps through the
    reference-side adapter, against the reference's emitted-C checksum."""
    ps = ",".join("%s=%d" % kv for kv in e["params"].items())
    rc, out, txt = _demo([os.path.join(KDIR, e["kernel"] + ".kernel"), ps, "--gpu-only"], timeout=900)
    assert rc == 0, txt
    assert int(out["GPU_FAMILY"][0]) == 5
    # dataflow over storage shadows, except heat1d-fig7: allocate()'s fold is
    # safe only for the lexicographic order there (its affine-split copy reads
    # the folded X outside the occupancy cone), which the interpreter detects
    # and answers with the reference's sequential order
    assert int(out["GPU_MODE"][0]) == (0 if e["kernel"] == "heat1d-fig7" else 2), txt
    assert out["GPU_CHECKSUM"] == [e["checksum"]], txt
    assert out["GPU_RERUN_CHECKSUM"] == [e["checksum"]]
