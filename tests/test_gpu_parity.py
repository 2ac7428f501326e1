"""GPU parity: the sm_100a kernels, called through the C ABI, against the
reference's outputs (goldens) and the oracle.  Bit-exact for every stencil
and Gauss-Seidel; GEMM within 1e-12 (normwise and componentwise).
"""
import numpy as np
import pytest

import paper_1802_00166_b200 as P
from tests import oracle_ctypes as O

pytestmark = pytest.mark.gpu

GOLD = [e for e in O.goldens() if e["kernel"] != "gemm"]


def _id(e):
    return "%s-%s" % (e["kernel"], "-".join("%s%d" % kv for kv in e["params"].items()))


def _golden(kernel, **params):
    for e in O.goldens():
        if e["kernel"] == kernel and e["params"] == params:
            return e["checksum"]
    raise KeyError((kernel, params))


@pytest.mark.parametrize("e", GOLD, ids=[_id(e) for e in GOLD])
def test_default_schedule_matches_reference(e):
    with P.GpuExecutor(O.kernel_path(e["kernel"]), e["params"]) as ex:
        r = ex.run_untiled()
        assert r.checksum_hex == e["checksum"]
        assert r.launches > 0
        if "points" in e:
            assert r.points == e["points"]
        if "out_hex" in e:
            out = ex.array_data("Out")
            want = np.array([int(h, 16) for h in e["out_hex"]], dtype=np.uint64)
            assert np.array_equal(out.view(np.uint64), want)


@pytest.mark.parametrize("bt", range(1, 9))
@pytest.mark.parametrize("scheme", ["slt", "cot"])
def test_jacobi2d_every_temporal_depth(bt, scheme):
    want = _golden("jacobi2d", T=40, N=1000)
    with P.GpuExecutor("jacobi2d", {"T": 40, "N": 1000}) as ex:
        r = ex.run(scheme, [bt, 64, 256])
        assert r.bt == bt
        assert r.checksum_hex == want


@pytest.mark.parametrize("bt", [1, 3, 5, 8])
def test_heat2d_ring_copied_every_depth(bt):
    want = _golden("heat2d", T=64, N=1024)
    with P.GpuExecutor(O.kernel_path("heat2d"), {"T": 64, "N": 1024}) as ex:
        assert ex.run("slt", [bt, 32, 32]).checksum_hex == want


@pytest.mark.parametrize("bt", [1, 2, 3, 4])
@pytest.mark.parametrize("kernel", ["heat3d_b", "heat3d"])
def test_heat3d_every_temporal_depth(kernel, bt):
    want = _golden(kernel, T=20, N=130)
    with P.GpuExecutor(O.kernel_path(kernel), {"T": 20, "N": 130}) as ex:
        assert ex.run("cot" if bt % 2 else "slt", [bt, 8, 8, 8]).checksum_hex == want


@pytest.mark.parametrize("tile", [(1, 8, 16), (2, 16, 64), (4, 32, 256), (8, 32, 128), (3, 17, 50)])
def test_gs2d_tile_shapes(tile):
    want = _golden("gs2d", T=16, N=1024)
    with P.GpuExecutor("gs2d", {"T": 16, "N": 1024}) as ex:
        assert ex.run("slt", list(tile)).checksum_hex == want


GS_PIPE_SHAPES = [(1, 3), (1, 34), (2, 35), (13, 66), (12, 97), (25, 100), (40, 130), (7, 1000)]


@pytest.mark.parametrize("variant", [0, 1, 2, 5, 6, 7, 8, 9, 11])
@pytest.mark.parametrize("T,N", GS_PIPE_SHAPES)
def test_gs2d_pipeline_matches_oracle(monkeypatch, variant, T, N):
    """Systolic pipeline (untiled default): every variant (warps per band x ring
    depth), level counts around the warp count, partial last bands."""
    monkeypatch.setenv("PCOTGPU_GS_PIPE_V", str(variant))
    F = O.init_array("F", N * N)
    want = O.gs2d9(N, T, F)
    with P.GpuExecutor("gs2d", {"T": T, "N": N}) as ex:
        ex.run_untiled()
        got = ex.array_data("Out")
    assert np.array_equal(got.view(np.uint64), want.view(np.uint64))


def test_gs2d_pipeline_multi_launch_segments():
    """T beyond one launch's level budget (progress words / band count): the
    pipeline splits the sweeps into launches that restart from the grid."""
    N, T = 130, 5000
    F = O.init_array("F", N * N)
    want = O.gs2d9(N, T, F)
    with P.GpuExecutor("gs2d", {"T": T, "N": N}) as ex:
        r = ex.run_untiled()
        assert r.bt == 0 and r.launches >= 2 + 3  # copy-in + ring, then >= 3 segment launches
        got = ex.array_data("Out")
    assert np.array_equal(got.view(np.uint64), want.view(np.uint64))


@pytest.mark.parametrize("variant", [0, 1, 2, 5, 6, 7, 8, 9, 11])
@pytest.mark.parametrize("T,N", [(16, 1024), (64, 4096)])
def test_gs2d_pipeline_goldens_repeated(monkeypatch, variant, T, N):
    """Reference checksums, three runs in a row on one executor (edge slots
    are re-armed per run; a scheduling race would show as a flaky checksum)."""
    monkeypatch.setenv("PCOTGPU_GS_PIPE_V", str(variant))
    want = _golden("gs2d", T=T, N=N)
    with P.GpuExecutor("gs2d", {"T": T, "N": N}) as ex:
        for _ in range(3):
            assert ex.run_untiled().checksum_hex == want


def _gemm_check(out, N, rows=None):
    A = O.init_array("A", N * N)
    B = O.init_array("B", N * N)
    ref = O.gemm(N, A, B, rows).reshape(N, N)
    got = out.reshape(N, N)
    if rows is not None:
        ref, got = ref[rows[0]:rows[1]], got[rows[0]:rows[1]]
    A2 = np.abs(2 * A - 1).reshape(N, N)
    B2 = np.abs(2 * B - 1).reshape(N, N)
    absab = (A2 @ B2) if rows is None else (A2[rows[0]:rows[1]] @ B2)
    diff = np.abs(got - ref)
    normwise = np.linalg.norm(diff) / np.linalg.norm(ref)
    componentwise = (diff / absab).max()
    assert normwise <= 1e-12, normwise
    assert componentwise <= 1e-12, componentwise
    return normwise, componentwise


@pytest.mark.parametrize("N", [1, 16, 33, 64, 127, 512, 1000])
@pytest.mark.parametrize("scheme", ["slt", "cot"])
def test_gemm_tolerance(N, scheme):
    with P.GpuExecutor("gemm", {"N": N}) as ex:
        ex.run(scheme, [16, 16, 16])
        _gemm_check(ex.array_data("Out"), N)


@pytest.mark.parametrize("variant", [0, 10, 9, 1])
@pytest.mark.parametrize("N", [2, 15, 130, 257, 1032])
def test_gemm_kernel_variants_ragged_sizes(monkeypatch, variant, N):
    """Every DGEMM load path on sizes that are not multiples of the 128x128 CTA
    tile, the 16-double TMA box or the k-block: the tensor-TMA ring (0: BK 32 x
    3 stages, 10: BK 16 x 6; out-of-bounds box parts are zero-filled by the TMA
    engine) and the cp.async kernels of round 1 (9, 1), Morton tile order."""
    monkeypatch.setenv("PCOTGPU_DGEMM_VARIANT", str(variant))
    with P.GpuExecutor("gemm", {"N": N}) as ex:
        ex.run("cot", [16, 16, 16])
        _gemm_check(ex.array_data("Out"), N)


@pytest.mark.parametrize("scheme", ["untiled", "slt"])
def test_gemm_config3_all_rows(scheme):
    """BASELINE config 3 (N=4096): every one of the 4096 rows against the
    sequential-k oracle (all host threads), normwise and componentwise 1e-12;
    and the reference's own sampled cells (its emitted-C dump)."""
    import json
    import os

    N = 4096
    with P.GpuExecutor("gemm", {"N": N}) as ex:
        ex.run(scheme, None if scheme == "untiled" else [64, 64, 64], skip_checksum=True)
        out = ex.array_data("Out")
    O.lib().oracle_set_threads(os.cpu_count() or 1)
    _gemm_check(out, N)
    with open(os.path.join(O.REPO, "tests", "golden", "gemm4096_samples.json")) as f:
        g = json.load(f)
    rows = np.arange(N)
    got = out.reshape(N, N)[rows, (rows * 2654435761 + 12345) % N]
    ref = np.array([int(h, 16) for h in g["out_hex"]], dtype=np.uint64).view(np.float64)
    assert (np.abs(got - ref) / np.array(g["absab"])).max() <= 1e-12


def test_storage_persists_and_reset():
    with P.GpuExecutor("jacobi2d", {"T": 16, "N": 64}) as ex:
        a = ex.run_untiled().checksum
        b = ex.run_untiled().checksum
        assert a == b  # every run restarts from F, as the reference's init statement does
        F = ex.array_data("F")
        assert np.array_equal(F, O.init_array("F", 64 * 64))
        ex.write_array("F", 2.0 * F)
        c = ex.run_untiled().checksum
        assert c != a
        out2 = ex.array_data("Out")
        ex.reset()
        assert ex.run_untiled().checksum == a
        # linearity by a power of two is exact in fp64 (no over/underflow here)
        assert np.array_equal(out2, 2.0 * ex.array_data("Out"))


def test_input_from_host_matches_device_init():
    N, T = 1000, 40
    with P.GpuExecutor("jacobi2d", {"T": T, "N": N}) as ex:
        ex.write_array("F", O.init_array("F", N * N))
        assert ex.run_untiled().checksum_hex == _golden("jacobi2d", T=T, N=N)


def _window_check(out2d, N, T, r0, c0, w):
    """Cells [r0, r0+w) x [c0, c0+w) of an N x N zero-ring Jacobi result depend
    only on F within distance T: recompute them with the oracle on a window."""
    lo_r, lo_c = max(0, r0 - T - 1), max(0, c0 - T - 1)
    hi_r, hi_c = min(N, r0 + w + T + 1), min(N, c0 + w + T + 1)
    # square window so the oracle's N x N routine applies; pad with ring cells
    S = max(hi_r - lo_r, hi_c - lo_c)
    lo_r, lo_c = min(lo_r, N - S), min(lo_c, N - S)
    F = O.init_window("F", N, lo_r, lo_c, S, S)
    ref = O.stencil2d5(S, T, 0, F).reshape(S, S)
    got = out2d[r0:r0 + w, c0:c0 + w]
    want = ref[r0 - lo_r:r0 - lo_r + w, c0 - lo_c:c0 - lo_c + w]
    # window edges that are not real grid edges are artificial zero rings; the
    # inner cells are at distance > T from them, so they are exact
    assert np.array_equal(got.view(np.uint64), want.view(np.uint64)), (r0, c0)


@pytest.mark.slow
def test_config4_full_size_windows_and_ring():
    """BASELINE config 4 (32768^2, T=512) on one GPU: exact windows at a corner,
    an edge and the centre, zero ring, and exact scaling by 2."""
    N, T = 32768, 512
    with P.GpuExecutor("jacobi2d", {"T": T, "N": N}) as ex:
        r = ex.run_untiled(skip_checksum=True)
        assert r.launches >= T // max(1, r.bt)
        out = ex.array_data("Out").reshape(N, N)
        assert not out[0].any() and not out[-1].any() and not out[:, 0].any() and not out[:, -1].any()
        for (r0, c0) in [(0, 0), (N - 40, 16000), (16380, 16380)]:
            _window_check(out, N, T, r0, c0, 40)
        corner = out[:64, :64].copy()
        del out
        F = ex.array_data("F")
        ex.write_array("F", F * 2.0)
        del F
        ex.run_untiled(skip_checksum=True)
        out2 = ex.array_data("Out").reshape(N, N)
        assert np.array_equal(out2[:64, :64], corner * 2.0)


@pytest.mark.slow
def test_config4_full_size_checksum():
    """BASELINE config 4 (32768^2, T=512): the FNV-1a checksum of the whole
    8 GiB output equals the reference's (its emitted C at full size,
    tests/golden/make_golden.py --cfg4), for the default and the COT order."""
    want = _golden("jacobi2d", T=512, N=32768)
    with P.GpuExecutor("jacobi2d", {"T": 512, "N": 32768}) as ex:
        assert ex.run_untiled().checksum_hex == want
        assert ex.run("cot", [8, 64, 256]).checksum_hex == want


@pytest.mark.parametrize("kernel,params,tile", [
    ("jacobi2d", {"T": 40, "N": 1000}, ("slt", [5, 64, 256])),
    ("heat3d_b", {"T": 20, "N": 130}, ("untiled", None)),
    ("gs2d", {"T": 16, "N": 1024}, ("untiled", None)),
    ("gemm", {"N": 127}, ("cot", [16, 16, 16])),
])
def test_run_batch_equals_single_runs(kernel, params, tile):
    """pcotgpu_run_batch: every instance's output equals a separate
    write_array -> run -> array_data sequence, bit for bit."""
    with P.GpuExecutor(O.kernel_path(kernel), params) as ex:
        names = ex.input_names
        base = [ex.array_data(nm) for nm in names]
        sets = [[b.copy() for b in base], [2.0 * b for b in base], [b[::-1].copy() for b in base]]
        outs = [np.empty(ex.array_words(ex.output_name)) for _ in sets]
        r = ex.run_batch([s if len(s) > 1 else s[0] for s in sets], outs, *tile)
        assert r.launches > 0
        for s, got in zip(sets, outs):
            for nm, a in zip(names, s):
                ex.write_array(nm, a)
            ex.run(*tile, skip_checksum=True)
            want = ex.array_data(ex.output_name)
            assert np.array_equal(got.view(np.uint64), want.view(np.uint64))
        assert r.checksum == P.fnv1a(outs[-1])


def test_run_batch_errors():
    with P.GpuExecutor("jacobi2d", {"T": 4, "N": 64}) as ex:
        F = ex.array_data("F")
        with pytest.raises(P.PcotError) as e:
            ex.run_batch([], [])
        assert e.value.kind == "Validation"
        with pytest.raises(P.PcotError) as e:
            ex.run_batch([F], [np.empty(10)])
        assert e.value.kind == "DimMismatch"
        one = np.empty(64 * 64)
        ex.run_batch([F], [one])
        ex.run_untiled()
        assert np.array_equal(one, ex.array_data("Out"))


@pytest.mark.parametrize("variant", [0, 5, 7, 9])
def test_gs2d_pipeline_nan_input_with_sentinel_bits(monkeypatch, variant):
    """An input NaN carrying the edge slots' "not yet written" bit pattern
    (0xffff...ffff) must neither stall the pipeline nor leak: the run returns,
    NaN spreads exactly where the oracle's does, every other cell is bit-exact."""
    monkeypatch.setenv("PCOTGPU_GS_PIPE_V", str(variant))
    N, T = 200, 9
    F = O.init_array("F", N * N)
    F.view(np.uint64)[57 * N + 101] = np.uint64(0xFFFFFFFFFFFFFFFF)
    F.view(np.uint64)[120 * N + 33] = np.uint64(0x7FF8000000000123)  # a NaN with another payload
    want = O.gs2d9(N, T, F)
    with P.GpuExecutor("gs2d", {"T": T, "N": N}) as ex:
        ex.write_array("F", F)
        ex.run_untiled()
        got = ex.array_data("Out")
    assert np.array_equal(np.isnan(got), np.isnan(want))
    ok = ~np.isnan(want)
    assert np.isnan(want).sum() > 100
    assert np.array_equal(got[ok].view(np.uint64), want[ok].view(np.uint64))


@pytest.mark.parametrize("bt,band", [(1, 8), (2, 64), (4, 100), (6, 333), (8, 1000)])
@pytest.mark.parametrize("kernel", ["jacobi2d", "heat2d"])
def test_space_time_cot_order_is_exact(kernel, bt, band):
    """COT across time (SPACE_TIME): one launch per (depth block, row band) in
    Morton order of the skewed box — every band through several depth blocks
    before its neighbours catch up — reproduces the reference bit for bit."""
    params = {"T": 40, "N": 1000} if kernel == "jacobi2d" else {"T": 64, "N": 1024}
    want = _golden(kernel, **params)
    with P.GpuExecutor(O.kernel_path(kernel), params) as ex:
        r = ex.run("cot-st", [bt, band, 256])
        nblk = -(-params["T"] // bt)
        nband = -(-params["N"] // max(band, 2 * bt))
        assert r.launches >= nblk * nband
        assert r.checksum_hex == want
