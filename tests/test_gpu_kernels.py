"""GPU: kernel-level properties that the end-to-end goldens do not isolate."""
import ctypes

import numpy as np
import pytest

import paper_1802_00166_b200 as P
from tests import oracle_ctypes as O

pytestmark = pytest.mark.gpu

torch = pytest.importorskip("torch")


def test_gauss_seidel_division_is_ieee_correctly_rounded():
    """The Gauss-Seidel kernel divides by 9.0 with a Markstein correction
    instead of the general division; it must equal __ddiv_rn bit for bit."""
    n = 1 << 26
    g = torch.Generator(device="cuda").manual_seed(1234)
    xs = [torch.rand(n, dtype=torch.float64, device="cuda", generator=g) * 9.0,
          torch.rand(n, dtype=torch.float64, device="cuda", generator=g),
          # sums of 9 cells of [0,1) values and their ulp neighbourhoods
          torch.rand(n, dtype=torch.float64, device="cuda", generator=g) * 9.0 + 1e-300]
    specials = torch.tensor([0.0, 9.0, 1.0, 4.5, 8.999999999999998, 2.0 ** -1000, 1e-310, 3.0,
                             27.0, 81.0, 6.0, 0.1111111111111111], dtype=torch.float64, device="cuda")
    ints = torch.arange(0, 1 << 20, dtype=torch.float64, device="cuda")
    # exact multiples of 9 and near-midpoint quotients
    mult = ints * 9.0
    bits = torch.randint(0, 1 << 52, (n,), generator=g, device="cuda", dtype=torch.int64)
    dense = (bits | (1023 << 52)).view(torch.float64) * 8.0  # [8, 16): every mantissa pattern
    for x in xs + [specials, ints, mult, dense]:
        q = torch.empty_like(x)
        r = torch.empty_like(x)
        s = torch.cuda.current_stream().cuda_stream
        P._check(P.lib().pcotgpu_test_div9(ctypes.c_void_p(x.data_ptr()), ctypes.c_void_p(q.data_ptr()),
                                           ctypes.c_void_p(r.data_ptr()), x.numel(), ctypes.c_void_p(s)))
        torch.cuda.synchronize()
        assert torch.equal(q.view(torch.int64), r.view(torch.int64))


def test_sharded_slabs_equal_single_grid_on_one_gpu():
    """The row-sharded driver's slab kernel on sub-ranges of rows (as the
    multi-GPU path launches it: boundary strips + interior) reproduces the
    single-launch result bit for bit."""
    from paper_1802_00166_b200.sharded import ShardedStencil2D

    N, T, bt = 1000, 40, 6
    dev = torch.device("cuda", 0)
    S = ShardedStencil2D(N, N, T, bt, device=dev)
    S.fill_init("F")
    S.snapshot_input()
    S.run()
    full = S.interior(S.cur).cpu().numpy().copy()
    want = O.reference_output("jacobi2d", {"T": T, "N": N}).reshape(N, N)
    assert np.array_equal(full.view(np.uint64), want.view(np.uint64))
    # same run, every block split into three launches over row ranges
    S.restart()
    t = 0
    while t < T:
        step = min(bt, T - t)
        src, dst = S.cur, S.cur ^ 1
        stream = torch.cuda.current_stream()
        for lo, hi in [(0, step), (N - step, N), (step, N - step)]:
            S.advance(src, dst, lo, hi, step, stream)
        S.cur = dst
        t += step
    split = S.interior(S.cur).cpu().numpy()
    assert np.array_equal(split.view(np.uint64), want.view(np.uint64))


@pytest.mark.parametrize("variant", [0, 1, 2, 3, 4, 10, 11, 12, 13, 14, 15, 16, 17, 18, 19, 20, 21, 22, 23, 24, 25, 26, 27, 28, 29, 30, 31])
def test_s3d7_variants_bit_exact(variant):
    """Every compiled (C, RJ, NW) variant of the 3-D kernel, all depths, both rules."""
    import subprocess
    import sys

    code = (
        "import numpy as np, paper_1802_00166_b200 as P\n"
        "from tests import oracle_ctypes as O\n"
        "for k in ('heat3d_b', 'heat3d'):\n"
        "    want = O.reference_output(k, {'T': 9, 'N': 77})\n"
        "    with P.GpuExecutor(O.kernel_path(k), {'T': 9, 'N': 77}) as ex:\n"
        "        for bt in range(1, 5):\n"
        "            for sch in ('slt', 'cot'):\n"
        "                ex.run(sch, [bt, 8, 8, 8], skip_checksum=True)\n"
        "                out = ex.array_data('Out')\n"
        "                assert np.array_equal(out.view(np.uint64), want.view(np.uint64)), (k, bt, sch)\n"
        "print('ok')\n")
    env = dict(**__import__("os").environ, PCOTGPU_S3D7_VARIANT=str(variant))
    p = subprocess.run([sys.executable, "-c", code], cwd=O.REPO, env=env, capture_output=True,
                       text=True, timeout=600)
    assert p.returncode == 0 and "ok" in p.stdout, p.stdout + p.stderr


@pytest.mark.parametrize("variant", list(range(16)))
def test_s2d5_variants_bit_exact(variant, monkeypatch):
    """Every compiled (C, NT, MINB) variant of the 2-D kernel (12-15: six
    columns per thread), all depths, zero ring (jacobi2d) and held ring (heat2d)."""
    import subprocess
    import sys

    code = (
        "import numpy as np, paper_1802_00166_b200 as P\n"
        "from tests import oracle_ctypes as O\n"
        "want = O.reference_output('jacobi2d', {'T': 24, 'N': 777})\n"
        "with P.GpuExecutor('jacobi2d', {'T': 24, 'N': 777}) as ex:\n"
        "    for bt in range(1, 9):\n"
        "        ex.run('slt', [bt, 8, 8], skip_checksum=True)\n"
        "        out = ex.array_data('Out')\n"
        "        assert np.array_equal(out.view(np.uint64), want.view(np.uint64)), bt\n"
        "want = O.reference_output('heat2d_hold', {'T': 19, 'N': 301})\n"
        "with P.GpuExecutor(O.kernel_path('heat2d_hold'), {'T': 19, 'N': 301}) as ex:\n"
        "    for bt in range(1, 9):\n"
        "        ex.run('cot', [bt, 8, 8], skip_checksum=True)\n"
        "        out = ex.array_data('Out')\n"
        "        assert np.array_equal(out.view(np.uint64), want.view(np.uint64)), ('hold', bt)\n"
        "print('ok')\n")
    env = dict(**__import__("os").environ, PCOTGPU_S2D5_VARIANT=str(variant))
    p = subprocess.run([sys.executable, "-c", code], cwd=O.REPO, env=env, capture_output=True,
                       text=True, timeout=600)
    assert p.returncode == 0 and "ok" in p.stdout, p.stdout + p.stderr


@pytest.mark.parametrize("env", [{}, {"PCOTGPU_PDL": "0"}, {"PCOTGPU_S2D5_CHUNKS": "1"},
                                 {"PCOTGPU_S2D5_CHUNKS": "333", "PCOTGPU_S3D7_CHUNKS": "29"}])
def test_launch_modes_bit_exact(env):
    """Programmatic dependent launch on/off and extreme row chunkings leave every
    bit unchanged: an L2-resident grid (short chunks filling the resident
    slots), a multi-wave HBM-streaming grid (> 2^24 cells, 13 back-to-back
    depth blocks) and the 3-D kernel."""
    import subprocess
    import sys

    code = (
        "import numpy as np, paper_1802_00166_b200 as P\n"
        "from tests import oracle_ctypes as O\n"
        "for k, prm, tiles in (('jacobi2d', {'T': 40, 'N': 2049}, ([8, 8, 8], [3, 8, 8])),\n"
        "                      ('jacobi2d', {'T': 13, 'N': 4500}, ([6, 8, 8], [1, 8, 8])),\n"
        "                      ('heat3d_b', {'T': 11, 'N': 97}, ([2, 8, 8, 8], [3, 8, 8, 8]))):\n"
        "    want = O.reference_output(k, prm)\n"
        "    with P.GpuExecutor(k, prm) as ex:\n"
        "        for tile in tiles:\n"
        "            ex.run('slt', tile, skip_checksum=True)\n"
        "            out = ex.array_data('Out')\n"
        "            assert np.array_equal(out.view(np.uint64), want.view(np.uint64)), (k, tile)\n"
        "print('ok')\n")
    e = dict(**__import__("os").environ, **env)
    p = subprocess.run([sys.executable, "-c", code], cwd=O.REPO, env=e, capture_output=True,
                       text=True, timeout=900)
    assert p.returncode == 0 and "ok" in p.stdout, p.stdout + p.stderr


def test_p2p_halo_mirror_stores_equal_single_grid():
    """The fused halo exchange of `ShardedStencil2D(halo="p2p")` on one GPU: two
    row shards in one process, each launch also storing its first/last bt
    output rows into the other shard's ghost rows (`pcotgpu_s2d5_advance_p2p`,
    addresses from `sharded.mirror_targets`), launches stream-ordered (no
    kernel waits on another).  No ghost row is copied after the start, so the
    result equals the single grid only if every mirror store lands in place."""
    import ctypes

    import torch

    from paper_1802_00166_b200.sharded import layout, mirror_targets

    N, T, bt = 600, 20, 6
    R = N // 2
    ld, ghost, padl, total = layout(R, N)
    dev = torch.device("cuda", 0)
    s = torch.cuda.current_stream(dev)
    lib = P.lib()
    buf = [[torch.zeros(total, dtype=torch.float64, device=dev) for _ in range(2)] for _ in range(2)]
    org = lambda k, b: buf[k][b].data_ptr() + (ghost * ld + padl) * 8  # noqa: E731
    for k in range(2):
        P._check(lib.pcotgpu_fill_init_value(ctypes.c_void_p(org(k, 0)), ld, R, N, b"F", k * R * N,
                                             ctypes.c_void_p(s.cuda_stream)))
        P._check(lib.pcotgpu_s2d5_prepare(ctypes.c_void_p(org(k, 0)), R, N, k * R, N, 0,
                                          ctypes.c_void_p(s.cuda_stream)))
    rows = lambda k, b, r0, r1: buf[k][b][(ghost + r0) * ld:(ghost + r1) * ld]  # noqa: E731
    rows(0, 0, R, R + ghost).copy_(rows(1, 0, 0, ghost))   # initial ghosts only
    rows(1, 0, -ghost, 0).copy_(rows(0, 0, R - ghost, R))
    cur, t = 0, 0
    while t < T:
        step = min(bt, T - t)
        for k in range(2):
            up, dn = mirror_targets(org(0, cur ^ 1) if k == 1 else None,
                                    org(1, cur ^ 1) if k == 0 else None, R, ld)
            P._check(lib.pcotgpu_s2d5_advance_p2p(
                ctypes.c_void_p(org(k, cur)), ctypes.c_void_p(org(k, cur ^ 1)), R, N, k * R, N, step,
                0, 0, 0, R, ctypes.c_void_p(up), ctypes.c_void_p(dn), step,
                ctypes.c_void_p(s.cuda_stream)))
        cur ^= 1
        t += step
    got = torch.cat([rows(k, cur, 0, R).view(R, ld)[:, padl:padl + N] for k in range(2)]).cpu().numpy()
    want = O.reference_output("jacobi2d", {"T": T, "N": N}).reshape(N, N)
    assert np.array_equal(got.view(np.uint64), want.view(np.uint64))


def test_sharded_p2p_mode_runs_through_symmetric_memory():
    """`ShardedStencil2D(halo="p2p")` at world size 1 (NCCL group of one): the
    symmetric-memory allocation, rendezvous, kernel launches with (null)
    mirrors and the per-block device barrier all run; result = oracle."""
    import subprocess
    import sys

    code = (
        "import os, numpy as np, torch, torch.distributed as dist\n"
        "os.environ.update(MASTER_ADDR='127.0.0.1', MASTER_PORT='29547', RANK='0', WORLD_SIZE='1')\n"
        "dev = torch.device('cuda', 0); torch.cuda.set_device(dev)\n"
        "dist.init_process_group('nccl', device_id=dev)\n"
        "from paper_1802_00166_b200.sharded import ShardedStencil2D\n"
        "from tests import oracle_ctypes as O\n"
        "N, T = 515, 23\n"
        "S = ShardedStencil2D(N, N, T, 6, device=dev, halo='p2p')\n"
        "assert S.p2p and len(S.symm) == 2\n"
        "S.fill_init('F'); S.run(); torch.cuda.synchronize()\n"
        "got = S.interior(S.cur).cpu().numpy()\n"
        "want = O.reference_output('jacobi2d', {'T': T, 'N': N}).reshape(N, N)\n"
        "assert np.array_equal(got.view(np.uint64), want.view(np.uint64))\n"
        "dist.destroy_process_group()\n"
        "print('ok')\n")
    p = subprocess.run([sys.executable, "-c", code], cwd=O.REPO, capture_output=True, text=True,
                       timeout=600)
    assert p.returncode == 0 and "ok" in p.stdout, p.stdout + p.stderr


def test_executors_on_concurrent_host_threads():
    """Distinct executors may run concurrently (reference sweep.cpp:82-128 runs one
    Executor per worker thread): four host threads, each with its own executor and
    kernel family, first launches racing on the per-(kernel, device) launch caches
    (kernel_slots) — every result equals the reference golden."""
    import threading

    from tests import oracle_ctypes as O

    cases = [("jacobi2d", {"T": 40, "N": 1000}), ("heat3d_b", {"T": 20, "N": 130}),
             ("gs2d", {"T": 16, "N": 1024}), ("jacobi2d", {"T": 64, "N": 1024})]
    want = {}
    for k, p in cases:
        want[(k, str(p))] = [e["checksum"] for e in O.goldens() if e["kernel"] == k and e["params"] == p][0]
    got, errors = {}, []
    start = threading.Barrier(len(cases))

    def work(k, p):
        try:
            with P.GpuExecutor(k, p) as ex:
                start.wait()
                for _ in range(3):
                    got.setdefault((k, str(p)), set()).add(ex.run("cot", None).checksum_hex)
        except Exception as e:  # surfaced below
            errors.append(repr(e))

    th = [threading.Thread(target=work, args=c) for c in cases]
    for t in th:
        t.start()
    for t in th:
        t.join(timeout=300)
    assert not errors, errors
    for key, w in want.items():
        assert got[key] == {w}, key


# ---------------------------------------------------------------- resident 2-D stencil
@pytest.mark.parametrize("kernel", ["jacobi2d", "heat2d_hold"])
@pytest.mark.parametrize("N,T", [(64, 4), (100, 7), (127, 9), (130, 16), (296, 5), (500, 33),
                                 (1000, 40), (1024, 12), (2047, 6), (2048, 10)])
def test_resident_stencil_matches_oracle(monkeypatch, kernel, N, T):
    """The on-chip resident kernel (PCOTGPU_RESIDENT=1, untiled schedule of
    grids up to 2048^2, stencil2d_res.cu) against the oracle, bit for bit:
    ragged widths, bands of 2..14 rows, odd and even step counts; and the
    streaming kernel on the same executor gives the same bits."""
    monkeypatch.setenv("PCOTGPU_RESIDENT", "1")
    want = O.reference_output(kernel, {"T": T, "N": N})
    with P.GpuExecutor(kernel, {"T": T, "N": N}) as ex:
        r = ex.run_untiled()
        assert r.bt == 0 and r.launches <= 4  # one persistent launch (+ copy-in, ring, flags)
        out = ex.array_data("Out")
        assert np.array_equal(out.view(np.uint64), want.view(np.uint64))
        monkeypatch.setenv("PCOTGPU_RESIDENT", "0")
        r2 = ex.run_untiled()
        assert r2.bt > 0 and r2.checksum_hex == r.checksum_hex


def test_resident_stencil_config0_golden_repeated(monkeypatch):
    """BASELINE config 0 through the resident kernel, three runs on one
    executor (flags and exchange lines are re-armed per run; a band-to-band
    ordering race would show as a flaky checksum)."""
    monkeypatch.setenv("PCOTGPU_RESIDENT", "1")
    want = [e["checksum"] for e in O.goldens()
            if e["kernel"] == "jacobi2d" and e["params"] == {"T": 256, "N": 2048}][0]
    with P.GpuExecutor("jacobi2d", {"T": 256, "N": 2048}) as ex:
        for _ in range(3):
            r = ex.run_untiled()
            assert r.bt == 0 and r.checksum_hex == want
