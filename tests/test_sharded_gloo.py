"""CPU, world_size 2 (gloo): the row-sharded driver's exchange logic.

Each rank owns half the rows of an N x N zero-ring Jacobi grid with ghost
rows; ShardedStencil2D sends/receives bt boundary rows every temporal block.
The slab kernel is replaced by a CPU restatement of one bt-step block (test
infrastructure); the gathered result must equal the oracle's single-grid run
bit for bit, which exercises ghost depth, ring rows at the global edges, the
last (shorter) block and the initial exchange.
"""
import os

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

from tests import oracle_ctypes as O


def cpu_block(S, src, dst, row_lo, row_hi, bt):
    """bt Jacobi steps on local rows [row_lo, row_hi) of S from buffer src to dst."""
    ld, g, pl, R, C = S.ld, S.ghost, S.padl, S.R, S.cols
    a = S.buf[src].view(R + 2 * g, ld)[:, pl:pl + C].clone()  # rows -g .. R+g-1
    rows = torch.arange(-g, R + g) + S.g0
    cols = torch.arange(C)
    interior = ((rows >= 1) & (rows <= S.nrows - 2))[:, None] & ((cols >= 1) & (cols <= C - 2))[None, :]
    for _ in range(bt):
        b = torch.zeros_like(a)
        mid = a[1:-1, 1:-1]
        s = mid + a[:-2, 1:-1]
        s = s + a[2:, 1:-1]
        s = s + a[1:-1, :-2]
        s = s + a[1:-1, 2:]
        b[1:-1, 1:-1] = 0.2 * s
        a = torch.where(interior, b, torch.zeros_like(b))
    out = S.buf[dst].view(R + 2 * g, ld)[:, pl:pl + C]
    out[g + row_lo:g + row_hi] = a[g + row_lo:g + row_hi]


def _geometry(N, R):
    return (N + 16, 12, 4, (R + 24) * (N + 16))


def _mirror_emulation(S, rank, world, peers, delay):
    """CPU stand-in for pcotgpu_s2d5_advance_p2p: compute the owned rows, then
    store the first / last bt output rows into the neighbours' ghost rows of
    `dst`, at the element offsets mirror_targets gives (peers[k][b] = rank k's
    shared-memory slab b)."""
    import time

    from paper_1802_00166_b200.sharded import mirror_targets

    org = S.origin_offset()

    def adv(src, dst, bt, stream):
        cpu_block(S, src, dst, 0, S.R, bt)
        if delay and rank == 0:
            time.sleep(delay)  # rank 1 runs ahead: without the barrier it reads stale ghosts
        up, dn = mirror_targets(org if rank > 0 else None, org if rank < world - 1 else None,
                                S.R, S.ld, elem=1)
        mine = S.buf[dst]
        for r in range(bt):
            if up is not None:
                peers[rank - 1][dst][up + r * S.ld:up + r * S.ld + S.cols] = \
                    mine[org + r * S.ld:org + r * S.ld + S.cols]
            rr = S.R - bt + r
            if dn is not None:
                peers[rank + 1][dst][dn + rr * S.ld:dn + rr * S.ld + S.cols] = \
                    mine[org + rr * S.ld:org + rr * S.ld + S.cols]
    return adv


def worker(rank, world, port, N, T, bt, q, mode="nccl", peers=None, delay=0.0):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    from paper_1802_00166_b200.sharded import ShardedStencil2D

    R = N // world
    calls = []
    if mode == "nccl" or mode == "late-sends":
        S = ShardedStencil2D(R, N, T, bt, advance=None, geometry=_geometry(N, R))
        if mode == "late-sends":  # negative control: rows posted before the edge strips are computed
            def bad_block(bt_, record=False, S=S):
                src, dst = S.cur, S.cur ^ 1
                reqs = dist.batch_isend_irecv(S._ops(dst, bt_))
                for r in reqs:
                    r.wait()
                S.advance(src, dst, 0, S.R, bt_, None)
                S.cur = dst
            S.block = bad_block
    else:
        S = ShardedStencil2D(R, N, T, bt, advance=None, geometry=_geometry(N, R), halo="p2p",
                             buffers=peers[rank], advance_p2p=lambda *a: None,
                             barrier=(lambda b: dist.barrier()) if mode == "p2p" else (lambda b: None))
        S.advance_p2p = _mirror_emulation(S, rank, world, peers, delay)

    def adv(src, dst, lo, hi, b, stream):
        calls.append((lo, hi))
        cpu_block(S, src, dst, lo, hi, b)
    S.advance = adv
    F = torch.from_numpy(O.init_array("F", N * N).reshape(N, N))
    F0 = F[rank * R:(rank + 1) * R].clone()
    if rank == 0:
        F0[0] = 0.0
    if rank == world - 1:
        F0[-1] = 0.0
    F0[:, 0] = 0.0
    F0[:, -1] = 0.0
    S.load(F0)
    S.run()
    mine = S.interior(S.cur).contiguous()
    parts = [torch.empty_like(mine) for _ in range(world)]
    dist.all_gather(parts, mine)
    if rank == 0:
        q.put((torch.cat(parts).numpy(), calls))
    dist.barrier()
    dist.destroy_process_group()


def _run(N, T, bt, mode="nccl", delay=0.0):
    world = 2
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = 29500 + (os.getpid() + N + T + 7 * len(mode)) % 2000
    peers = None
    if mode.startswith("p2p"):
        R = N // world
        geo = _geometry(N, R)
        peers = [[torch.zeros(geo[3], dtype=torch.float64).share_memory_() for _ in range(2)]
                 for _ in range(world)]
    procs = [ctx.Process(target=worker, args=(r, world, port, N, T, bt, q, mode, peers, delay))
             for r in range(world)]
    for p in procs:
        p.start()
    got, calls = q.get(timeout=120)
    for p in procs:
        p.join(timeout=120)
        assert p.exitcode == 0
    want = O.reference_output("jacobi2d", {"T": T, "N": N}).reshape(N, N)
    return np.array_equal(got.view(np.uint64), want.view(np.uint64)), calls


@pytest.mark.parametrize("N,T,bt", [(64, 13, 4), (48, 7, 3), (40, 1, 1)])
def test_two_rank_halo_exchange_matches_single_grid(N, T, bt):
    """The overlapped sequence itself (edge strips, sends posted, interior,
    receives waited) — the code path the GPUs run — on CPU lanes."""
    ok, calls = _run(N, T, bt)
    assert ok
    R, e = N // 2, bt
    blocks = -(-T // bt)
    assert calls[:3] == [(0, e), (R - e, R), (e, R - e)]  # edges first, then the interior
    assert len(calls) == 3 * blocks


def test_exchange_ordering_is_what_makes_it_exact():
    """Negative control: posting the boundary rows before the edge strips are
    computed (stale rows reach the neighbour) must break bit-exactness."""
    ok, _ = _run(64, 13, 4, mode="late-sends")
    assert not ok


@pytest.mark.parametrize("N,T,bt", [(64, 13, 4), (40, 9, 2)])
def test_p2p_mode_ordering_with_emulated_mirror_stores(N, T, bt):
    """halo="p2p": one fused advance per block (mirror stores of the first/last
    bt rows into the neighbours' ghost rows, emulated into shared memory at
    mirror_targets' offsets), then the barrier — equal to the single grid."""
    ok, calls = _run(N, T, bt, mode="p2p", delay=0.02)
    assert ok
    assert calls == []  # no separate edge / interior launches in this mode


def test_p2p_mode_needs_its_barrier():
    """Negative control: without the per-block barrier a rank reads ghost rows
    its neighbour has not stored yet."""
    ok, _ = _run(64, 13, 4, mode="p2p-nobarrier", delay=0.2)
    assert not ok


def test_p2p_mirror_targets_address_neighbour_ghost_rows():
    """halo="p2p": output row r of rank k, stored at mirror + (r*ld + c)*8, must be
    the upper neighbour's row R + r (r < bt) and the lower neighbour's row r - R
    (r >= R - bt) — the rows the NCCL path sends (`_ops`)."""
    from paper_1802_00166_b200.sharded import mirror_targets

    R, ld, bt = 40, 96, 5
    up_origin, dn_origin = 1 << 30, 1 << 34
    up, dn = mirror_targets(up_origin, dn_origin, R, ld)
    for r in range(bt):
        assert up + (r * ld + 7) * 8 == up_origin + ((R + r) * ld + 7) * 8
    for r in range(R - bt, R):
        assert dn + (r * ld + 7) * 8 == dn_origin + ((r - R) * ld + 7) * 8
    assert mirror_targets(None, None, R, ld) == (None, None)


def test_halo_mode_is_validated():
    from paper_1802_00166_b200.sharded import ShardedStencil2D

    with pytest.raises(ValueError):
        ShardedStencil2D(16, 16, 4, 2, halo="udp", geometry=(16, 8, 2, 16 * 32))
