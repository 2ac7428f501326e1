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


def worker(rank, world, port, N, T, bt, q):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    from paper_1802_00166_b200.sharded import ShardedStencil2D

    R = N // world
    S = ShardedStencil2D(R, N, T, bt, advance=None, geometry=(N + 16, 12, 4, (R + 24) * (N + 16)))
    S.advance = lambda src, dst, lo, hi, b, stream: cpu_block(S, src, dst, lo, hi, b)
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
        q.put(torch.cat(parts).numpy())
    dist.barrier()
    dist.destroy_process_group()


@pytest.mark.parametrize("N,T,bt", [(64, 13, 4), (48, 7, 3), (40, 1, 1)])
def test_two_rank_halo_exchange_matches_single_grid(N, T, bt):
    world = 2
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = 29500 + (os.getpid() + N + T) % 2000
    procs = [ctx.Process(target=worker, args=(r, world, port, N, T, bt, q)) for r in range(world)]
    for p in procs:
        p.start()
    got = q.get(timeout=300)
    for p in procs:
        p.join(timeout=120)
        assert p.exitcode == 0
    want = O.reference_output("jacobi2d", {"T": T, "N": N}).reshape(N, N)
    assert np.array_equal(got.view(np.uint64), want.view(np.uint64))


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
