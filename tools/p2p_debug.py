"""Debug aid: two row shards on one GPU with P2P mirror stores vs the oracle;
prints where they differ (mode 'mirror') or the same with host ghost copies
after every block (mode 'copy')."""
import ctypes
import sys

import numpy as np
import torch

sys.path.insert(0, ".")
import paper_1802_00166_b200 as P  # noqa: E402
from paper_1802_00166_b200.sharded import layout, mirror_targets  # noqa: E402
from tests import oracle_ctypes as O  # noqa: E402

mode = sys.argv[1]
N, T, bt = 600, int(sys.argv[2]), 6
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
rows(0, 0, R, R + ghost).copy_(rows(1, 0, 0, ghost))
rows(1, 0, -ghost, 0).copy_(rows(0, 0, R - ghost, R))
cur, t = 0, 0
while t < T:
    step = min(bt, T - t)
    for k in range(2):
        up, dn = mirror_targets(org(0, cur ^ 1) if k == 1 else None,
                                org(1, cur ^ 1) if k == 0 else None, R, ld)
        if mode == "copy":
            up = dn = None
        P._check(lib.pcotgpu_s2d5_advance_p2p(
            ctypes.c_void_p(org(k, cur)), ctypes.c_void_p(org(k, cur ^ 1)), R, N, k * R, N, step,
            0, 0, 0, R, ctypes.c_void_p(up), ctypes.c_void_p(dn), step if mode == "mirror" else 0,
            ctypes.c_void_p(s.cuda_stream)))
    if mode == "copy":
        rows(0, cur ^ 1, R, R + step).copy_(rows(1, cur ^ 1, 0, step))
        rows(1, cur ^ 1, -step, 0).copy_(rows(0, cur ^ 1, R - step, R))
    cur ^= 1
    t += step
got = torch.cat([rows(k, cur, 0, R).view(R, ld)[:, padl:padl + N] for k in range(2)]).cpu().numpy()
want = O.reference_output("jacobi2d", {"T": T, "N": N}).reshape(N, N)
bad = np.argwhere(got.view(np.uint64) != want.view(np.uint64))
print(mode, "T", T, "mismatches", len(bad))
if len(bad):
    print("rows", np.unique(bad[:, 0])[:40], "cols", np.unique(bad[:, 1])[:20])
    g1 = rows(1, cur, -bt, 0).view(bt, ld)[:, padl:padl + 8].cpu().numpy()
    print("B ghost rows above (first cols):", g1)
