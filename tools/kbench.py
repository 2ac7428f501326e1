#!/usr/bin/env python3
"""Kernel-level timing sweeps (CUDA events, warm, no profiler).

    python tools/kbench.py s2d5 [--rows R --cols C --bts 1,2,...]
    python tools/kbench.py s3d7 [--n 384 --bts 1,2,3,4]
    python tools/kbench.py jac  [--n 2048 --T 256 --bts 2,4,6]   (executor, jacobi2d)
    python tools/kbench.py gs   [--n 4096 --T 64 --tiles 4x32x256,...]
    python tools/kbench.py gemm [--n 4096]
"""
import argparse
import json
import os
import sys

REPO = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, REPO)

import torch  # noqa: E402

import paper_1802_00166_b200 as P  # noqa: E402


def ev_time(fn, reps=3):
    s = torch.cuda.current_stream()
    fn()
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record(s)
    for _ in range(reps):
        fn()
    e1.record(s)
    torch.cuda.synchronize()
    return e0.elapsed_time(e1) / reps


def s2d5(a):
    from paper_1802_00166_b200.sharded import ShardedStencil2D

    S = ShardedStencil2D(a.rows, a.cols, 8, 8, device=torch.device("cuda", 0))
    S.fill_init("F")
    cells = a.rows * a.cols
    orders = [0] if a.orders == "slt" else [1] if a.orders == "cot" else [0, 1]
    for bt in [int(x) for x in a.bts.split(",")]:
        for order in orders:
            S.order = order

            def one():
                S.advance(0, 1, 0, S.R, bt, torch.cuda.current_stream())
            ms = ev_time(one, a.reps)
            print(json.dumps({"kernel": "s2d5", "bt": bt, "order": "slt" if order == 0 else "cot",
                              "ms": round(ms, 4), "GUpd/s": round(cells * bt / ms / 1e6, 1),
                              "GB/s(16B/cell)": round(16 * cells / ms / 1e6, 1)}), flush=True)


def executor(a, kernel, params, tiles):
    with P.GpuExecutor(kernel, params) as ex:
        for tile in tiles:
            ex.run("slt", tile, skip_checksum=True)
            rs = [ex.run("slt", tile, skip_checksum=True) for _ in range(a.reps)]
            ms = sorted(r.device_ms for r in rs)[len(rs) // 2]
            print(json.dumps({"kernel": kernel, "params": params, "tile": tile, "bt": rs[0].bt,
                              "ms": round(ms, 3), "launches": rs[0].launches}), flush=True)
            yield ms


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("which")
    ap.add_argument("--rows", type=int, default=32768)
    ap.add_argument("--cols", type=int, default=32768)
    ap.add_argument("--bts", default="1,2,3,4,5,6,7,8")
    ap.add_argument("--n", type=int, default=0)
    ap.add_argument("--T", type=int, default=0)
    ap.add_argument("--tiles", default="")
    ap.add_argument("--reps", type=int, default=3)
    ap.add_argument("--orders", default="both")
    a = ap.parse_args()
    torch.cuda.set_device(0)
    if a.which == "s2d5":
        s2d5(a)
    elif a.which == "s3d7":
        n, T = a.n or 384, a.T or 100
        tiles = [[int(b), 8, 8, 8] for b in a.bts.split(",") if int(b) <= 4]
        for ms in executor(a, "heat3d_b", {"T": T, "N": n}, tiles):
            print("  GUpd/s %.1f" % (n ** 3 * T / ms / 1e6))
    elif a.which == "jac":
        n, T = a.n or 2048, a.T or 256
        tiles = [[int(b), 8, 8] for b in a.bts.split(",")]
        for ms in executor(a, "jacobi2d", {"T": T, "N": n}, tiles):
            print("  GUpd/s %.1f" % (n * n * T / ms / 1e6))
    elif a.which == "gs":
        n, T = a.n or 4096, a.T or 64
        tiles = [[int(v) for v in t.split("x")] for t in (a.tiles or "4x32x256").split(",")]
        for ms in executor(a, "gs2d", {"T": T, "N": n}, tiles):
            print("  GUpd/s %.1f" % (n * n * T / ms / 1e6))
    elif a.which == "gemm":
        n = a.n or 4096
        for ms in executor(a, "gemm", {"N": n}, [[16, 16, 16]]):
            print("  GFLOP/s %.1f" % (2 * n ** 3 / ms / 1e6))


if __name__ == "__main__":
    main()
