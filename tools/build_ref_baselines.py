#!/usr/bin/env python3
"""Build the reference's compiled CPU path for the bench's CPU baseline.

CPU-BASELINE INFRASTRUCTURE (never the product): the reference's tiled CPU
path is its emitted recursive C (emit_c with use_alloc, reference
core/src/emit_c.cpp:342-380), compiled with the reference's own build line
`cc -std=c99 -O2 -ffp-contract=off -fopenmp` (tools/pcot.cpp:489-493).
oracle/_ref/pcot_ref (the unmodified reference library) emits the C here; the
binaries land in oracle/_ref/emit/ (git-ignored, shipped to the GPU box).

Each sample has an init-only twin (T=0) so the bench can subtract input
initialisation from the wall time, as BASELINE.md §3 prescribes.
"""
import json
import os
import subprocess
import sys

REPO = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
REF = os.path.join(REPO, "oracle", "_ref", "pcot_ref")
OUT = os.path.join(REPO, "oracle", "_ref", "emit")
GCC = "/usr/bin/gcc" if os.path.exists("/usr/bin/gcc") else "gcc"

# (tag, kernel, params, leaf sizes) — bounded samples of the BASELINE workloads
# (the leaf sizes are the binaries' defaults; they also take b0..bd-1 on argv,
# which the bench uses for its leaf sweep).  "_seq" = emitted without OpenMP.
SAMPLES = [
    ("jacobi2d_N8192_T160", "jacobi2d", {"T": 160, "N": 8192}, (16, 128, 1024)),
    ("jacobi2d_N8192_T0", "jacobi2d", {"T": 0, "N": 8192}, (1, 128, 1024)),
    ("jacobi2d_N4096_T32_seq", "jacobi2d", {"T": 32, "N": 4096}, (16, 128, 1024)),
    ("jacobi2d_N4096_T0_seq", "jacobi2d", {"T": 0, "N": 4096}, (1, 128, 1024)),
    ("jacobi2d_N2048_T256", "jacobi2d", {"T": 256, "N": 2048}, (32, 128, 512)),
    ("jacobi2d_N2048_T0", "jacobi2d", {"T": 0, "N": 2048}, (1, 128, 512)),
    ("heat3d_b_N384_T8", "heat3d_b", {"T": 8, "N": 384}, (8, 32, 32, 128)),
    ("heat3d_b_N384_T20", "heat3d_b", {"T": 20, "N": 384}, (8, 32, 32, 128)),
    ("heat3d_b_N384_T0", "heat3d_b", {"T": 0, "N": 384}, (1, 32, 32, 128)),
    ("gs2d_N4096_T8", "gs2d", {"T": 8, "N": 4096}, (8, 64, 1024)),
    ("gs2d_N4096_T16", "gs2d", {"T": 16, "N": 4096}, (16, 64, 1024)),
    ("gs2d_N4096_T0", "gs2d", {"T": 0, "N": 4096}, (1, 64, 1024)),
    ("gemm_N1024", "gemm", {"N": 1024}, (64, 64, 64)),
    ("gemm_N2048", "gemm", {"N": 2048}, (64, 64, 64)),
    ("gemm_N1", "gemm", {"N": 1}, (1, 1, 1)),
]


def main():
    if not os.path.exists(REF):
        sys.exit("oracle/_ref/pcot_ref missing: make -C oracle (needs /root/reference)")
    os.makedirs(OUT, exist_ok=True)
    manifest = {}
    for tag, kern, params, leaf in SAMPLES:
        c = os.path.join(OUT, tag + ".c")
        b = os.path.join(OUT, tag)
        pstr = ",".join("%s=%d" % kv for kv in params.items())
        kpath = os.path.join(REPO, "kernels", kern + ".kernel")
        if not os.path.exists(b) or os.path.getmtime(b) < os.path.getmtime(kpath):
            seq = tag.endswith("_seq")
            subprocess.run([REF, "emit", kpath, pstr] + ([] if seq else ["--openmp"]) +
                           ["--leaf", ",".join(map(str, leaf)), "-o", c], check=True)
            subprocess.run([GCC, "-std=c99", "-O2", "-ffp-contract=off"] +
                           ([] if seq else ["-fopenmp"]) + [c, "-lm", "-o", b], check=True)
        manifest[tag] = {"kernel": kern, "params": params, "leaf": list(leaf), "binary": b}
    with open(os.path.join(OUT, "manifest.json"), "w") as f:
        json.dump(manifest, f, indent=1)
    print("reference baselines in", OUT)


if __name__ == "__main__":
    main()
