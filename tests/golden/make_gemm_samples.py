#!/usr/bin/env python3
"""Sampled golden of BASELINE config 3 (gemm N=4096) from the UNMODIFIED reference.

TEST INFRASTRUCTURE (build container only; needs oracle/_ref/pcot_ref).  The
reference's emitted C for gemm.kernel at N=4096 (emit_c use_alloc + OpenMP,
built with the reference line `cc -std=c99 -O2 -ffp-contract=off -fopenmp`,
tools/pcot.cpp:489-493) is run with `--dump`; one entry per row i at column
j(i) = (i * 2654435761 + 12345) mod N is kept as its exact bit pattern,
together with (|2A-1| |2B-1|)_ij, the componentwise-error denominator
(SURVEY §8d).  bench.py checks its GEMM result on these 4096 cells; the GPU
test suite checks all 4096 rows against the oracle restatement.

    python tests/golden/make_gemm_samples.py   -> tests/golden/gemm4096_samples.json
"""
import json
import os
import re
import subprocess
import sys
import tempfile

import numpy as np

REPO = os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
sys.path.insert(0, REPO)
REF_BIN = os.path.join(REPO, "oracle", "_ref", "pcot_ref")
OUT = os.path.join(REPO, "tests", "golden", "gemm4096_samples.json")
GCC = "/usr/bin/gcc" if os.path.exists("/usr/bin/gcc") else "gcc"
N = 4096


def sample_col(i, n=N):
    return (i * 2654435761 + 12345) % n


def main():
    from tests import oracle_ctypes as O

    cols = [sample_col(i) for i in range(N)]
    want = {i * N + cols[i]: i for i in range(N)}
    vals = [None] * N
    with tempfile.TemporaryDirectory() as d:
        c, b = os.path.join(d, "g.c"), os.path.join(d, "g")
        subprocess.run([REF_BIN, "emit", os.path.join(REPO, "kernels", "gemm.kernel"), "N=%d" % N,
                        "--openmp", "--leaf", "64,64,64", "-o", c], check=True)
        subprocess.run([GCC, "-std=c99", "-O2", "-ffp-contract=off", "-fopenmp", c, "-lm", "-o", b],
                       check=True)
        p = subprocess.Popen([b, "--dump"], stdout=subprocess.PIPE, text=True, bufsize=1 << 20)
        checksum, flat, in_arr = None, 0, False
        for line in p.stdout:
            if in_arr:
                if flat in want:
                    vals[want[flat]] = line.strip()
                flat += 1
            elif line.startswith("CHECKSUM"):
                checksum = line.split()[1]
            elif line.startswith("ARRAY Out"):
                in_arr = True
        if p.wait() != 0 or flat != N * N:
            sys.exit("reference run failed (%d cells)" % flat)
    A = np.abs(2 * O.init_array("A", N * N) - 1).reshape(N, N)
    B = np.abs(2 * O.init_array("B", N * N) - 1).reshape(N, N)
    absab = [float(A[i] @ B[:, cols[i]]) for i in range(N)]
    with open(OUT, "w") as f:
        json.dump({"generator": "tests/golden/make_gemm_samples.py",
                   "source": "reference emitted C (emit_c use_alloc, -O2 -ffp-contract=off -fopenmp), "
                             "leaf [64,64,64], --dump",
                   "kernel": "gemm", "params": {"N": N}, "checksum": checksum,
                   "column_rule": "j(i) = (i * 2654435761 + 12345) mod N",
                   "out_hex": vals, "absab": absab}, f)
        f.write("\n")
    print("wrote", OUT, "checksum", checksum)


if __name__ == "__main__":
    main()
