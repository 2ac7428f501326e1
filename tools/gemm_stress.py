"""Repeat small GEMM executor runs and count results outside 1e-12 (race hunt)."""
import sys

import numpy as np

sys.path.insert(0, ".")
import paper_1802_00166_b200 as P  # noqa: E402
from tests import oracle_ctypes as O  # noqa: E402

reps = int(sys.argv[1]) if len(sys.argv) > 1 else 100
for N in (33, 64, 96, 130, 257):
    A = O.init_array("A", N * N)
    B = O.init_array("B", N * N)
    ref = O.gemm(N, A, B, None).reshape(N, N)
    for scheme in ("cot", "slt"):
        bad = 0
        worst = 0.0
        for _ in range(reps):
            with P.GpuExecutor("gemm", {"N": N}) as ex:
                ex.run(scheme, [16, 16, 16])
                got = ex.array_data("Out").reshape(N, N)
            err = np.linalg.norm(got - ref) / np.linalg.norm(ref)
            worst = max(worst, err)
            bad += err > 1e-12
        print("N", N, scheme, "bad", bad, "of", reps, "worst %.3g" % worst, flush=True)
