"""One executor run of a kernel (profiling helper): python tools/one_run.py KERNEL T N [reps]
(T is ignored for gemm).  Default schedule, checksum printed."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_1802_00166_b200 as P  # noqa: E402

k, T, N = sys.argv[1], int(sys.argv[2]), int(sys.argv[3])
reps = int(sys.argv[4]) if len(sys.argv) > 4 else 3
params = {"N": N} if k == "gemm" else {"T": T, "N": N}
with P.GpuExecutor(k, params) as ex:
    for i in range(reps):
        r = ex.run_untiled(skip_checksum=(i + 1 < reps))
    print(k, params, "bt", r.bt, "%.3f ms" % r.device_ms, r.checksum_hex, "launches", r.launches)
