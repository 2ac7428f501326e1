"""Gauss-Seidel executor runs (profiling helper): python tools/gs_once.py T N [reps]

Prints device time and the output checksum (compare across PCOTGPU_GS_PIPE /
PCOTGPU_GS_PIPE_V settings; the tile kernel is the parity-tested baseline)."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_1802_00166_b200 as P  # noqa: E402

T, N = int(sys.argv[1]), int(sys.argv[2])
reps = int(sys.argv[3]) if len(sys.argv) > 3 else 1
with P.GpuExecutor("gs2d", {"T": T, "N": N}) as ex:
    best = None
    for _ in range(reps):
        ex.reset()
        r = ex.run_untiled()
        best = r.device_ms if best is None else min(best, r.device_ms)
    upd = (N - 2) ** 2 * T
    print("gs2d T=%d N=%d pipe=%s v=%s %.3f ms %.1f GUpd/s checksum=%016x" % (
        T, N, os.environ.get("PCOTGPU_GS_PIPE", "1"), os.environ.get("PCOTGPU_GS_PIPE_V", "1"),
        best, upd / best / 1e6, r.checksum))
