cd $GRAFT_REPO_ROOT
timeout 600 python -m pytest tests/test_gpu_kernels.py tests/test_gpu_parity.py -q -m gpu -x -k "s2d5 or jacobi or heat2d" > gpurun_out/pytest_s2b.log 2>&1; echo "pytest rc=$?" >> gpurun_out/pytest_s2b.log
python - > gpurun_out/cfg0b.log 2>&1 <<'PY'
import os
import paper_1802_00166_b200 as P
with P.GpuExecutor("jacobi2d", {"T": 256, "N": 2048}) as ex:
    for bt in (2, 4, 6, 8):
        ex.run("slt", [bt, 64, 256], skip_checksum=True)
        rs = [ex.run("slt", [bt, 64, 256], skip_checksum=True) for _ in range(5)]
        ms = sorted(r.device_ms for r in rs)[2]
        print("cfg0 jacobi2d 2048^2 T=256 bt=%d: %.3f ms  %.1f GUpd/s" % (bt, ms, 2048*2048*256/ms/1e6))
PY
PCOTGPU_S2D5_VARIANT=10 python - >> gpurun_out/cfg0b.log 2>&1 <<'PY'
import paper_1802_00166_b200 as P
with P.GpuExecutor("jacobi2d", {"T": 256, "N": 2048}) as ex:
    for bt in (2, 4, 6, 8):
        ex.run("slt", [bt, 64, 256], skip_checksum=True)
        rs = [ex.run("slt", [bt, 64, 256], skip_checksum=True) for _ in range(5)]
        ms = sorted(r.device_ms for r in rs)[2]
        print("v10 cfg0 jacobi2d 2048^2 T=256 bt=%d: %.3f ms  %.1f GUpd/s" % (bt, ms, 2048*2048*256/ms/1e6))
PY
timeout 900 python -m paper_1802_00166_b200.sweep jacobi2d -p T=48,N=16384 --tiles 4x64x256,6x64x256 --schemes slt,cot --ncu --csv gpurun_out/sweep_jacobi.csv > gpurun_out/sweep_j.log 2>&1
timeout 900 python -m paper_1802_00166_b200.sweep gemm -p N=4096 --tiles 16x16x16 --schemes slt,cot --ncu --csv gpurun_out/sweep_gemm.csv > gpurun_out/sweep_g.log 2>&1
tail -2 gpurun_out/pytest_s2b.log; cat gpurun_out/cfg0b.log gpurun_out/sweep_j.log gpurun_out/sweep_g.log
