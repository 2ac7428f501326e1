cd $GRAFT_REPO_ROOT
./tools/fp64_peaks > gpurun_out/fp64_peaks.log 2>&1
timeout 300 python tools/kbench.py s2d5 > gpurun_out/kb_s2d5.log 2>&1
timeout 300 python tools/kbench.py s3d7 --bts 1,2,3,4 > gpurun_out/kb_s3d7.log 2>&1
timeout 300 python tools/kbench.py gs --tiles 4x32x256,8x32x256,4x64x256,8x64x128,2x32x512 > gpurun_out/kb_gs.log 2>&1
timeout 300 python tools/kbench.py gemm > gpurun_out/kb_gemm.log 2>&1
timeout 1200 python -m pytest tests/test_gpu_parity.py -q -m gpu -k "gs2d or gemm or storage or host or config4" > gpurun_out/pytest_gpu2.log 2>&1; echo "pytest rc=$?" >> gpurun_out/pytest_gpu2.log
cat gpurun_out/fp64_peaks.log gpurun_out/kb_*.log; tail -15 gpurun_out/pytest_gpu2.log
