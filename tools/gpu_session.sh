cd $GRAFT_REPO_ROOT
timeout 900 python -m pytest tests/test_gpu_kernels.py tests/test_gpu_parity.py -q -m gpu -x > gpurun_out/pytest_gpu3.log 2>&1; echo "pytest rc=$?" >> gpurun_out/pytest_gpu3.log
for v in 0 3; do echo "variant $v"; PCOTGPU_S2D5_VARIANT=$v timeout 300 python tools/kbench.py s2d5 --bts 4,5,6,7,8 --orders slt 2>&1 | grep -v Warn; done > gpurun_out/kb_variants2.log 2>&1
timeout 300 python tools/kbench.py gs --tiles 8x64x128,16x64x128,8x128x64,16x32x256,4x128x128,32x32x128 > gpurun_out/kb_gs2.log 2>&1
timeout 600 python bench.py --steps 3 --warmup 2 > gpurun_out/bench2.log 2>&1; echo "bench rc=$?" >> gpurun_out/bench2.log
tail -4 gpurun_out/pytest_gpu3.log; cat gpurun_out/kb_variants2.log gpurun_out/kb_gs2.log; tail -2 gpurun_out/bench2.log
