cd $GRAFT_REPO_ROOT
timeout 900 python -m pytest tests/test_gpu_kernels.py tests/test_gpu_parity.py -q -m gpu -x -k "variants or jacobi or heat2d or sharded or storage or host" > gpurun_out/pytest_v.log 2>&1; echo "pytest rc=$?" >> gpurun_out/pytest_v.log
for v in 5 6 8; do echo "variant $v"; PCOTGPU_S2D5_VARIANT=$v timeout 300 python tools/kbench.py s2d5 --bts 3,4,5,6,7 --orders slt 2>&1 | grep -v Warn; done > gpurun_out/kb_variants5.log 2>&1
tail -3 gpurun_out/pytest_v.log; cat gpurun_out/kb_variants5.log
