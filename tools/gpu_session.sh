cd $GRAFT_REPO_ROOT
timeout 900 python -m pytest tests/test_gpu_kernels.py tests/test_gpu_parity.py -q -m gpu -x -k "s2d5 or jacobi or heat2d or sharded or storage or host" > gpurun_out/pytest_s2c.log 2>&1; echo "pytest rc=$?" >> gpurun_out/pytest_s2c.log
timeout 300 python tools/kbench.py s2d5 --bts 4,5,6,7,8 --orders slt > gpurun_out/kb_auto.log 2>&1
timeout 600 python bench.py --no-cpu-baseline --no-e2e --steps 3 --warmup 2 2>&1 | tail -1 > gpurun_out/bench4.log
tail -2 gpurun_out/pytest_s2c.log; cat gpurun_out/kb_auto.log; cut -c1-200 gpurun_out/bench4.log
