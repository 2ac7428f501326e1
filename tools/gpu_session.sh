cd $GRAFT_REPO_ROOT
timeout 900 python -m pytest tests/test_gpu_kernels.py tests/test_gpu_parity.py -q -m gpu -x -k "s3d7 or heat3d or smoke" > gpurun_out/pytest_s3.log 2>&1; echo "pytest rc=$?" >> gpurun_out/pytest_s3.log
for v in 0 1 2 3 4; do echo "variant $v"; PCOTGPU_S3D7_VARIANT=$v timeout 300 python tools/kbench.py s3d7 --bts 1,2,3,4 2>&1 | grep -v Warn | paste - - ; done > gpurun_out/kb_s3v.log 2>&1
tail -3 gpurun_out/pytest_s3.log; cat gpurun_out/kb_s3v.log
