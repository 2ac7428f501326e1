o=gpurun_out
rm -f $o/s5c_*.log
timeout 300 python -m pytest tests/test_gpu_kernels.py -m gpu -q -x -k resident > $o/s5c_res.log 2>&1; echo rc $? >> $o/s5c_res.log
timeout 120 python tools/one_run.py jacobi2d 256 2048 5 >> $o/s5c_time.log 2>&1
echo nosync >> $o/s5c_time.log
PCOTGPU_RES_NOSYNC=1 timeout 120 python tools/one_run.py jacobi2d 256 2048 5 >> $o/s5c_time.log 2>&1
timeout 120 python tools/one_run.py jacobi2d 64 1024 5 >> $o/s5c_time.log 2>&1
timeout 120 python tools/one_run.py jacobi2d 1024 2048 5 >> $o/s5c_time.log 2>&1
timeout 120 python tools/one_run.py heat2d_hold 256 2000 5 >> $o/s5c_time.log 2>&1
