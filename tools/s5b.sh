o=gpurun_out
timeout 300 python -m pytest tests/test_gpu_kernels.py -m gpu -q -x -k resident > $o/s5b_res.log 2>&1; echo rc $? >> $o/s5b_res.log
for w in -1 0 4 8 10 11; do
  if [ $w -ge 0 ]; then export PCOTGPU_RES_WAIT=$w; fi
  echo "wait $w" >> $o/s5b_time.log
  timeout 120 python tools/one_run.py jacobi2d 256 2048 >> $o/s5b_time.log 2>&1
done
unset PCOTGPU_RES_WAIT
PCOTGPU_RESIDENT=0 timeout 120 python tools/one_run.py jacobi2d 256 2048 >> $o/s5b_time.log 2>&1
timeout 120 python tools/one_run.py jacobi2d 64 1024 >> $o/s5b_time.log 2>&1
PCOTGPU_RESIDENT=0 timeout 120 python tools/one_run.py jacobi2d 64 1024 >> $o/s5b_time.log 2>&1
# DGEMM ncu
python tools/one_run.py gemm 0 4096 > $o/s5b_gemm_plain.log 2>&1
timeout 600 ncu --set full --import-source on --clock-control none -k regex:dgemm_tma -s 2 -c 1 -f -o $o/ncu_cfg3_dgemm_tma_r02 \
    python tools/one_run.py gemm 0 4096 > $o/s5b_gemm_ncu.log 2>&1
python tools/ncu_summary.py $o/ncu_cfg3_dgemm_tma_r02.ncu-rep $o/ncu_cfg3_dgemm_tma_r02 >> $o/s5b_gemm_ncu.log 2>&1
