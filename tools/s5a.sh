o=gpurun_out
timeout 600 python -m pytest tests/test_gpu_parity.py -m gpu -q -k gemm > $o/s5a_gemm.log 2>&1; echo rc $? >> $o/s5a_gemm.log
for v in 0 10 9; do PCOTGPU_DGEMM_VARIANT=$v timeout 120 python tools/kbench.py gemm --reps 7 >> $o/s5a_kb.log 2>&1; done
for n in 2048 8192; do for v in 0 9; do PCOTGPU_DGEMM_VARIANT=$v timeout 120 python tools/kbench.py gemm --n $n --reps 5 >> $o/s5a_kb.log 2>&1; done; done
timeout 2400 python -m pytest tests -m gpu -q > $o/s5a_pytest.log 2>&1; echo rc $? >> $o/s5a_pytest.log
timeout 900 python bench.py > $o/s5a_bench.log 2>&1; echo rc $? >> $o/s5a_bench.log
