o=gpurun_out
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm,power.limit --format=csv > $o/r2a_smi.txt 2>&1
nproc >> $o/r2a_smi.txt; free -g >> $o/r2a_smi.txt; lscpu | head -20 >> $o/r2a_smi.txt
timeout 1500 python -m pytest tests -m gpu -x -q > $o/r2a_pytest.log 2>&1; echo rc $? >> $o/r2a_pytest.log
timeout 600 python tools/configs_bench.py --reps 5 > $o/r2a_configs.json 2> $o/r2a_configs.err
timeout 600 python bench.py > $o/r2a_bench.log 2>&1; echo rc $? >> $o/r2a_bench.log
