o=gpurun_out
timeout 1800 python -m pytest tests -m gpu -x -q > $o/r2b_pytest.log 2>&1; echo rc $? >> $o/r2b_pytest.log
timeout 900 python bench.py > $o/r2b_bench.log 2>&1; echo rc $? >> $o/r2b_bench.log
