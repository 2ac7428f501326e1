o=gpurun_out
timeout 1800 python -m pytest tests -m gpu -q > $o/r2o_pytest.log 2>&1; echo rc $? >> $o/r2o_pytest.log
timeout 900 python bench.py > $o/r2o_bench.log 2>&1; echo rc $? >> $o/r2o_bench.log
timeout 1500 bash tools/ncu_round2.sh
