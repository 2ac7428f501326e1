o=gpurun_out
timeout 2400 python -m pytest tests -m gpu -q --durations=15 > $o/r2j_pytest.log 2>&1; echo rc $? >> $o/r2j_pytest.log
