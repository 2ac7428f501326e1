o=gpurun_out
timeout 1500 python -m pytest tests/test_ref_adapter.py -m gpu -q -k large --durations=10 > $o/r2d_pytest.log 2>&1; echo rc $? >> $o/r2d_pytest.log
