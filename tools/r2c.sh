o=gpurun_out
timeout 1500 python -m pytest tests/test_ref_adapter.py tests/test_generic.py tests/test_sweep.py -m gpu -q > $o/r2c_pytest.log 2>&1; echo rc $? >> $o/r2c_pytest.log
timeout 600 python -m pytest tests/test_gpu_parity.py -m gpu -q -k "gs2d" > $o/r2c_gs.log 2>&1; echo rc $? >> $o/r2c_gs.log
