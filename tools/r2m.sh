o=gpurun_out
timeout 1200 python -m pytest tests/test_gpu_parity.py -m gpu -q -x -k "gs2d or space_time" > $o/r2m_pytest.log 2>&1; echo rc $? >> $o/r2m_pytest.log
bash tools/r2l.sh
