o=gpurun_out
for v in 5 6 7 8; do PCOTGPU_GS_PIPE_V=$v timeout 120 python tools/gs_once.py 16 1024 1; done > $o/r2e_quick.log 2>&1
timeout 900 python -m pytest tests/test_gpu_parity.py -m gpu -q -k "gs2d_pipeline" > $o/r2e_pytest.log 2>&1; echo rc $? >> $o/r2e_pytest.log
GSV="0 5 6 7 8" bash tools/gs_variants.sh; cp $o/gs_variants.log $o/r2e_variants.log
