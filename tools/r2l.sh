o=gpurun_out
timeout 900 python -m pytest tests/test_gpu_parity.py -m gpu -q -k "gs2d_pipeline" -x > $o/r2l_pytest.log 2>&1; echo rc $? >> $o/r2l_pytest.log
for v in 0 9 11; do echo "== v$v"; PCOTGPU_GS_PROF=1 PCOTGPU_GS_PIPE_V=$v timeout 120 python tools/gs_once.py 64 4096 1 2>&1 | grep -E "profile|timeline"; PCOTGPU_GS_PIPE_V=$v timeout 120 python tools/gs_once.py 64 4096 5; PCOTGPU_GS_PIPE_V=$v timeout 120 python tools/gs_once.py 256 4096 3; done > $o/r2l_gs.log 2>&1
