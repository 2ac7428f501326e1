o=gpurun_out
PCOTGPU_GS_PROF=2 timeout 120 python tools/gs_once.py 64 4096 1 > $o/s6h_b0.log 2>&1
PCOTGPU_GS_PROF=66 timeout 120 python tools/gs_once.py 64 4096 1 > $o/s6h_b64.log 2>&1
