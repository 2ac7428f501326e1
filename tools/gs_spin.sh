for sp in 0 32 64 128 256 1024; do echo "spin $sp: $(PCOTGPU_GS_SPIN=$sp timeout 120 python tools/gs_once.py 64 4096 20 2>&1 | tail -1)"; done > gpurun_out/gs_spin.log
