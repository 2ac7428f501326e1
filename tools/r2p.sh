o=gpurun_out
for w in 0 8 32 100 250 500; do for sp in 64 256 1000; do
  echo "wait=$w spin=$sp $(PCOTGPU_GS_WAIT=$w PCOTGPU_GS_SPIN=$sp timeout 60 python tools/gs_once.py 64 4096 5 | tail -1) | $(PCOTGPU_GS_WAIT=$w PCOTGPU_GS_SPIN=$sp timeout 60 python tools/gs_once.py 256 4096 3 | tail -1)"
done; done > $o/r2p_gs.log 2>&1
