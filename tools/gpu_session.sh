cd $GRAFT_REPO_ROOT
PCOTGPU_S2D5_VARIANT=0 timeout 300 python tools/kbench.py s2d5 --rows 8192 --bts 7 --orders slt > gpurun_out/kb_plain.log 2>&1 && \
PCOTGPU_S2D5_VARIANT=0 timeout 900 ncu --set full --import-source on --clock-control none -k regex:s2d5 -s 1 -c 1 -o gpurun_out/prof_s2d5_v0_bt7 python tools/kbench.py s2d5 --rows 8192 --bts 7 --orders slt > gpurun_out/ncu_s2d5.log 2>&1
echo "ncu rc=$?"; cat gpurun_out/kb_plain.log
