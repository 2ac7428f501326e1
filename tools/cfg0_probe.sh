#!/bin/bash
# cfg0 probe: SM clock during back-to-back executor runs, and the per-launch
# kernel durations (ncu, serialised) to compare with the event-timed runs.
o=gpurun_out
nvidia-smi --query-gpu=clocks.sm,clocks_throttle_reasons.active --format=csv,noheader -lms 50 > $o/cfg0_clocks.csv &
SMI=$!
for v in 10 8; do
  PCOTGPU_S2D5_VARIANT=$v timeout 120 python tools/kbench.py jac --bts 4,6,8 --reps 300 > $o/cfg0_probe_v$v.log 2>&1
done
kill $SMI
PCOTGPU_S2D5_VARIANT=10 timeout 300 ncu --metrics gpu__time_duration.sum,smsp__cycles_elapsed.avg.per_second --clock-control none -k regex:s2d5 -c 200 --csv \
  --log-file $o/cfg0_ncu.csv python tools/kbench.py jac --bts 4,6 --reps 1 > $o/cfg0_ncu.log 2>&1
