#!/bin/bash
# ncu --set full captures (one launch each) of the bench kernel (config 4, bt=6)
# and the small-grid kernel (config 0, bt=8), summarised into gpurun_out/.
o=gpurun_out
python bench.py --steps 1 --warmup 3 --no-e2e --no-cpu-baseline --no-depth-sweep > $o/nr_plain.log 2>&1 || exit 1
ncu --set full --import-source on --clock-control none -k regex:s2d5 -s 6 -c 1 -f -o /tmp/nr_bench \
  python bench.py --steps 1 --warmup 3 --no-e2e --no-cpu-baseline --no-depth-sweep > $o/nr_bench.log 2>&1
python tools/ncu_summary.py /tmp/nr_bench.ncu-rep $o/ncu_bench_s2d5_bt6_r01 --cells $((32768*32768)) --bt 6 >> $o/nr_bench.log 2>&1
ncu --set full --import-source on --clock-control none -k regex:s2d5 -s 20 -c 1 -f -o /tmp/nr_cfg0 \
  python tools/kbench.py jac --bts 8 --reps 3 > $o/nr_cfg0.log 2>&1
python tools/ncu_summary.py /tmp/nr_cfg0.ncu-rep $o/ncu_cfg0_s2d5_bt8_r01 --cells $((2048*2048)) --bt 8 >> $o/nr_cfg0.log 2>&1
ls -la /tmp/*.ncu-rep > $o/nr_sizes.txt
