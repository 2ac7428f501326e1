#!/bin/bash
# One GPU session: parity suite, per-config numbers, 3-D depth sweep (PDL on/off),
# the bench line, then the bench launch list under ncu (after the plain run).
o=gpurun_out
python -m pytest tests -m gpu -x -q > $o/rc_pytest.log 2>&1; echo rc $? >> $o/rc_pytest.log
python tools/configs_bench.py --reps 5 > $o/rc_configs.json 2> $o/rc_configs.err
python tools/kbench.py s3d7 --bts 1,2,3 --reps 10 > $o/rc_s3d7_pdl.log 2>&1
: PCOTGPU_PDL=0 python tools/kbench.py s3d7 --bts 1,2,3 --reps 10 > $o/rc_s3d7_nopdl.log 2>&1
python bench.py > $o/rc_bench.log 2>&1; echo rc $? >> $o/rc_bench.log
ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file $o/rc_launches.csv \
  python bench.py --steps 2 --warmup 1 > $o/rc_ncu.log 2>&1
