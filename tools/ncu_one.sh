#!/bin/bash
# One `ncu --set full` capture of a kernel of a default-schedule executor run,
# summarised on the box (large reports do not travel):
#   bash tools/ncu_one.sh KERNEL T N KERNEL_REGEX OUT_TAG [SKIP]
o=gpurun_out
python tools/one_run.py $1 $2 $3 > $o/$5_plain.log 2>&1 || exit 1
timeout 900 ncu --set full --import-source on --clock-control none -k regex:$4 -s ${6:-4} -c 1 -f -o /tmp/$5 \
    python tools/one_run.py $1 $2 $3 > $o/$5_ncu.log 2>&1
python tools/ncu_summary.py /tmp/$5.ncu-rep $o/$5 >> $o/$5_ncu.log 2>&1
python tools/ncu_hot.py /tmp/$5.ncu-rep 25 > $o/$5_hot.txt 2>&1
