o=gpurun_out
rm -f $o/s6b_*.log
timeout 900 python -m pytest tests -m gpu -q -x -k "heat3d or s3d7 or 3d" > $o/s6b_t.log 2>&1; echo rc $? >> $o/s6b_t.log
for bt in 1 2 3; do timeout 200 python tools/kbench.py s3d7 --bts $bt --reps 80 >> $o/s6b_s3d.log 2>&1; done
