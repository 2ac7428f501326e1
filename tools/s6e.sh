o=gpurun_out
timeout 900 python -m pytest tests -m gpu -q -x -k "heat3d or s3d7 or 3d" > $o/s6e_t.log 2>&1; echo rc $? >> $o/s6e_t.log
timeout 900 python bench.py --steps 2 --no-e2e --no-depth-sweep --no-cpu-baseline > $o/s6e_bench.log 2>&1; echo rc $? >> $o/s6e_bench.log
