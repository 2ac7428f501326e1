#!/bin/bash
# Round-2 profiles: the bench launch list (gpu__time_duration per launch, the
# recipe's pass) and one `ncu --set full` capture per hot kernel, summarised
# into gpurun_out/ (copied to profiles/ by hand).  Each ncu run follows a plain
# run of the same command that exited 0.
o=gpurun_out
python bench.py --steps 2 --warmup 3 --no-e2e --no-cpu-baseline --no-depth-sweep --no-per-config > $o/n2_plain.log 2>&1 || exit 1
ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file $o/launches_r02.csv \
  python bench.py --steps 2 --warmup 3 --no-e2e --no-cpu-baseline --no-depth-sweep --no-per-config > $o/n2_launches.log 2>&1
ncu --set full --import-source on --clock-control none -k regex:s2d5 -s 6 -c 1 -f -o /tmp/n2_bench \
  python bench.py --steps 1 --warmup 3 --no-e2e --no-cpu-baseline --no-depth-sweep --no-per-config > $o/n2_bench.log 2>&1
python tools/ncu_summary.py /tmp/n2_bench.ncu-rep $o/ncu_bench_s2d5_bt6_r02 --cells $((32768*32768)) --bt 6 >> $o/n2_bench.log 2>&1
for spec in "jacobi2d 256 2048 s2d5 cfg0_s2d5_bt8" "heat3d_b 100 384 s3d7 cfg1_s3d7v2_bt2" "gs2d 64 4096 gs2d_pipe cfg2_gs2d_pipe" "gemm 0 4096 dgemm cfg3_dgemm"; do
  set -- $spec
  python tools/one_run.py $1 $2 $3 > $o/n2_$5_plain.log 2>&1 || continue
  ncu --set full --import-source on --clock-control none -k regex:$4 -s 2 -c 1 -f -o /tmp/n2_$5 \
    python tools/one_run.py $1 $2 $3 > $o/n2_$5.log 2>&1
  python tools/ncu_summary.py /tmp/n2_$5.ncu-rep $o/ncu_$5_r02 >> $o/n2_$5.log 2>&1
done
