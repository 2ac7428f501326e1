cd $GRAFT_REPO_ROOT
timeout 900 python bench.py > gpurun_out/bench3.log 2>&1; echo "bench rc=$?" >> gpurun_out/bench3.log
timeout 600 python bench.py --steps 2 --warmup 1 > gpurun_out/bench_plain.log 2>&1 && \
timeout 1200 ncu --metrics gpu__time_duration.sum --clock-control none -c 700 --csv --log-file gpurun_out/launches_r01.csv python bench.py --steps 2 --warmup 1 > gpurun_out/ncu_launches.log 2>&1
echo "launches rc=$?"
timeout 600 python bench.py --steps 1 --warmup 1 --no-e2e --no-cpu-baseline > gpurun_out/bench_small.log 2>&1 && \
timeout 1200 ncu --set full --import-source on --clock-control none -k regex:s2d5 -s 90 -c 1 -o gpurun_out/prof_bench_s2d5 python bench.py --steps 1 --warmup 1 --no-e2e --no-cpu-baseline > gpurun_out/ncu_full.log 2>&1
echo "full rc=$?"
tail -2 gpurun_out/bench3.log
