cd $GRAFT_REPO_ROOT
timeout 300 python tools/kbench.py gs --tiles 4x32x64 --reps 1 > /dev/null 2>&1 && timeout 900 ncu --set full --import-source on --clock-control none -k regex:lines -s 1 -c 1 -o gpurun_out/prof_gslines python tools/kbench.py gs --tiles 4x32x64 --reps 1 > gpurun_out/ncu_gsl.log 2>&1; echo "ncu rc=$?"
