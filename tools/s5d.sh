o=gpurun_out
timeout 600 ncu --set full --import-source on --clock-control none -k regex:s2d5_res -s 1 -c 1 -f -o $o/ncu_cfg0_res_b \
    python tools/one_run.py jacobi2d 256 2048 3 > $o/s5d_ncu.log 2>&1
python tools/ncu_summary.py $o/ncu_cfg0_res_b.ncu-rep $o/ncu_cfg0_res_b >> $o/s5d_ncu.log 2>&1
