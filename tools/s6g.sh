o=gpurun_out
python tools/one_run.py gs2d 64 4096 > $o/s6g_plain.log 2>&1
timeout 900 ncu --set full --import-source on --clock-control none -k regex:gs2d_pipe -s 1 -c 1 -f -o /tmp/ncu_gs_x \
    python tools/one_run.py gs2d 64 4096 > $o/s6g_ncu.log 2>&1
ls -la /tmp/ncu_gs_x.ncu-rep >> $o/s6g_ncu.log
ncu -i /tmp/ncu_gs_x.ncu-rep --page source --csv --print-source sass 2>/dev/null | cut -d, -f1-8 | gzip > $o/s6g_sass.csv.gz
ncu -i /tmp/ncu_gs_x.ncu-rep --page source --csv --print-source cuda 2>/dev/null | gzip > $o/s6g_cuda.csv.gz
