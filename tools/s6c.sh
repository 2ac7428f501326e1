o=gpurun_out
python tools/one_run.py heat3d_b 100 384 > $o/s6c_plain.log 2>&1
timeout 600 ncu --set full --import-source on --clock-control none -k regex:s3d7 -s 4 -c 1 -f -o /tmp/ncu_cfg1_s3d7_x \
    python tools/one_run.py heat3d_b 100 384 > $o/s6c_ncu.log 2>&1
ls -la /tmp/ncu_cfg1_s3d7_x.ncu-rep >> $o/s6c_ncu.log
python tools/ncu_hot.py /tmp/ncu_cfg1_s3d7_x.ncu-rep 60 > $o/s6c_hot.txt 2>&1
python tools/ncu_summary.py /tmp/ncu_cfg1_s3d7_x.ncu-rep $o/ncu_cfg1_s3d7_x >> $o/s6c_ncu.log 2>&1
ncu -i /tmp/ncu_cfg1_s3d7_x.ncu-rep --page source --csv --print-source sass 2>/dev/null | cut -d, -f1-8 | gzip > $o/s6c_sass.csv.gz
