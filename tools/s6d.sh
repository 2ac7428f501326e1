o=gpurun_out
rm -f $o/s6d_*.log
L=paper_1802_00166_b200/libpcotgpu.so
for v in A B A B; do
  cp _exp/lib_$v.so $L
  echo "lib $v" >> $o/s6d_ab.log
  timeout 200 python tools/kbench.py s3d7 --bts 2 --reps 150 2>&1 | grep GUpd >> $o/s6d_ab.log
done
for v in A B; do
  cp _exp/lib_$v.so $L
  echo "lib $v bt1 bt3" >> $o/s6d_ab.log
  timeout 200 python tools/kbench.py s3d7 --bts 1,3 --reps 60 2>&1 | grep GUpd >> $o/s6d_ab.log
done
cp _exp/lib_B.so $L
timeout 900 python -m pytest tests -m gpu -q -x -k "heat3d or s3d7 or 3d" > $o/s6d_t.log 2>&1; echo rc $? >> $o/s6d_t.log
