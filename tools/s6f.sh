o=gpurun_out
rm -f $o/s6f_*.log
L=paper_1802_00166_b200/libpcotgpu.so
for v in F G F G; do
  cp _exp/lib_$v.so $L
  echo "lib $v" >> $o/s6f_ab.log
  timeout 300 python tools/kbench.py s2d5 --bts 6 --orders slt --reps 400 2>&1 | tail -1 >> $o/s6f_ab.log
done
cp _exp/lib_F.so $L
