o=gpurun_out
rm -f $o/s6d_*.log
L=paper_1802_00166_b200/libpcotgpu.so
for lib in B D; do
  cp _exp/lib_$lib.so $L
  for v in 28 26 15 24 27; do
    echo "lib $lib variant $v bt2" >> $o/s6d_ab.log
    PCOTGPU_S3D7_VARIANT=$v timeout 300 python tools/kbench.py s3d7 --bts 2 --reps 60 2>&1 | grep GUpd >> $o/s6d_ab.log
  done
done
cp _exp/lib_E.so $L
