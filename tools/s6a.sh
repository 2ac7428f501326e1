o=gpurun_out
timeout 300 python -m pytest tests/test_gpu_kernels.py -m gpu -q -x -k resident > $o/s6a_res.log 2>&1; echo rc $? >> $o/s6a_res.log
for v in 28 15 26 27; do for bt in 2 3; do
  echo "variant $v bt $bt" >> $o/s6a_s3d.log
  PCOTGPU_S3D7_VARIANT=$v timeout 200 python tools/kbench.py s3d7 --bts $bt --reps 80 >> $o/s6a_s3d.log 2>&1
done; done
