o=gpurun_out
export PCOT_KERNEL_PATH=kernels
for spec in "heat1d-fig7 T=50,N=200" "lud N=512" "heat1d-fig7 T=2048,N=8192" "osp N=256" "triangle N=4096"; do
  set -- $spec
  s=$(date +%s.%N)
  echo "== $spec"; PCOTGPU_GENERIC_DEBUG=1 timeout 600 oracle/_ref/ref_adapter_demo kernels/$1.kernel $2 --gpu-only 2>&1 | grep -v "^MAP"
  e=$(date +%s.%N); python -c "print('wall %.1f s' % ($e - $s))"
done > $o/r2g_generic.log 2>&1
for v in 0 7; do
  PCOTGPU_GS_PIPE_V=$v timeout 120 python tools/gs_once.py 64 4096 3 >> $o/r2g_gs.log 2>&1
  PCOTGPU_GS_PIPE_V=$v timeout 300 ncu --set full --import-source on --clock-control none -k regex:gs2d_pipe -s 1 -c 1 -f -o /tmp/gs_v$v python tools/gs_once.py 64 4096 2 > $o/r2g_ncu_v$v.log 2>&1
  ncu -i /tmp/gs_v$v.ncu-rep --page raw --csv > $o/r2g_raw_v$v.csv 2>&1
  ncu -i /tmp/gs_v$v.ncu-rep --page source --csv > $o/r2g_src_v$v.csv 2>&1
  python tools/ncu_summary.py /tmp/gs_v$v.ncu-rep $o/ncu_gs_v$v >> $o/r2g_gs.log 2>&1
done
