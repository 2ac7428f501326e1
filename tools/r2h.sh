o=gpurun_out
export PCOT_KERNEL_PATH=kernels
for v in 0 7 5; do echo "== v$v"; PCOTGPU_GS_PROF=1 PCOTGPU_GS_PIPE_V=$v timeout 120 python tools/gs_once.py 64 4096 1; done > $o/r2h_prof.log 2>&1
for spec in "heat1d-fig7 T=50,N=200" "heat1d-fig7 T=512,N=4096"; do
  set -- $spec
  s=$(date +%s.%N)
  echo "== $spec"; PCOTGPU_GENERIC_DEBUG=1 timeout 600 oracle/_ref/ref_adapter_demo kernels/$1.kernel $2 2>&1 | grep -v "^MAP"
  e=$(date +%s.%N); python -c "print('wall %.1f s' % ($e - $s))"
done > $o/r2h_generic.log 2>&1
timeout 900 python -m pytest tests/test_cli.py -m gpu -q > $o/r2h_cli.log 2>&1; echo rc $? >> $o/r2h_cli.log
