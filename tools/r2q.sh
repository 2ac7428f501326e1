o=gpurun_out
export PCOT_KERNEL_PATH=kernels
timeout 1500 python -m pytest tests/test_emitter.py tests/test_generic.py tests/test_ref_adapter.py tests/test_cli.py -m gpu -q --durations=8 > $o/r2q_pytest.log 2>&1; echo rc $? >> $o/r2q_pytest.log
for jit in 1 0; do for spec in "lud N=512" "osp N=256" "triangle N=4096" "heat1d-fig7 T=256,N=2048"; do
  set -- $spec
  s=$(date +%s.%N)
  r=$(PCOTGPU_GENERIC_JIT=$jit timeout 600 oracle/_ref/pcot_run kernels/$1.kernel -p $2 --alloc --executor gpu 2>&1 | grep -E "CHECKSUM|wall_ms")
  e=$(date +%s.%N)
  echo "jit=$jit $spec $(echo $r | tr '\n' ' ') total $(python -c "print('%.2f s' % ($e - $s))")"
done; done > $o/r2q_time.log 2>&1
