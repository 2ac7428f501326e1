o=gpurun_out
export PCOT_KERNEL_PATH=kernels PCOTGPU_GENERIC_DEBUG=1
for spec in "lud N=40" "lud N=128" "heat1d-fig7 T=50,N=200" "triangle N=100" "osp N=30"; do
  set -- $spec
  echo "== $spec"; timeout 300 oracle/_ref/ref_adapter_demo kernels/$1.kernel $2 2>&1 | grep -v "^MAP"
  echo "== $spec single"; timeout 300 oracle/_ref/ref_adapter_demo kernels/$1.kernel $2 --single 2>&1 | grep -v "^MAP"
done > $o/r2f_generic.log 2>&1
bash tools/r2e.sh
