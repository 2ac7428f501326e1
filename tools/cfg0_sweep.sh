#!/bin/bash
# cfg0 (jacobi2d 2048^2 T=256) variant x row-chunk sweep through the executor
# (chunks 0 = automatic sizing).  Output: gpurun_out/cfg0_sweep${TAG}.log
out=gpurun_out/cfg0_sweep${TAG}.log; : > $out
for v in ${VARIANTS:-9 8 10 6}; do
  for ch in ${CHUNKS:-0}; do
    echo "== variant $v chunks $ch" >> $out
    PCOTGPU_S2D5_VARIANT=$v PCOTGPU_S2D5_CHUNKS=$ch timeout 120 python tools/kbench.py jac --n ${N:-2048} --T ${T:-256} --bts ${BTS:-2,3,4,5,6,8} --reps ${REPS:-5} 2>&1 | grep GUpd >> $out
  done
done
