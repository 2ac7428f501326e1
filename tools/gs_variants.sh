#!/bin/bash
# Gauss-Seidel pipeline variants (NW warps, RS ring, S clocks/chunk; gs2d.cu kPipeVariants)
for v in ${GSV:-0 1 2 3 4}; do
  for T in 64 256; do
    echo "v$v $(PCOTGPU_GS_PIPE_V=$v timeout 120 python tools/gs_once.py $T 4096 10 2>&1 | tail -1)"
  done
done > gpurun_out/gs_variants.log
