#!/bin/bash
# SLT vs COT (Morton CTA order) vs COT across time (cot-st: one launch per
# (depth block, row band), Morton order of the skewed box) on Jacobi-2D:
# device time (mean / CoV over samples, every sample checksum-verified) and,
# per cell, ncu DRAM bytes + L2 hit summed over all the cell's launches.
# Sized so cot-st cells stay below ~300 launches (ncu profiles every launch).
o=gpurun_out
run() {  # kernel params tiles schemes tag
  timeout 1200 python -m paper_1802_00166_b200.sweep $1 -p $2 --tiles $3 --schemes $4 --samples 5 --ncu \
      --csv $o/st_$5.csv > $o/st_$5.log 2>&1
}
run jacobi2d T=16,N=8192 1x1024x256,2x1024x256,4x1024x256 slt,cot,cot-st n8192
run jacobi2d T=32,N=4096 1x512x256,2x512x256,1x1024x256 slt,cot,cot-st n4096
