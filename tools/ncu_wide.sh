#!/bin/bash
# full-set ncu capture (with source) of the wide kernel for the given cfg2 schemes (default grk ahk)
mkdir -p gpurun_out/ncu
for sc in ${SCHEMES:-grk ahk}; do
  cmd="python tools/prof_solve.py --scheme $sc --iters 50 --reps 1"
  $cmd > gpurun_out/ncu/plain_wide_$sc.log 2>&1 && \
  ncu --set full --clock-control none --import-source on -k regex:wide_kernel -c 1 -o gpurun_out/ncu/full_wide_$sc $cmd \
      > gpurun_out/ncu/full_wide_$sc.log 2>&1
done
ls -la gpurun_out/ncu
