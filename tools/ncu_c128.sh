#!/bin/bash
# full-set ncu capture (with source) of the complex128 lockstep kernel (cfg2 grk, T=50)
mkdir -p gpurun_out/ncu
cmd="python tools/prof_solve.py --scheme ${SCHEME:-grk} --dtype c128 --iters 50 --reps 1"
$cmd > gpurun_out/ncu/plain_c128.log 2>&1 && \
ncu --set full --clock-control none --import-source on -k regex:lockstep_kernel -c 1 -o gpurun_out/ncu/full_c128_${SCHEME:-grk} $cmd \
    > gpurun_out/ncu/full_c128.log 2>&1
ls -la gpurun_out/ncu | grep c128
