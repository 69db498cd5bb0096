#!/bin/bash
# ncu evidence for profiles/ (run on the GPU box; each ncu run only after the same command exited 0 plainly).
set -u
mkdir -p gpurun_out/ncu
for sc in urk grk vr-ogrk ahk vr-oahk; do
  cmd="python tools/prof_solve.py --scheme $sc --iters 200 --reps 1"
  $cmd > gpurun_out/ncu/plain_$sc.log 2>&1 && \
  ncu --metrics dram__bytes_read.sum,dram__bytes_write.sum,gpu__time_duration.sum,lts__t_bytes.sum \
      --clock-control none -k regex:"wide_kernel|rkwarp" -c 1 --csv $cmd > gpurun_out/ncu/traffic_$sc.csv 2> gpurun_out/ncu/traffic_$sc.err
done
# full section set of the dominant kernel (vr-oahk), smaller T to bound replay time
cmd="python tools/prof_solve.py --scheme vr-oahk --iters 50 --reps 1"
$cmd > gpurun_out/ncu/plain_full.log 2>&1 && \
ncu --set full --clock-control none --import-source on -k regex:wide_kernel -c 1 -o gpurun_out/ncu/full_vroahk $cmd \
    > gpurun_out/ncu/full.log 2>&1
# launch list of the benchmark step
bcmd="python bench.py --steps 2 --warmup 1 --no-cpu-baseline --no-e2e --no-c128 --no-configs"
$bcmd > gpurun_out/ncu/bench_plain.log 2>&1 && \
ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/ncu/launches.csv $bcmd \
    > gpurun_out/ncu/launch_run.log 2>&1
echo done
