#!/bin/bash
# ncu --set full captures of this round's dominant kernels (one tool per gpurun call): the wide kernel (cfg2 vr-oahk,
# grk) and the cluster kernel (cfg4 grk residual, cfg3 vr-oahk)
mkdir -p gpurun_out/ncu
for c in "cfg2 vr-oahk 148 --iters 50 wide" "cfg2 grk 148 --iters 50 wide" "cfg4 grk 14 --residual 1e-4 cluster" "cfg3 vr-oahk 64 --iters 20 cluster"; do
  set -- $c
  cmd="python tools/prof_solve.py --config $1 --scheme $2 --batch $3 $4 $5 --reps 1"
  tag=$1_$2
  $cmd > gpurun_out/ncu/plain_$tag.log 2>&1 && \
  ncu --set full --clock-control none --import-source on -k regex:$6_kernel -c 1 -o gpurun_out/ncu/r02_full_$tag $cmd \
      > gpurun_out/ncu/r02_full_$tag.log 2>&1
done
ls -la gpurun_out/ncu
# the reports are large: keep the text exports only (details page, raw metrics, per-line source counters)
for r in gpurun_out/ncu/r02_full_*.ncu-rep; do
  b=${r%.ncu-rep}
  ncu -i $r --page details --csv > $b.details.csv 2>/dev/null
  ncu -i $r --page raw --csv > $b.raw.csv 2>/dev/null
  ncu -i $r --page source --csv --print-source sass > $b.source.csv 2>/dev/null
  gzip -f $b.source.csv $b.raw.csv
  rm -f $r
done
du -sh gpurun_out/ncu
