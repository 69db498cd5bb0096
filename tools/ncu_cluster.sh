mkdir -p gpurun_out/ncu
for c in "cfg5 ahk 64 20" "cfg3 vr-oahk 128 20"; do
  set -- $c
  cmd="python tools/prof_solve.py --config $1 --scheme $2 --batch $3 --iters $4 --reps 1"
  $cmd > gpurun_out/ncu/plain_$1_$2.log 2>&1 && \
  ncu --set full --clock-control none --import-source on -k regex:cluster_kernel -c 1 -o gpurun_out/ncu/full_$1_$2 $cmd \
      > gpurun_out/ncu/full_$1_$2.log 2>&1
done
ls -la gpurun_out/ncu
