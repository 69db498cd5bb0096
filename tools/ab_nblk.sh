for nb in 2 8; do KZ_CLUSTER_NBLK=$nb python -m pytest tests/test_gpu_cluster.py -x -q 2>&1 | tail -1; done
for c in "cfg3 vr-oahk 256 50" "cfg5 ahk 256 50" "cfg5 vr-oahk 256 50" "cfg4 grk 64 0 1e-4" "cfg4 vr-oahk 128 0 1e-4"; do
  set -- $c
  for rep in 1 2; do for nb in 2 4 8; do
    echo "nblk=$nb $(KZ_CLUSTER_NBLK=$nb python tools/prof_solve.py --config $1 --scheme $2 --batch $3 --iters $4 --reps 5 ${5:+--residual $5} | tail -1) [$1]"
  done; done
done
