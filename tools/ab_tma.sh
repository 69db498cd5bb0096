#!/bin/bash
# same-box A/B of the TMA staging: A = KZ_NO_TMA=1 (asynchronous-copy / load staging), B = TMA tensor copies
run() { python tools/prof_solve.py "$@" --reps 3 | tail -1; }
for args in "--scheme grk --iters 200" "--scheme vr-oahk --iters 200" "--config cfg3 --scheme vr-oahk --batch 512 --iters 50" \
            "--config cfg4 --scheme vr-oahk --batch 512 --residual 1e-4" "--config cfg4 --scheme grk --batch 256 --residual 1e-4"; do
  for rep in 1 2; do
    echo "A $(KZ_NO_TMA=1 run $args)"
    echo "B $(run $args)"
  done
done
