#!/bin/bash
# A/B timing of the lockstep kernels over the cfg2 schemes (run on the GPU box)
for sc in urk grk vr-ogrk ahk vr-oahk; do
  python tools/prof_solve.py --scheme $sc --iters 200 --reps 2 | tail -1
  KZ_CHUNKED_C64=1 python tools/prof_solve.py --scheme $sc --iters 200 --reps 2 | tail -1 | sed 's/^/chunked /'
done
python tools/prof_solve.py --scheme grk --dtype c128 --iters 200 --reps 2 | tail -1
python tools/prof_solve.py --scheme vr-oahk --dtype c128 --iters 200 --reps 2 | tail -1
