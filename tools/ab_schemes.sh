#!/bin/bash
# kernel timings over the cfg2 schemes (run on the GPU box)
for sc in urk grk vr-ogrk ahk vr-oahk; do
  python tools/prof_solve.py --scheme $sc --iters 200 --reps 3 | tail -1
done
python tools/prof_solve.py --scheme grk --dtype c128 --iters 200 --reps 2 | tail -1
python tools/prof_solve.py --scheme vr-oahk --dtype c128 --iters 200 --reps 2 | tail -1
