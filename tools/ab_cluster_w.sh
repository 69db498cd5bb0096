#!/bin/bash
# same-box A/B of the cluster kernel's CTA shape: default pick vs 128-antenna CTAs (W=4, two CTAs per SM)
run() { for w in 0 4; do echo "W=$w $(KZ_CLUSTER_W=$w KZ_VERBOSE=1 python tools/prof_solve.py "$@" --reps 2 2>&1 | grep -E 'picked|min' | tr '\n' ' ')"; done; }
run --config cfg3 --scheme vr-oahk --batch 512 --iters 50
run --config cfg5 --scheme ahk --batch 256 --iters 50
run --config cfg5 --scheme vr-oahk --batch 256 --iters 50
run --config cfg3 --scheme vr-oahk-g --groups 4 --cap 8 --batch 512 --iters 20
