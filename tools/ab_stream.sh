#!/bin/bash
# same-box A/B of the cluster kernel's streamed variant (KZ_CLUSTER_STREAM=1, default) against the staged one (=0)
run() { for st in 0 1; do echo "stream=$st $(KZ_CLUSTER_STREAM=$st python tools/prof_solve.py "$@" --reps 2 | tail -1)"; done; }
run --config cfg4 --scheme grk --batch 128 --residual 1e-4
run --config cfg4 --scheme vr-oahk --batch 256 --residual 1e-4
run --config cfg3 --scheme vr-oahk --batch 512 --iters 50
run --config cfg5 --scheme ahk --batch 256 --iters 20
run --config cfg5 --scheme vr-oahk --batch 256 --iters 20
