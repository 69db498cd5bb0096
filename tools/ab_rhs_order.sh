#!/bin/bash
# same-box A/B of the residual-mode rhs grouping (KZ_CLUSTER_RHS_ORDER=1 default) against the index order (=0)
for rep in 1 2; do
  for o in 0 1; do
    echo "order=$o $(KZ_CLUSTER_RHS_ORDER=$o python tools/prof_solve.py --config cfg4 --scheme grk --batch 256 --residual 1e-4 --reps 2 | tail -1)"
  done
done
