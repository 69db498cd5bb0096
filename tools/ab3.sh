#!/bin/bash
# same-box A/B/C of cfg2 solve launches: arms = KZ_LIB_VARIANT values ("" = the current build), interleaved
ARMS=${ARMS:-"ab half cur"}
for sc in ${SCHEMES:-grk vr-ogrk ahk vr-oahk}; do
  for rep in 1 2; do
    for arm in $ARMS; do
      v=$arm; [ "$arm" = cur ] && v=""
      echo "$arm $(KZ_LIB_VARIANT=$v python tools/prof_solve.py --scheme $sc --iters 200 --reps 3 | tail -1)"
    done
  done
done
