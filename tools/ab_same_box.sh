#!/bin/bash
# same-box A/B of the cfg2 schemes: A = libkaczmarz_b200_ab.so (tools/build_ab.py), B = current build; interleaved
for sc in ${SCHEMES:-grk vr-ogrk ahk vr-oahk}; do
  for rep in 1 2; do
    echo "A $(KZ_LIB_VARIANT=ab python tools/prof_solve.py --scheme $sc --iters 200 --reps 3 | tail -1)"
    echo "B $(python tools/prof_solve.py --scheme $sc --iters 200 --reps 3 | tail -1)"
  done
done
