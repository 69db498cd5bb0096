#!/bin/bash
# same-box A/B of the complex128 (oracle-mode) lockstep kernel: A = libkaczmarz_b200_ab.so, B = current build
for sc in ${SCHEMES:-grk vr-ogrk ahk vr-oahk}; do
  for rep in 1 2; do
    echo "A $(KZ_LIB_VARIANT=ab python tools/prof_solve.py --scheme $sc --dtype c128 --iters 200 --reps 2 | tail -1)"
    echo "B $(python tools/prof_solve.py --scheme $sc --dtype c128 --iters 200 --reps 2 | tail -1)"
  done
done
