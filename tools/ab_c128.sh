#!/bin/bash
# c128 parity + same-box A/B (A = libkaczmarz_b200_ab.so from tools/build_ab.py, main = current build)
python -m pytest tests/test_gpu_parity.py -x -q 2>&1 | tail -1
for sc in ${SCHEMES:-grk vr-ogrk ahk vr-oahk urk}; do for v in ab main; do vv=$v; [ $v = main ] && vv=""
  echo "$v $(KZ_LIB_VARIANT=$vv python tools/prof_solve.py --scheme $sc --dtype c128 --iters 200 --reps 3 | tail -1)"
done; done
