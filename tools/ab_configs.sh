#!/bin/bash
# same-box A/B on BASELINE configs: A = libkaczmarz_b200_ab.so (tools/build_ab.py), B = current build
# usage: CASES="cfg3:vr-oahk:256:50 cfg5:ahk:256:50" bash tools/ab_configs.sh
for c in ${CASES:-cfg3:vr-oahk:256:50 cfg4:grk:64:60 cfg5:ahk:256:50}; do
  IFS=: read cfg sc b t <<< "$c"
  for rep in 1 2; do
    echo "A $(KZ_LIB_VARIANT=ab python tools/prof_solve.py --config $cfg --scheme $sc --batch $b --iters $t --reps 2 | tail -1) [$cfg]"
    echo "B $(python tools/prof_solve.py --config $cfg --scheme $sc --batch $b --iters $t --reps 2 | tail -1) [$cfg]"
  done
done
