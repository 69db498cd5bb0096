#!/bin/bash
# same-box A/B of the per-config timings: A = libkaczmarz_b200_ab.so (tools/build_ab.py), B = current build
CFGS=${CFGS:-cfg3,cfg4,cfg5}
for rep in 1 2; do
  echo "== A rep $rep"; KZ_LIB_VARIANT=ab python tools/bench_configs.py --configs $CFGS ${BATCH:+--batch $BATCH} 2>&1 | grep -v "^\[kz"
  echo "== B rep $rep"; python tools/bench_configs.py --configs $CFGS ${BATCH:+--batch $BATCH} 2>&1 | grep -v "^\[kz"
done
