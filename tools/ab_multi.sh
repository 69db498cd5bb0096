#!/bin/bash
# interleaved same-box timing of several library variants (tools/build_ab.py --name=X; "" = current build)
# usage: VARIANTS="ab c1 c2 main" CASES="cfg3:vr-oahk:256:50 cfg4:grk:64:0:1e-4 ..." bash tools/ab_multi.sh
# (case = config:scheme:batch:T[:residual tolerance])
for c in ${CASES:-cfg3:vr-oahk:256:50 cfg5:ahk:256:50}; do
  IFS=: read cfg sc b t tol <<< "$c"
  for rep in 1 2; do
    for v in ${VARIANTS:-ab main}; do
      vv=$v; [ "$v" = main ] && vv=""
      echo "$v $(KZ_LIB_VARIANT=$vv python tools/prof_solve.py --config $cfg --scheme $sc --batch $b --iters $t --reps ${REPS:-5} ${tol:+--residual $tol} | tail -1) [$cfg]"
    done
  done
done
