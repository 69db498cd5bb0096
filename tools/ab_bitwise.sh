#!/bin/bash
# bitwise A/B of two builds of the library on one box: V / iters / flops of a cfg2 solve per scheme
#   ARMS="ab cur" SCHEMES="ahk vr-oahk" bash tools/ab_bitwise.sh
ARMS=${ARMS:-"ab cur"}
set -- $ARMS
for sc in ${SCHEMES:-grk vr-ogrk ahk vr-oahk}; do
  for arm in $ARMS; do
    v=$arm; [ "$arm" = cur ] && v=""
    KZ_LIB_VARIANT=$v python tools/prof_solve.py --config ${CONFIG:-cfg2} --scheme $sc --batch ${BATCH:-64} --iters ${ITERS:-200} --reps 1 --dump /tmp/abv_$arm.npz > /dev/null
  done
  python - "$sc" /tmp/abv_$1.npz /tmp/abv_$2.npz <<'PY'
import sys, numpy as np
a, b = np.load(sys.argv[2]), np.load(sys.argv[3])
same = all(np.array_equal(a[k].view(np.uint8), b[k].view(np.uint8)) for k in ("v", "iters", "flops"))
rel = np.linalg.norm(a["v"] - b["v"]) / np.linalg.norm(a["v"])
print(f"{sys.argv[1]}: bitwise {'identical' if same else 'DIFFERENT'} (rel V diff {rel:.3e})")
PY
done
