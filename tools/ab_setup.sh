python -m pytest tests/test_gpu_parity.py tests/test_gpu_primitives.py -x -q 2>&1 | tail -1
SCHEMES="grk ahk vr-oahk" bash tools/ab_c128.sh 2>&1 | tail -6
for v in ab main; do vv=$v; [ $v = main ] && vv=""; echo "$v $(KZ_LIB_VARIANT=$vv python tools/prof_solve.py --config cfg1 --scheme grk --iters 50 --reps 5 | tail -1) [cfg1 c64]"; echo "$v $(KZ_LIB_VARIANT=$vv python tools/prof_solve.py --config cfg1 --scheme grk --dtype c128 --iters 50 --reps 5 | tail -1) [cfg1 c128]"; done
