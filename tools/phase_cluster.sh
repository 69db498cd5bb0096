set -x
export KZ_LIB_VARIANT=timing KZ_VERBOSE=1
python tools/phase_times.py --config cfg4 --scheme vr-oahk --batch 28 --residual 1e-4 --cluster-w 8 --cluster-g 16 2>&1 | grep -v "^\[kz cluster\] scheme"
python tools/phase_times.py --config cfg4 --scheme grk --batch 28 --residual 1e-4 --cluster-w 8 --cluster-g 32 2>&1 | grep -v "^\[kz cluster\] scheme"
python tools/phase_times.py --config cfg3 --scheme vr-oahk --batch 296 --iters 50 --cluster-w 8 --cluster-g 16 2>&1 | grep -v "^\[kz cluster\] scheme"
python tools/phase_times.py --config cfg5 --scheme ahk --batch 148 --iters 50 --cluster-w 8 --cluster-g 32 2>&1 | grep -v "^\[kz cluster\] scheme"
