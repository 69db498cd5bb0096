#!/bin/bash
for sc in grk vr-oahk ahk urk vr-ogrk; do
  KZ_LIB_VARIANT=timing python tools/phase_times.py --scheme $sc
  KZ_CHUNKED_C64=1 KZ_LIB_VARIANT=timing python tools/phase_times.py --scheme $sc | sed 's/^/[chunked] /'
done
