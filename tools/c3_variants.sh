#!/bin/bash
# Config-3 (2048^3 u16) fused-pass variants on one B200: launch shapes of the
# default build, then a COLS=8 build, then one ncu --set full capture of the
# default kernel.  Output under gpurun_out/.
set -u
OUT=gpurun_out/c3var
mkdir -p $OUT
for v in 0 1 2 3 4; do
  CTP_PREVIEW_VARIANT=$v timeout 300 python tools/prof_preview.py --config c3 --schemes 1024,512,256,128 --time --reps 8 2>&1 | tail -1 | sed "s/^/cols4 /" >> $OUT/times.txt
done
if [ -n "${EXTRA:-}" ]; then
  for ex in $EXTRA; do
    CTP_NVCC_EXTRA="$ex" python - <<PY
from pathlib import Path
from paper_2311_15038_b200 import _build
_build.LIB = Path("/tmp/libvariant.so")
_build.build(verbose=False, force=True)
PY
    for v in 0 1 2 3 4; do
      CTP_PREVIEW_VARIANT=$v timeout 300 python tools/prof_preview.py --lib /tmp/libvariant.so --config c3 --schemes 1024,512,256,128 --time --reps 8 2>&1 | tail -1 | sed "s/^/$ex /" >> $OUT/times.txt
    done
  done
fi
if [ "${NCU:-1}" = 1 ]; then
  timeout 900 ncu --set full --clock-control none --import-source on -k regex:preview_kernel -c 1 -o $OUT/c3_default -f \
    python tools/prof_preview.py --config c3 --schemes 1024,512,256,128 --reps 1 > $OUT/ncu.log 2>&1
fi
cat $OUT/times.txt
