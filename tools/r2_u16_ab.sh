set -u
for lib in default variants/libhot0.so variants/libhot384.so; do
  arg=""; [ "$lib" != default ] && arg="--lib $lib"
  for v in 0 1; do
    CTP_PREVIEW_VARIANT=$v timeout 300 python tools/prof_preview.py $arg --config c3 --schemes 1024,512,256,128 --time --reps 8 2>&1 | tail -1 | sed "s|^|$lib |"
  done
done
timeout 900 python -m pytest tests/test_gpu_parity.py -m gpu -x -q -k "u16 or sweep or c3_full or c5 or level0 or wide" -p no:warnings 2>&1 | tail -3
