# A/B: u16 fused pass with table-relative offsets (default) vs absolute addresses (variants/libabs.so, -DCTP_U16_ABS_ADDR)
set -u
for rep in 1 2 3; do
for lib in default variants/libabs.so; do
  arg=""; [ "$lib" != default ] && arg="--lib $lib"
  timeout 300 python tools/prof_preview.py $arg --config c3 --schemes 1024,512,256,128 --time --reps 8 2>&1 | tail -1 | sed "s|^|$lib |"
done
done
timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_ingest.py -m gpu -x -q -k "u16 or sweep or c3_full or c5 or level0 or wide or artifact or session" -p no:warnings 2>&1 | tail -2
