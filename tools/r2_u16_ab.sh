# A/B of u16 fused-pass builds on config 3 (prof_preview: the fused pass alone, 8 reps), interleaved
set -u
for rep in 1 2; do
for lib in default variants/libhot_prev.so; do
  arg=""; [ "$lib" != default ] && arg="--lib $lib"
  timeout 300 python tools/prof_preview.py $arg --config c3 --schemes 1024,512,256,128 --time --reps 8 2>&1 | tail -1 | sed "s|^|$lib |"
done
done
