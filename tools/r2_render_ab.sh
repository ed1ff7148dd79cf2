for rep in 1 2; do
for lib in default variants/libprev.so; do
  arg=""; [ "$lib" != default ] && arg="--lib $lib"
  python tools/prof_render.py $arg --mode mip --batches 2 | sed "s|^|$lib |"
  python tools/prof_render.py $arg --mode alpha --batches 2 | sed "s|^|$lib |"
done
done
