# config-3 fused pass by level count (tile geometry: L=4 tiles are 128 voxels wide, L=3 512)
set -u
for sch in 1024 1024,512 1024,512,256 1024,512,256,128; do
  timeout 300 python tools/prof_preview.py --config c3 --schemes $sch --time --reps 6 2>&1 | tail -1 | sed "s|^|schemes=$sch |"
done
