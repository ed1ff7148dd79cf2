# general-ratio downscale (ctp_downscale_u8): the warp-per-row kernel vs round 1's (CTP_DOWNSCALE_OLD=1),
# clocks warmed up for 1 s before each timing, then the parity tests
set -u
for a in "--c5" "--target 512" "--target 768" "--target 300" "--target 1000"; do
  python tools/prof_downscale.py $a
  CTP_DOWNSCALE_OLD=1 python tools/prof_downscale.py $a | sed 's/^/old: /'
done
timeout 900 python -m pytest tests/test_gpu_parity.py -m gpu -x -q -k "downscale or c5 or interactive or bundles or anisotropic or data_preview or acceptance" -p no:warnings 2>&1 | tail -3
