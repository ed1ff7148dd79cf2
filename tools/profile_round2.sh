#!/bin/bash
# One B200 pass producing round 2's evidence under gpurun_out/prof2/ (summarised into
# profiles/ by tools/summarise_r02.py): the bench line (driver's K/W), the reference arm,
# the ncu launch list of the bench's c2 step, and ncu --set full captures of the c2 step
# kernel, the config-3 u16 fused pass and every other kernel (tools/prof_secondary.py).
set -u
OUT=gpurun_out/prof2
mkdir -p $OUT
python bench.py --steps 20 --warmup 5 > $OUT/bench.jsonl 2> $OUT/bench.err; echo "bench rc=$?"
python bench.py --impl reference --steps 20 --warmup 5 > $OUT/bench_reference.jsonl 2> $OUT/bench_reference.err; echo "reference rc=$?"
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file $OUT/launches.csv \
  python bench.py --steps 20 --warmup 3 --no-mip --no-cpu-baseline --no-configs --no-e2e --no-sustained > $OUT/launches.log 2>&1; echo "launch list rc=$?"
timeout 900 ncu --set full --clock-control none --import-source on -k regex:preview_kernel -s 5 -c 1 -o $OUT/fused_c2_step -f \
  python bench.py --steps 3 --warmup 3 --no-mip --no-e2e --no-cpu-baseline --no-configs --no-sustained > $OUT/ncu_c2.log 2>&1; echo "ncu c2 rc=$?"
timeout 900 ncu --set full --clock-control none --import-source on -k regex:preview_kernel -s 1 -c 1 -o $OUT/fused_c3_u16 -f \
  python tools/prof_preview.py --config c3 --schemes 1024,512,256,128 --reps 2 > $OUT/ncu_c3.log 2>&1; echo "ncu c3 rc=$?"
timeout 1500 ncu --set full --clock-control none --import-source on -k 'regex:^(?!synth)' -c 40 -o $OUT/secondary -f \
  python tools/prof_secondary.py > $OUT/ncu_secondary.log 2>&1; echo "ncu secondary rc=$?"
# summarise on the box (ncu is there) and keep the returned directory small
python tools/summarise_r02.py --tag r02 > $OUT/summary.log 2>&1; echo "summary rc=$?"
mkdir -p $OUT/profiles && cp profiles/r02_* profiles/traffic_fused_c2.json $OUT/profiles/ 2>/dev/null
du -sh $OUT/*.ncu-rep
rm -f $OUT/*.ncu-rep  # 35-80 MB each: over the 64 MiB return limit (the summaries carry the numbers)
