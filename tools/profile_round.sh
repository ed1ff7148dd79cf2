#!/bin/bash
# One B200 pass producing the evidence under profiles/: the full bench line, the
# reference arm, the ncu launch list of the bench's c2 step and one ncu --set full
# capture of the step kernel.  Outputs under gpurun_out/prof/ (summarised into
# profiles/ by tools/summarise_profiles.py).
set -u
OUT=gpurun_out/prof
mkdir -p $OUT
python bench.py > $OUT/bench.jsonl 2> $OUT/bench.err; echo "bench rc=$?"
python bench.py --impl reference --steps 3 --warmup 1 > $OUT/bench_reference.jsonl 2> $OUT/bench_reference.err; echo "reference rc=$?"
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file $OUT/launches.csv \
  python bench.py --steps 20 --warmup 3 --no-mip --no-cpu-baseline --no-configs > $OUT/launches.log 2>&1; echo "launch list rc=$?"
timeout 900 ncu --set full --clock-control none --import-source on -k regex:preview_kernel -s 5 -c 1 -o $OUT/fused_c2_step -f \
  python bench.py --steps 3 --warmup 3 --no-mip --no-e2e --no-cpu-baseline --no-configs > $OUT/ncu_full.log 2>&1; echo "ncu full rc=$?"
