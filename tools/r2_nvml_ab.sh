# does the in-process NVML clock sampler (1 kHz) perturb the timed c2 steps?  A/B in one call, alternating
for i in 1 2 3; do
  for nv in 0 1; do
    CTP_BENCH_NVML=$nv python bench.py --steps 20 --warmup 5 --no-mip --no-configs --no-cpu-baseline --no-e2e 2>/dev/null | python -c "
import json,sys
d=json.loads(sys.stdin.read().strip().splitlines()[-1]); print('nvml=$nv', 'step_ms', round(d['ms_per_step'],5), 'kernel_ms', round(d['roofline']['kernel_ms'],5), 'frac', round(d['roofline']['frac'],4), d['clocks'].get('samples'))"
  done
done
for nv in 0 1; do
  CTP_BENCH_NVML=$nv python bench.py --steps 2000 --warmup 20 --no-mip --no-configs --no-cpu-baseline --no-e2e 2>/dev/null | python -c "
import json,sys
d=json.loads(sys.stdin.read().strip().splitlines()[-1]); print('K=2000 nvml=$nv', 'step_ms', round(d['ms_per_step'],5), 'kernel_ms', round(d['roofline']['kernel_ms'],5), 'frac', round(d['roofline']['frac'],4), d['clocks'].get('samples'))"
done
