# does the MIP leg of bench.py reproduce its slow mode (1.84 instead of 1.08 ms/frame)?  per-batch times + clocks
for k in 2000 20 2000 20; do
  python bench.py --steps $k --warmup 5 --no-configs 2>/dev/null | python -c "
import json,sys
d=json.loads(sys.stdin.read().strip().splitlines()[-1]); m=d['mip']
print('K=$k value', round(d['value'],1), 'frac', round(d['roofline']['frac'],4), d['clocks']['sm_mhz'], d['clocks']['reasons'], '| mip', round(m['value'],1), [round(x,1) for x in m['batch_ms']], m['clocks']['sm_mhz'], m['clocks']['reasons'], m['clocks']['samples'])"
done
