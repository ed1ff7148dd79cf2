# MIP inside the full bench.py (e2e + CPU baseline in a CUDA-free subprocess) vs tools/prof_render.py
python bench.py --steps 20 --warmup 5 --no-configs | python -c "import json,sys; d=json.loads(sys.stdin.read().strip().splitlines()[-1]); print('e2e+cpu:', d['mip']['value'], json.dumps(d['cpu_baseline'])[:300])"
python tools/prof_render.py --mode mip --batches 4
