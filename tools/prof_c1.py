"""Config 1 (256^3 u8, one 16x16-grid 4096^2 atlas): the one-launch step replayed
from a CUDA graph (launch-bound size), for launch-shape variants
(CTP_PREVIEW_VARIANT).

usage: CTP_PREVIEW_VARIANT=2 python tools/prof_c1.py
"""
import os
import sys
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
import torch  # noqa: E402

from paper_2311_15038_b200 import _lib, synth  # noqa: E402
from paper_2311_15038_b200.device import AtlasSpec  # noqa: E402
from paper_2311_15038_b200.pipeline import plan_preview, run_preview  # noqa: E402

_lib.load()
spec = synth.config("c1")
vol = synth.generate(spec)
plan = plan_preview(spec.shape, {256: AtlasSpec(256, 4096, 16, 1)})
res = run_preview(vol, plan)
ref = res.atlases[256].clone()
side = torch.cuda.Stream()
side.wait_stream(torch.cuda.current_stream())
with torch.cuda.stream(side):
    for _ in range(3):
        run_preview(vol, plan, hist=res.hist)
torch.cuda.current_stream().wait_stream(side)
g = torch.cuda.CUDAGraph()
with torch.cuda.graph(g):
    r2 = run_preview(vol, plan, hist=res.hist)
for _ in range(20):
    g.replay()
e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
e0.record()
for _ in range(500):
    g.replay()
e1.record()
torch.cuda.synchronize()
us = e0.elapsed_time(e1) / 500 * 1e3
ok = torch.equal(r2.atlases[256], ref)
print(f"variant={os.environ.get('CTP_PREVIEW_VARIANT', 'default')} c1 {us:.2f} us/step "
      f"({2 * vol.numel() / us / 1e3:.0f} GB/s) equal={ok}")
