"""Time the c2 step (ONE cooperative launch: artifact LUT + fused pass), as bench.py's
headline, for A/B builds of the library.

usage: python tools/prof_step.py [--lib PATH] [--steps 500]
"""
import argparse
import sys
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
import torch  # noqa: E402

from paper_2311_15038_b200 import _lib, device as dev, synth  # noqa: E402
from paper_2311_15038_b200.device import AtlasSpec  # noqa: E402
from paper_2311_15038_b200.pipeline import plan_preview  # noqa: E402
from paper_2311_15038_b200.types import plan_scheme  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--lib", default=None)
ap.add_argument("--steps", type=int, default=500)
a = ap.parse_args()
if a.lib:
    _lib._lib = _lib.load(a.lib)
_lib.load()
spec = synth.config("c2")
vol = synth.generate(spec)
plan = plan_preview(spec.shape, {s: AtlasSpec.of(plan_scheme(s)) for s in (512, 256, 128)})
outs, hist, lut, flags = dev.preview_step(vol, plan.fused)
for _ in range(20):
    dev.preview_step(vol, plan.fused, hist=hist, out_tensors=outs)
torch.cuda.synchronize()
e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
e0.record()
for _ in range(a.steps):
    dev.preview_step(vol, plan.fused, hist=hist, out_tensors=outs)
e1.record()
torch.cuda.synchronize()
ms = e0.elapsed_time(e1) / a.steps
print(f"lib={a.lib or 'default'} c2 step {ms * 1e3:.1f} us  {1.2268e9 / ms / 1e6:.0f} GB/s  hist_ok={int(hist.sum()) == vol.numel()}")
