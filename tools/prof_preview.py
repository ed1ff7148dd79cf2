"""Run the c2 fused preview pass a few times (for ncu / variant timing).

usage: python tools/prof_preview.py [--reps N] [--config c2] [--time]
"""
import argparse
import os
import sys
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))

import torch  # noqa: E402

from paper_2311_15038_b200 import _lib, device as dev, synth  # noqa: E402
from paper_2311_15038_b200.device import AtlasSpec  # noqa: E402
from paper_2311_15038_b200.pipeline import plan_preview  # noqa: E402
from paper_2311_15038_b200.types import plan_scheme  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--reps", type=int, default=3)
ap.add_argument("--config", default="c2")
ap.add_argument("--time", action="store_true")
ap.add_argument("--schemes", default="512,256,128")
ap.add_argument("--lib", default=None, help="alternative build of the shared library (A/B timing)")
a = ap.parse_args()
if a.lib:
    _lib._lib = _lib.load(a.lib)
_lib.load()
spec = synth.config(a.config)
vol = synth.generate(spec)
schemes = {}
for s in a.schemes.split(","):
    s = int(s)
    if s in (128, 256, 512):
        schemes[s] = AtlasSpec.of(plan_scheme(s))
    elif s == 1024:  # config 3 level 1: 64 maps of 4x4 slices, capped at 4096^2
        schemes[s] = AtlasSpec(1024, 4096, 4, 64)
    else:
        schemes[s] = AtlasSpec(s, 8 * s, 8, -(-s // 64))
plan = plan_preview(spec.shape, schemes)
lut, _ = dev.artifact_lut(vol)
hist = torch.zeros(256 if spec.dtype == "u8" else 4096, dtype=torch.int64, device="cuda")
outs = dev.preview(vol, lut, plan.fused, hist=hist)
torch.cuda.synchronize()
ts = []
for _ in range(a.reps):
    e0 = torch.cuda.Event(enable_timing=True)
    e1 = torch.cuda.Event(enable_timing=True)
    e0.record()
    dev.preview(vol, lut, plan.fused, hist=hist, out_tensors=outs)
    e1.record()
    torch.cuda.synchronize()
    ts.append(e0.elapsed_time(e1))
if a.time:
    alg = vol.numel() * vol.element_size() + sum(t.numel() for t in outs.values())
    print(f"voxels={vol.numel()} alg_bytes={alg} GVoxel/s={vol.numel() / min(ts) / 1e6:.1f}")
    best = min(ts)
    print(f"variant={os.environ.get('CTP_PREVIEW_VARIANT', 'default')} config={a.config} best_ms={best:.4f} "
          f"median_ms={sorted(ts)[len(ts) // 2]:.4f} GB/s={alg / best / 1e6:.1f}")
