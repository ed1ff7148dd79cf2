"""Time config-4 rendering (36 azimuths, 1024^2, 0.5-voxel steps over 1024^3): MIP / alpha / additive.

usage: python tools/prof_render.py [--mode mip] [--views 36] [--dim 1024] [--n 1024] [--batches 1] [--fp64]
"""
import argparse
import math
import sys
import time
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
import torch  # noqa: E402

from paper_2311_15038_b200 import _lib, device as dev, synth  # noqa: E402
from paper_2311_15038_b200.types import ViewParams  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--mode", default="mip")
ap.add_argument("--views", type=int, default=36)
ap.add_argument("--dim", type=int, default=1024)
ap.add_argument("--n", type=int, default=1024)
ap.add_argument("--batches", type=int, default=1)
ap.add_argument("--fp64", action="store_true")
ap.add_argument("--lib", default=None, help="alternative build of the shared library (A/B timing)")
a = ap.parse_args()
if a.lib:
    _lib._lib = _lib.load(a.lib)
_lib.load()
spec = synth.config("c4")
if a.n != 1024:
    spec = synth.small((a.n, a.n, a.n), seed=0, n_shells=3, speckle_p=0.0)
vol = synth.generate(spec)
steps = math.ceil(4 * math.sqrt(3.0) / 2.0 * a.n)
views = [ViewParams(azimuth_deg=360.0 * k / a.views, image_dim=a.dim, steps=steps, mode=a.mode) for k in range(a.views)]
ch = 4 if a.mode in ("mip", "alpha") else 1
out = dev.render(vol, views, channels=ch, fp32=not a.fp64)
torch.cuda.synchronize()
w0 = time.perf_counter()
while time.perf_counter() - w0 < 1.0:  # clocks up from idle before timing
    dev.render(vol, views, channels=ch, fp32=not a.fp64, out=out)
    torch.cuda.synchronize()
e0 = torch.cuda.Event(enable_timing=True)
e1 = torch.cuda.Event(enable_timing=True)
e0.record()
for _ in range(a.batches):
    dev.render(vol, views, channels=ch, fp32=not a.fp64, out=out)
e1.record()
torch.cuda.synchronize()
ms = e0.elapsed_time(e1)
frames = a.views * a.batches
print(f"mode={a.mode} fp64={a.fp64} n={a.n} dim={a.dim} steps={steps} frames={frames} ms/frame={ms / frames:.3f} "
      f"fps={frames / ms * 1e3:.1f} Gsamples/s={frames * a.dim * a.dim * steps / ms / 1e6:.1f} "
      f"mean={out.float().mean().item():.3f}")
