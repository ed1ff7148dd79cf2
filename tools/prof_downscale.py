"""Time the general-ratio downscale (volume.py:277-309, ctp_downscale_u8) on
device-resident volumes: the config-2 volume to a cube target, or config 5's
level 1 (768^2 x 1024) to the 512 scheme (1.5:1 in x, y; 2:1 in z).

usage: python tools/prof_downscale.py [--target 768 | --c5] [--lib path] [--reps 5]
"""
import argparse
import sys
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
import torch  # noqa: E402

from paper_2311_15038_b200 import _lib, device as dev, synth  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--target", type=int, default=768)
ap.add_argument("--c5", action="store_true", help="config-5 level 1: (1024, 768, 768) -> 512^3")
ap.add_argument("--lib", default=None)
ap.add_argument("--reps", type=int, default=20)
a = ap.parse_args()
if a.lib:
    _lib._lib = _lib.load(a.lib)
_lib.load()
if a.c5:
    vol = synth.generate(synth.small((1024, 768, 768), seed=5, n_shells=6))
    t = (512, 512, 512)
else:
    vol = synth.generate(synth.config("c2"))
    t = (a.target,) * 3
out = dev.downscale(vol, t)
torch.cuda.synchronize()
import time  # noqa: E402
w0 = time.perf_counter()
while time.perf_counter() - w0 < 1.0:  # clocks up from idle before timing
    dev.downscale(vol, t)
    torch.cuda.synchronize()
e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
e0.record()
for _ in range(a.reps):
    dev.downscale(vol, t)
e1.record()
torch.cuda.synchronize()
ms = e0.elapsed_time(e1) / a.reps
print(f"downscale {tuple(vol.shape)} -> {t[::-1]}: {ms:.4f} ms, {(vol.numel() + out.numel()) / ms / 1e6:.1f} GB/s, "
      f"checksum={int(out.sum())}")
