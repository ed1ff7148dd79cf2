"""Time the general-ratio downscale (volume.py:277-309) on the config-2 volume.

usage: python tools/prof_downscale.py [--target 768] [--lib path]
"""
import argparse
import sys
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
import torch  # noqa: E402

from paper_2311_15038_b200 import _lib, device as dev, synth  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--target", type=int, default=768)
ap.add_argument("--lib", default=None)
a = ap.parse_args()
if a.lib:
    _lib._lib = _lib.load(a.lib)
_lib.load()
vol = synth.generate(synth.config("c2"))
t = (a.target,) * 3
out = dev.downscale(vol, t)
torch.cuda.synchronize()
e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
e0.record()
for _ in range(5):
    dev.downscale(vol, t)
e1.record()
torch.cuda.synchronize()
ms = e0.elapsed_time(e1) / 5
print(f"downscale 1024^3 -> {a.target}^3: {ms:.3f} ms, {(vol.numel() + out.numel()) / ms / 1e6:.1f} GB/s, "
      f"checksum={int(out.sum())}")
