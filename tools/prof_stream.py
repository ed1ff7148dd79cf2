"""Config 5 on one GPU: a stream of 1536^2 x 2048 12-bit u16 volumes (9 GiB each),
each reduced end to end (hist, filter o rescale, L1..L4 atlases, 36-view 512^2 MIP
strip).  Reports volumes/min and GVoxel/s with the volume resident in HBM (each
volume generated on the device before its timed pass) and, separately, the PCIe
H2D time of one volume from pinned host memory.

usage: python tools/prof_stream.py [--volumes 4]
"""
import argparse
import sys
import time
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
import torch  # noqa: E402

from paper_2311_15038_b200 import _lib, synth  # noqa: E402
from paper_2311_15038_b200.stream import PreviewStream  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--volumes", type=int, default=4)
a = ap.parse_args()
_lib.load()
spec0 = synth.config("c5", seed=0)
ps = PreviewStream(spec0.shape, torch.uint16, device="cuda")
vol = torch.empty(spec0.shape, dtype=torch.uint16, device="cuda")
synth.generate(spec0, out=vol)
ps.process(vol)  # warm-up
torch.cuda.synchronize()
times = []
for i in range(a.volumes):
    synth.generate(synth.config("c5", seed=i), out=vol)
    torch.cuda.synchronize()
    e0 = torch.cuda.Event(enable_timing=True)
    e1 = torch.cuda.Event(enable_timing=True)
    e0.record()
    ps.process(vol)
    e1.record()
    torch.cuda.synchronize()
    times.append(e0.elapsed_time(e1))
host = torch.empty(spec0.shape, dtype=torch.uint16, pin_memory=True)
host.copy_(vol)
torch.cuda.synchronize()
t = time.perf_counter()
vol.copy_(host, non_blocking=True)
torch.cuda.synchronize()
h2d = time.perf_counter() - t
n = vol.numel()
ms = sum(times) / len(times)
print(f"c5 volumes={a.volumes} ms_per_volume={ms:.3f} (min {min(times):.3f}) volumes_per_min={60000 / ms:.0f} "
      f"GVoxel/s={n / ms / 1e6:.1f} thumb_level={ps.thumb_level} thumb_shape={ps.thumb_shape} steps={ps.steps} "
      f"h2d_ms={h2d * 1e3:.1f} volumes_per_min_with_h2d={60 / (h2d + ms / 1e3):.0f}")
