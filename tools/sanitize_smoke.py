"""Small calls of every kernel, for compute-sanitizer (memcheck / racecheck / synccheck).

usage: compute-sanitizer --tool memcheck python tools/sanitize_smoke.py
"""
import sys
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
import numpy as np  # noqa: E402
import torch  # noqa: E402

import paper_2311_15038_b200 as P  # noqa: E402
from paper_2311_15038_b200 import device as dev, synth  # noqa: E402
from paper_2311_15038_b200.device import AtlasSpec  # noqa: E402
from paper_2311_15038_b200.stream import PreviewStream  # noqa: E402

torch.cuda.set_device(0)
# fused pass, u8, levels 0..3 (atlases + dense), partial tiles (ny not a multiple of the tile height)
v8 = synth.generate(synth.small((64, 72, 96), seed=1))
lut, flags = dev.artifact_lut_fused(v8)
hist = torch.zeros(256, dtype=torch.int64, device="cuda")
dev.preview(v8, lut, {0: "xyz", 1: AtlasSpec(64, 512, 8, 1), 2: "xyz", 3: AtlasSpec(16, 64, 4, 1)}, hist=hist)
# u16, level 4
v16 = synth.generate(synth.small((64, 64, 128), dtype="u16", seed=2))
lut16, _ = dev.artifact_lut_fused(v16)
h16 = torch.zeros(4096, dtype=torch.int64, device="cuda")
dev.preview(v16, lut16, {1: "xyz", 4: AtlasSpec(8, 32, 4, 1)}, hist=h16)
# the whole step in one cooperative launch (in-kernel artifact LUT + grid barrier), u8 and u16
# (the u16 hot window chosen from each CTA's first tile; its LUT staged in the level-1 sum buffers)
dev.preview_step(v8, {1: AtlasSpec(64, 512, 8, 1), 2: "xyz", 3: AtlasSpec(16, 64, 4, 1)})
dev.preview_step(v16, {1: "xyz", 2: AtlasSpec(32, 256, 8, 1), 4: AtlasSpec(8, 32, 4, 1)})
# stand-alone kernels
dev.hist_u8(v8, (3, 40))
dev.lut_apply_u8(v8[:, :, :37].contiguous(), lut, hist=hist)
dev.lut_apply_u16(v16[:, :, :37].contiguous(), lut16, hist=h16)      # any-length u16 filter o rescale
dev.downscale(v8, (37, 29, 23))               # warp-per-row kernel, x cells <= 4
dev.downscale(v8, (64, 48, 32))                # x cells <= 2 (1.5:1, config 5's level-1 ratio), 4-output stores
dev.downscale(v8, (5, 7, 3))                   # wide cells: the float rounding path
dev.circle_mask(v8, 40.5, 30.25, 25.0 ** 2)
f = dev.png_filter(dev.encode_atlas(v8[:64, :64, :64].contiguous(), AtlasSpec(64, 512, 8, 1)))
from paper_2311_15038_b200.png import deflate_device  # noqa: E402
deflate_device(f)
dev.encode_atlas(v8[:48, :48, :48].contiguous(), AtlasSpec(64, 512, 8, 1))
dev.decode_atlas(dev.encode_atlas(v8[:64, :64, :64].contiguous(), AtlasSpec(64, 512, 8, 1)), AtlasSpec(64, 512, 8, 1))
# renders: exact fp64 modes, fp32 MIP (row planes) and alpha (texture)
for m in ("surface", "additive"):
    dev.render(v8, [P.ViewParams(azimuth_deg=a, image_dim=32, steps=48, mode=m, threshold=60) for a in (0.0, 37.0)])
import os  # noqa: E402
os.environ["CTP_RENDER_FP64_TEX"] = "1"  # fp64 through the texture gathers, every mode
for m in ("surface", "additive", "mip", "alpha"):
    dev.render(v8, [P.ViewParams(azimuth_deg=a, image_dim=32, steps=48, mode=m, threshold=60) for a in (0.0, 37.0)],
               channels=4 if m in ("mip", "alpha") else 1)
del os.environ["CTP_RENDER_FP64_TEX"]
dev.render(v8, [P.ViewParams(azimuth_deg=15.0, image_dim=32, steps=48, mode="mip")], channels=4, fp32=True)
dev.render(v8, [P.ViewParams(azimuth_deg=15.0, image_dim=32, steps=48, mode="alpha")], channels=4, fp32=True)
dev.image_hist(torch.zeros((3, 16, 16), dtype=torch.uint8, device="cuda"))
# config-5 stream processor at a small shape
ps = PreviewStream((128, 96, 96), torch.uint16, thumb_dim=32, n_views=2)
ps.process(synth.generate(synth.small((128, 96, 96), dtype="u16", seed=3)))
torch.cuda.synchronize()
print("sanitize smoke done", int(hist.sum().item()), int(h16.sum().item()))
