"""One launch of each kernel besides the fused pass, on config-sized data (for an ncu
capture of every kernel): general downscale 1024^3 -> 512^3 (warp-per-row kernel) and the
config-5 level 768^2 x 1024 -> 512^3, atlas encode / decode, PNG filter + device deflate,
circle mask (span kernels), 256-bin and 4096-bin histograms, the filter LUT kernels (u8,
u16), per-image histograms (image_entropy), and the renderers: fp64 surface and additive
(the reference's modes), fp32 MIP (row planes) and alpha."""
import math
import sys
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
import torch  # noqa: E402

from paper_2311_15038_b200 import _lib, device as dev, synth  # noqa: E402
from paper_2311_15038_b200.device import AtlasSpec  # noqa: E402
from paper_2311_15038_b200.png import deflate_device  # noqa: E402
from paper_2311_15038_b200.types import ViewParams, plan_scheme  # noqa: E402

_lib.load()
vol = synth.generate(synth.config("c2"))
lv = dev.downscale(vol, (512, 512, 512))
l1 = synth.generate(synth.small((1024, 768, 768), seed=5, n_shells=6))
dev.downscale(l1, (512, 512, 512))
del l1
spec512 = AtlasSpec.of(plan_scheme(512))
atl = dev.encode_atlas(lv, spec512)
dev.decode_atlas(atl, spec512)
f = dev.png_filter(atl)
deflate_device(f)
dev.circle_mask(vol, 511.5, 500.25, 480.0 ** 2)
dev.hist_u8(vol)
lut, _ = dev.artifact_lut(vol)
dev.lut_apply_u8(vol, lut)
v16 = synth.generate(synth.small((256, 1024, 1024), dtype="u16", seed=2))
dev.hist_u16(v16)
lut16, _ = dev.artifact_lut(v16)
dev.lut_apply_u16(v16, lut16)
del v16
steps = math.ceil(4 * math.sqrt(3.0) / 2.0 * 1024)
imgs = dev.render(vol, [ViewParams(azimuth_deg=30.0 * k, image_dim=1024, steps=steps, mode="surface", threshold=100)
                        for k in range(2)], channels=1)
dev.image_hist(imgs)
dev.render(vol, [ViewParams(azimuth_deg=10.0 * k, image_dim=1024, steps=steps, mode="additive") for k in range(2)],
           channels=1)
dev.render(vol, [ViewParams(azimuth_deg=10.0 * k, image_dim=1024, steps=steps, mode="mip") for k in range(8)],
           channels=4, fp32=True)
dev.render(vol, [ViewParams(azimuth_deg=10.0 * k, image_dim=1024, steps=steps, mode="alpha") for k in range(8)],
           channels=4, fp32=True)
torch.cuda.synchronize()
print("done")
