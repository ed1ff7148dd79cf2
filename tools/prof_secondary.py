"""One launch of each secondary kernel on config-2-sized data (for an ncu launch list):
general downscale 1024^3 -> 512^3 and -> 300^3, atlas encode of the 512^3 level,
PNG filter + device deflate of its 8 x 4096^2 atlases, circle mask, 256-bin histogram."""
import sys
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
import torch  # noqa: E402

from paper_2311_15038_b200 import _lib, device as dev, synth  # noqa: E402
from paper_2311_15038_b200.device import AtlasSpec  # noqa: E402
from paper_2311_15038_b200.png import deflate_device  # noqa: E402
from paper_2311_15038_b200.types import plan_scheme  # noqa: E402

_lib.load()
vol = synth.generate(synth.config("c2"))
lv = dev.downscale(vol, (512, 512, 512))
dev.downscale(vol, (300, 300, 300))
atl = dev.encode_atlas(lv, AtlasSpec.of(plan_scheme(512)))
f = dev.png_filter(atl)
deflate_device(f)
dev.circle_mask(vol, 511.5, 500.25, 480.0 ** 2)
dev.hist_u8(vol)
torch.cuda.synchronize()
print("done")
