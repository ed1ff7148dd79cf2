"""One device-deflate launch over the c2 512-scheme atlases (8 x 4096^2), for ncu."""
import sys
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
import torch  # noqa: E402

from paper_2311_15038_b200 import _lib, device as dev, synth  # noqa: E402
from paper_2311_15038_b200.device import AtlasSpec  # noqa: E402
from paper_2311_15038_b200.pipeline import plan_preview, run_preview  # noqa: E402
from paper_2311_15038_b200.png import deflate_device  # noqa: E402
from paper_2311_15038_b200.types import plan_scheme  # noqa: E402

_lib.load()
spec = synth.config("c2")
vol = synth.generate(spec)
res = run_preview(vol, plan_preview(spec.shape, {512: AtlasSpec.of(plan_scheme(512))}))
del vol
f = dev.png_filter(res.atlases[512])
deflate_device(f)
torch.cuda.synchronize()
print("done")
