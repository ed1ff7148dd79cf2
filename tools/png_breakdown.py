"""Where the time of encode_pngs_device goes on the c2 atlases (cProfile, host side)."""
import cProfile
import pstats
import sys
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
import torch  # noqa: E402

from paper_2311_15038_b200 import _lib, synth  # noqa: E402
from paper_2311_15038_b200.device import AtlasSpec  # noqa: E402
from paper_2311_15038_b200.pipeline import plan_preview, run_preview  # noqa: E402
from paper_2311_15038_b200.png import encode_pngs_device  # noqa: E402
from paper_2311_15038_b200.types import plan_scheme  # noqa: E402

_lib.load()
spec = synth.config("c2")
vol = synth.generate(spec)
schemes = {s: AtlasSpec.of(plan_scheme(s)) for s in (512, 256, 128)}
res = run_preview(vol, plan_preview(spec.shape, schemes))
del vol
atl = [res.atlases[s] for s in schemes]
encode_pngs_device(atl)
torch.cuda.synchronize()
pr = cProfile.Profile()
pr.enable()
encode_pngs_device(atl)
pr.disable()
pstats.Stats(pr).sort_stats("cumulative").print_stats(18)
