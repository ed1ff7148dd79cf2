"""Time the small secondary kernels (CUDA events, clocks warmed up): atlas decode of the
512 scheme, the u16 filter o rescale LUT (vector path), atlas encode, the 8-bit LUT.

usage: python tools/prof_small_kernels.py
"""
import sys
import time
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
import torch  # noqa: E402

from paper_2311_15038_b200 import _lib, device as dev, synth  # noqa: E402
from paper_2311_15038_b200.device import AtlasSpec  # noqa: E402
from paper_2311_15038_b200.types import plan_scheme  # noqa: E402

_lib.load()


def bench(name, fn, nbytes, reps=50):
    fn()
    t0 = time.perf_counter()
    while time.perf_counter() - t0 < 0.5:
        fn()
        torch.cuda.synchronize()
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    a.record()
    for _ in range(reps):
        fn()
    b.record()
    torch.cuda.synchronize()
    ms = a.elapsed_time(b) / reps
    print(f"{name:40s} {ms * 1e3:9.1f} us  {nbytes / ms / 1e6:8.0f} GB/s")


vol = synth.generate(synth.config("c2"))
lv = dev.downscale(vol, (512, 512, 512))
sp = AtlasSpec.of(plan_scheme(512))
atl = dev.encode_atlas(lv, sp)
assert torch.equal(dev.decode_atlas(atl, sp), lv)
bench("encode_atlas 512^3 -> 8 x 4096^2", lambda: dev.encode_atlas(lv, sp), 2 * lv.numel())
bench("decode_atlas 8 x 4096^2 -> 512^3", lambda: dev.decode_atlas(atl, sp), 2 * lv.numel())
lut, _ = dev.artifact_lut(vol)
bench("lut_apply_u8 1 GiB", lambda: dev.lut_apply_u8(vol, lut), 2 * vol.numel())
del vol
v16 = synth.generate(synth.small((256, 1024, 1024), dtype="u16", seed=2))
lut16, _ = dev.artifact_lut(v16)
bench("lut_apply_u16 256 Mi voxels", lambda: dev.lut_apply_u16(v16, lut16), 3 * v16.numel())
