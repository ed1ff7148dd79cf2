"""Config 1 (256^3): where the 16.4 us of the one-launch step go -- the fused pass alone (LUT given, plain launch),
the artifact-LUT launch alone, and the cooperative step, each replayed from a CUDA graph."""
import sys
from pathlib import Path
sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
import torch
from paper_2311_15038_b200 import _lib, device as dev, synth
from paper_2311_15038_b200.device import AtlasSpec
from paper_2311_15038_b200.pipeline import plan_preview, run_preview

_lib.load()
spec = synth.config("c1")
vol = synth.generate(spec)
plan = plan_preview(spec.shape, {256: AtlasSpec(256, 4096, 16, 1)})
res = run_preview(vol, plan)
lut, _ = dev.artifact_lut(vol)
hist = torch.zeros(256, dtype=torch.int64, device="cuda")
outs = dev.preview(vol, lut, plan.fused, hist=hist)


def timed(name, fn, n=500):
    side = torch.cuda.Stream()
    side.wait_stream(torch.cuda.current_stream())
    with torch.cuda.stream(side):
        for _ in range(3):
            fn()
    torch.cuda.current_stream().wait_stream(side)
    g = torch.cuda.CUDAGraph()
    with torch.cuda.graph(g):
        fn()
    for _ in range(20):
        g.replay()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(n):
        g.replay()
    e1.record()
    torch.cuda.synchronize()
    print(f"{name:44s} {e0.elapsed_time(e1) / n * 1e3:7.2f} us")


timed("cooperative step (LUT phase + pass)", lambda: run_preview(vol, plan, hist=res.hist))
timed("fused pass alone (LUT given, plain launch)", lambda: dev.preview(vol, lut, plan.fused, hist=hist, out_tensors=outs))
timed("artifact LUT launch alone", lambda: dev.artifact_lut(vol))
empty = torch.zeros(1, device="cuda")
timed("empty elementwise kernel (launch floor)", lambda: empty.add_(1))
timed("copy 16 MiB -> 16 MiB (same bytes, torch)", lambda: outs[0].view(-1).copy_(vol.view(-1)) if 0 in outs else None)
