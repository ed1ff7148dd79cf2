"""Config 2 from a PNG slice stack (ctprev's load_slice_stack format, volume.py:167-202):
time ingest.preview_from_slice_stack (parallel decode straight into the streaming pass)
against the reference's way of ingesting (serial Pillow decode into one host array).

usage: python tools/prof_stack.py [--threads 16] [--n 1024]
"""
import argparse
import json
import os
import sys
import tempfile
import time
from concurrent.futures import ThreadPoolExecutor
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
import numpy as np  # noqa: E402
import torch  # noqa: E402
from PIL import Image  # noqa: E402

from paper_2311_15038_b200 import _lib, synth  # noqa: E402
from paper_2311_15038_b200.device import AtlasSpec  # noqa: E402
from paper_2311_15038_b200.ingest import preview_from_slice_stack  # noqa: E402
from paper_2311_15038_b200.pipeline import PreviewSession  # noqa: E402
from paper_2311_15038_b200.types import plan_scheme  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--threads", type=int, default=os.cpu_count() or 8)
a = ap.parse_args()
_lib.load()
spec = synth.config("c2")
vol = synth.generate(spec).cpu().numpy()
nz, ny, nx = vol.shape
with tempfile.TemporaryDirectory() as td:
    td = Path(td)
    names = [f"s_{z:04d}.png" for z in range(nz)]
    t0 = time.perf_counter()
    with ThreadPoolExecutor(a.threads) as ex:
        list(ex.map(lambda z: Image.fromarray(vol[z]).save(td / names[z], compress_level=1), range(nz)))
    print(f"wrote {nz} PNG slices in {time.perf_counter() - t0:.1f} s "
          f"({sum((td / n).stat().st_size for n in names) / 1e6:.0f} MB)")
    (td / "stack.json").write_text(json.dumps({"name": "c2", "slices": names, "bit_depth": 8}))
    schemes = (512, 256, 128)
    sess = PreviewSession(vol.shape, torch.uint8, {s: AtlasSpec.of(plan_scheme(s)) for s in schemes})
    preview_from_slice_stack(td / "stack.json", schemes, session=sess, threads=a.threads)
    ts = []
    for _ in range(2):
        t0 = time.perf_counter()
        res = preview_from_slice_stack(td / "stack.json", schemes, session=sess, threads=a.threads)
        ts.append(time.perf_counter() - t0)
    print(f"preview_from_slice_stack: {min(ts) * 1e3:.0f} ms/volume ({nz * ny * nx / min(ts) / 1e9:.2f} GVoxel/s), "
          f"{a.threads} decode threads; hist ok={int(res.histogram.sum()) == vol.size}")
    t0 = time.perf_counter()
    stack = np.empty_like(vol)
    for z in range(nz):  # the reference's ingest: serial decode (volume.py:193-201)
        with Image.open(td / names[z]) as im:
            stack[z] = np.asarray(im, dtype=np.uint8)
    t_ref = time.perf_counter() - t0
    print(f"serial decode into one array (the reference's load_slice_stack): {t_ref * 1e3:.0f} ms; "
          f"equal={np.array_equal(stack, vol)}")
