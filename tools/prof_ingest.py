"""Time ingest.preview_from_raw on config 2 (1 GiB raw file, page cache hot) for
several reader thread counts.

usage: python tools/prof_ingest.py [--threads 4,8,16] [--chunk 64]
"""
import argparse
import json
import os
import sys
import tempfile
import time
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
import torch  # noqa: E402

from paper_2311_15038_b200 import _lib, synth  # noqa: E402
from paper_2311_15038_b200.device import AtlasSpec  # noqa: E402
from paper_2311_15038_b200.ingest import preview_from_raw  # noqa: E402
from paper_2311_15038_b200.pipeline import PreviewSession  # noqa: E402
from paper_2311_15038_b200.types import plan_scheme  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--threads", default="4,8,16")
ap.add_argument("--chunk", type=int, default=64)
a = ap.parse_args()
_lib.load()
spec = synth.config("c2")
vol = synth.generate(spec)
nz, ny, nx = spec.shape
with tempfile.TemporaryDirectory() as td:
    vol.cpu().numpy().tofile(os.path.join(td, "c2.raw"))
    with open(os.path.join(td, "c2.json"), "w") as f:
        json.dump({"dims": [nx, ny, nz], "dtype": "u8", "order": "xyz", "voxel_size_um": None}, f)
    del vol
    sess = PreviewSession(spec.shape, torch.uint8, {s: AtlasSpec.of(plan_scheme(s)) for s in (512, 256, 128)},
                          chunk_slices=a.chunk)
    hdr = os.path.join(td, "c2.json")
    preview_from_raw(hdr, session=sess)
    for th in [int(x) for x in a.threads.split(",")]:
        ts = []
        for _ in range(3):
            t0 = time.perf_counter()
            preview_from_raw(hdr, session=sess, threads=th)
            ts.append(time.perf_counter() - t0)
        print(f"threads={th} chunk={a.chunk} best_ms={min(ts) * 1e3:.1f} GB/s={nz * ny * nx / min(ts) / 1e9:.1f}")
