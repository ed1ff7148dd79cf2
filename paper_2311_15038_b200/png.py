"""Atlas PNG writing: ``save_slicemaps`` (slicemap.py:158-166).

The reference writes every atlas with ``Image.fromarray(atlas, "L").save(...)``:
one thread filters and deflates 16 MB per 4096^2 atlas.  Here the PNG scanline
filter (adaptive per row, ``ctp_png_filter_u8``) runs on the device over all
atlases of a set at once, and the host deflates blocks of filtered rows in
parallel: each block is an independent raw-deflate stream ended by a full
flush (the last by Z_FINISH), so their concatenation is one valid zlib stream
(the pigz construction); the Adler-32 is computed over the filtered bytes.
Files, names and ``manifest.json`` are the reference's; the pixels round-trip
losslessly through any PNG decoder (tests: Pillow).  The compressed bytes are
not Pillow's (different filter choice / block boundaries), which nothing in
the reference depends on (load_slicemaps, slicemap.py:169-197, decodes).
"""
from __future__ import annotations

import json
import struct
import zlib
from concurrent.futures import ThreadPoolExecutor
from pathlib import Path

import numpy as np
import torch

_SIG = b"\x89PNG\r\n\x1a\n"
_POOL: ThreadPoolExecutor | None = None


def _pool() -> ThreadPoolExecutor:
    global _POOL
    if _POOL is None:
        import os
        _POOL = ThreadPoolExecutor(max_workers=max(2, min(32, os.cpu_count() or 4)))
    return _POOL


def _chunk(tag: bytes, data: bytes) -> bytes:
    return struct.pack(">I", len(data)) + tag + data + struct.pack(">I", zlib.crc32(tag + data) & 0xFFFFFFFF)


def _deflate_block(mv, level: int, last: bool) -> bytes:
    c = zlib.compressobj(level, zlib.DEFLATED, -15, 9)
    return c.compress(mv) + c.flush(zlib.Z_FINISH if last else zlib.Z_FULL_FLUSH)


def _submit(filtered: np.ndarray, level: int, block_rows: int):
    h, w1 = filtered.shape
    raw = memoryview(np.ascontiguousarray(filtered).reshape(-1))
    step = block_rows * w1
    starts = list(range(0, h * w1, step))
    pool = _pool()
    futs = [pool.submit(_deflate_block, raw[a:a + step], level, i == len(starts) - 1) for i, a in enumerate(starts)]
    adler = pool.submit(zlib.adler32, raw)
    return h, w1, futs, adler


def _assemble(h: int, w1: int, futs, adler) -> bytes:
    body = b"".join(f.result() for f in futs)
    z = b"\x78\x9c" + body + struct.pack(">I", adler.result() & 0xFFFFFFFF)
    ihdr = struct.pack(">IIBBBBB", w1 - 1, h, 8, 0, 0, 0, 0)  # 8-bit grayscale, no interlace
    return _SIG + _chunk(b"IHDR", ihdr) + _chunk(b"IDAT", z) + _chunk(b"IEND", b"")


def png_from_filtered(filtered: np.ndarray, level: int = 6, block_rows: int = 256) -> bytes:
    """PNG file bytes of one grayscale image from its filtered scanlines (H, W + 1)."""
    return _assemble(*_submit(filtered, level, block_rows))


def encode_pngs(images, level: int = 6, block_rows: int = 256) -> list[bytes]:
    """PNG bytes of each (H, W) u8 image of ``images``: a numpy (n, H, W) array, a CUDA
    tensor, or a list of them (sets of different sizes).  One device filter launch
    per array, then every deflate block of every image in flight on the host pool."""
    from . import device as dev
    stacks = images if isinstance(images, (list, tuple)) else [images]
    jobs = []
    for st in stacks:
        t = st if isinstance(st, torch.Tensor) else torch.from_numpy(np.ascontiguousarray(st))
        if not t.is_cuda:
            t = t.to("cuda", non_blocking=False)
        filt = dev.png_filter(t.contiguous()).cpu().numpy()
        jobs += [_submit(filt[i], level, block_rows) for i in range(filt.shape[0])]
    return [_assemble(*j) for j in jobs]


def save_slicemaps(sset, out_dir, level: int = 6) -> Path:
    """slicemap.py:158-166: atlases as PNG (``sm_<s>_<i>.png``) + ``manifest.json``."""
    out_dir = Path(out_dir)
    out_dir.mkdir(parents=True, exist_ok=True)
    names = sset.scheme.atlas_names()
    pngs = encode_pngs(np.stack(sset.atlases), level)
    for name, data in zip(names, pngs):
        (out_dir / name).write_bytes(data)
    manifest_path = out_dir / "manifest.json"
    manifest_path.write_text(json.dumps(sset.manifest(), indent=2) + "\n")
    return manifest_path
