"""Ingest straight into the device path.

ctprev stores a volume as ``<name>.raw`` (x-fastest voxel bytes) plus a JSON
header ``<name>.json`` (``save_volume``, volume.py:205-226) and reads it back
whole with ``np.fromfile`` (``load_volume``, volume.py:229-249).  For a 16 GiB
scan that is a 16 GiB host array before the first GPU byte moves.  Here the
header is validated exactly as ``load_volume`` does (same checks, same order,
same error classes), then the raw file streams through a small ring of pinned
host chunks: reading chunk c+1 from disk overlaps chunk c's H2D copy and fused
pass (``PreviewSession.run_reader``), and only ``ring`` chunks of host memory
are ever held.  The top ``n_top`` slices (the artifact-bin slab, mask.py:227)
are read first -- they are the END of the file.
"""
from __future__ import annotations

import json
import os
from pathlib import Path

import numpy as np
import torch

from .device import AtlasSpec
from .errors import DimensionMismatch, InvalidManifest, MissingSlice, UnsupportedPixelFormat
from .pipeline import PreviewSession, check_top
from .types import FACTORY, plan_scheme


def read_header(header_path) -> tuple[tuple[int, int, int], Path, object]:
    """volume.py:229-247: ((nz, ny, nx), raw path, voxel_size_um) or the reference's error."""
    header_path = Path(header_path)
    try:
        header = json.loads(header_path.read_text())
    except (OSError, json.JSONDecodeError) as exc:
        raise InvalidManifest(f"{header_path}: {exc}") from exc
    if header.get("dtype") != "u8":
        raise UnsupportedPixelFormat(f"dtype {header.get('dtype')!r}, expected 'u8'")
    if header.get("order") != "xyz":
        raise UnsupportedPixelFormat(f"order {header.get('order')!r}, expected 'xyz'")
    try:
        nx, ny, nz = (int(d) for d in header["dims"])
    except (KeyError, TypeError, ValueError) as exc:
        raise InvalidManifest(f"{header_path}: bad 'dims'") from exc
    raw_path = header_path.with_suffix(".raw")
    if not raw_path.is_file():
        raise MissingSlice(str(raw_path))
    size = os.path.getsize(raw_path)
    if size != nx * ny * nz:
        raise DimensionMismatch(f"{raw_path.name}: {size} bytes, header implies {nx * ny * nz}")
    return (nz, ny, nx), raw_path, header.get("voxel_size_um")


def _check_session_args(session, shape, n_top: int, frac: float, what: str) -> None:
    """Before any read: the artifact-bin arguments as artifact_bins checks them
    (mask.py:223-226), and a reused session must match the volume and arguments."""
    check_top(n_top, frac, shape[0])
    if session is None:
        return
    if session.shape != shape:
        raise DimensionMismatch(f"session shape {session.shape} != {what} {shape}")
    if (session.n_top, session.frac) != (n_top, frac):
        raise ValueError(f"session built for n_top={session.n_top}, frac={session.frac}; "
                         f"called with n_top={n_top}, frac={frac}")


class RawReader:
    """Reads z-slabs of a raw x-fastest volume into caller-provided (pinned) arrays,
    with ``threads`` concurrent ``preadv`` calls of ``piece`` bytes (the GIL is
    released while the kernel copies, so pieces land in parallel)."""

    def __init__(self, raw_path, shape, dtype=np.uint8, threads: int = 8, piece: int = 8 << 20):
        from concurrent.futures import ThreadPoolExecutor
        self.path = Path(raw_path)
        self.shape = tuple(shape)
        self.slice_bytes = self.shape[1] * self.shape[2] * np.dtype(dtype).itemsize
        self.piece = piece
        self._fd = os.open(self.path, os.O_RDONLY)
        self._pool = ThreadPoolExecutor(max_workers=threads) if threads > 1 else None

    def _read_piece(self, mv, offset: int) -> None:
        got = 0
        while got < len(mv):
            n = os.preadv(self._fd, [mv[got:]], offset + got)
            if not n:
                raise DimensionMismatch(f"{self.path.name}: short read at byte {offset + got}")
            got += n

    def __call__(self, z0: int, z1: int, out: np.ndarray) -> None:
        want = (z1 - z0) * self.slice_bytes
        mv = memoryview(out.reshape(-1).view(np.uint8))[:want]
        base = z0 * self.slice_bytes
        starts = range(0, want, self.piece)
        if self._pool is None or len(starts) == 1:
            for a in starts:
                self._read_piece(mv[a:a + self.piece], base + a)
            return
        for f in [self._pool.submit(self._read_piece, mv[a:a + self.piece], base + a) for a in starts]:
            f.result()

    def close(self) -> None:
        if self._pool is not None:
            self._pool.shutdown()
        os.close(self._fd)

    def __enter__(self):
        return self

    def __exit__(self, *exc):
        self.close()


def preview_from_raw(header_path, schemes=(512, 256, 128), n_top: int = 3, frac: float = 0.0005,
                     chunk_slices: int = 64, session: PreviewSession | None = None, threads: int = 8):
    """``preview_pipeline(load_volume(header_path), schemes)`` without materialising
    the volume on the host: returns the same ``PreviewResult`` (histogram,
    artifact bins, per-scheme SlicemapSets).  Pass a ``session`` to reuse its
    pinned and device buffers across volumes of one shape; ``threads`` concurrent
    preadv calls fill each pinned chunk."""
    from .ops import PreviewResult
    shape, raw_path, _ = read_header(header_path)
    _check_session_args(session, shape, n_top, frac, "volume")
    sch = {}
    for sc in schemes:
        sc = plan_scheme(sc) if isinstance(sc, int) else sc
        sch[sc.s] = sc
    if session is None:
        session = PreviewSession(shape, torch.uint8, {s: AtlasSpec.of(sc) for s, sc in sch.items()}, n_top=n_top,
                                 frac=frac, chunk_slices=chunk_slices)
    with RawReader(raw_path, shape, threads=threads) as rd:
        out = session.run_reader(rd)
    slicemaps = {}
    for s, sc in sch.items():
        a = out["atlases"][s].numpy()
        slicemaps[s] = FACTORY.SlicemapSet(scheme=sc, atlases=tuple(a[m].copy() for m in range(sc.map_count)))
    flags = out["flags"].numpy()
    return PreviewResult(out["hist"].numpy().copy(), frozenset(int(b) for b in np.nonzero(flags)[0]), slicemaps,
                         {}, None)


# ---------------------------------------------------------------------------
# slice stacks (volume.py:167-202 load_slice_stack): a JSON manifest listing one
# 8-bit grayscale PNG per z slice.  The reference decodes every slice serially
# into one host array; here the manifest is validated as load_slice_stack does
# (same checks, same error classes), and the slices are decoded by a thread pool
# (Pillow releases the GIL while decoding) straight into the pinned chunk ring of
# PreviewSession.run_reader, so decoding chunk c+1 overlaps chunk c's H2D copy
# and fused pass and no whole-volume host array exists.

def _open_slice(path: Path):
    from PIL import Image
    if not path.is_file():
        raise MissingSlice(str(path))                      # volume.py:157-158
    im = Image.open(path)
    if im.mode != "L":                                     # volume.py:160-163
        im.close()
        raise UnsupportedPixelFormat(f"{path.name}: mode {im.mode!r}, need 8-bit grayscale ('L')")
    return im


class ManifestPaths(list):
    """The resolved slice paths, with ``names``: the manifest entries as written
    (the reference formats its slice-size message with the entry, volume.py:199)."""

    names: list


def read_manifest(manifest_path) -> tuple[list, tuple[int, int, int]]:
    """volume.py:176-196: (slice paths in z order, (nz, ny, nx)) or the reference's error."""
    manifest_path = Path(manifest_path)
    try:
        manifest = json.loads(manifest_path.read_text())
    except (OSError, json.JSONDecodeError) as exc:
        raise InvalidManifest(f"{manifest_path}: {exc}") from exc
    if not isinstance(manifest, dict) or "slices" not in manifest:
        raise InvalidManifest(f"{manifest_path}: no 'slices' key")
    if manifest.get("bit_depth", 8) != 8:
        raise UnsupportedPixelFormat(f"bit_depth {manifest.get('bit_depth')}, only 8 is supported")
    rel = manifest["slices"]
    if not isinstance(rel, list) or len(rel) == 0:
        raise InvalidManifest(f"{manifest_path}: manifest lists no slices")
    paths = ManifestPaths(manifest_path.parent / name for name in rel)
    paths.names = [str(name) for name in rel]
    with _open_slice(paths[0]) as im:
        nx, ny = im.size
    return paths, (len(paths), ny, nx)


class SliceStackReader:
    """``read(z0, z1, out)`` for PreviewSession.run_reader: decodes slices [z0, z1)
    of a stack into ``out`` with ``threads`` concurrent Pillow decodes; every slice
    is checked against the first slice's size (volume.py:197-201)."""

    def __init__(self, paths, shape, threads: int = 8):
        from concurrent.futures import ThreadPoolExecutor
        self.paths = list(paths)
        self.names = list(getattr(paths, "names", None) or [p.name for p in self.paths])
        self.shape = tuple(shape)
        self._pool = ThreadPoolExecutor(max_workers=threads) if threads > 1 else None

    def _decode(self, z: int, dst: np.ndarray) -> None:
        path = self.paths[z]
        with _open_slice(path) as im:
            if (im.size[1], im.size[0]) != self.shape[1:]:
                raise DimensionMismatch(f"slice {self.names[z]}: {im.size} does not match first slice "
                                        f"{(self.shape[2], self.shape[1])}")
            dst[...] = np.asarray(im, dtype=np.uint8)

    def __call__(self, z0: int, z1: int, out: np.ndarray) -> None:
        if self._pool is None:
            for z in range(z0, z1):
                self._decode(z, out[z - z0])
            return
        for f in [self._pool.submit(self._decode, z, out[z - z0]) for z in range(z0, z1)]:
            f.result()

    def close(self) -> None:
        if self._pool is not None:
            self._pool.shutdown()

    def __enter__(self):
        return self

    def __exit__(self, *exc):
        self.close()


def preview_from_slice_stack(manifest_path, schemes=(512, 256, 128), n_top: int = 3, frac: float = 0.0005,
                             chunk_slices: int = 64, session: PreviewSession | None = None, threads: int = 8):
    """``preview_pipeline(load_slice_stack(manifest_path), schemes)`` with the slices
    decoded in parallel straight into the streaming pass: returns the same
    ``PreviewResult`` (histogram, artifact bins, per-scheme SlicemapSets)."""
    from .ops import PreviewResult
    paths, shape = read_manifest(manifest_path)
    _check_session_args(session, shape, n_top, frac, "stack")
    sch = {}
    for sc in schemes:
        sc = plan_scheme(sc) if isinstance(sc, int) else sc
        sch[sc.s] = sc
    if session is None:
        session = PreviewSession(shape, torch.uint8, {s: AtlasSpec.of(sc) for s, sc in sch.items()}, n_top=n_top,
                                 frac=frac, chunk_slices=chunk_slices)
    with SliceStackReader(paths, shape, threads=threads) as rd:
        out = session.run_reader(rd)
    slicemaps = {}
    for s, sc in sch.items():
        a = out["atlases"][s].numpy()
        slicemaps[s] = FACTORY.SlicemapSet(scheme=sc, atlases=tuple(a[m].copy() for m in range(sc.map_count)))
    flags = out["flags"].numpy()
    return PreviewResult(out["hist"].numpy().copy(), frozenset(int(b) for b in np.nonzero(flags)[0]), slicemaps,
                         {}, None)
