"""Config 5: a stream of anisotropic 12-bit volumes, each reduced end to end on
one GPU (one volume per GPU when several are present: replicas, no collective).

Per volume, the composition SURVEY.md s8(d) derives for config 5 (the reference
has no uint16 path; the 12-bit rules are config 3's):
  * 4096-bin histogram, artifact bins of the top 3 slices, filter o 16->8 rescale;
  * pyramid levels L1..L4 of the filtered volume, each straight from full
    resolution (exact block sums, volume.py:306-308 rounding, pipeline.py:275);
  * every level packed into a planned slicemap scheme with the reference's
    ``_scheme_volume`` + ``_pad_to_cube`` semantics (pipeline.py:215-237): the
    scheme is the smallest planned edge (128/256/512, slicemap.py:40) holding
    the level's largest axis, capped at 512; a level larger than its scheme is
    box-downscaled to ``min(s, n)`` per axis (volume.py:277-309, any ratio) and
    every level is zero-padded to s^3.  For 1536^2 x 2048:
        L1 768^2 x 1024 -> 512^2 x 512 (1.5:1 in x, y; 2:1 in z) -> scheme 512
        L2 384^2 x 512  -> identity, padded                       -> scheme 512
        L3 192^2 x 256  -> identity, padded                       -> scheme 256
        L4  96^2 x 128  -> identity, padded                       -> scheme 128
  * a 36-view MIP strip of ``thumb_dim``^2 RGBA8 thumbnails rendered from the
    first level whose largest axis fits ``thumb_dim`` (L2 for 512), 0.5-voxel
    steps of that level.
One fused pass writes the identity levels' padded atlases directly and the
levels that are needed dense (the downscaled L1, the thumbnail level); then the
general-ratio kernel, the atlas packer and one render batch.

``variant="pow2-1024"`` is round 1's layout, kept under that name: every level
in the smallest power-of-two scheme holding it (L1 -> SlicemapScheme(1024, 4096,
4, 64), no general-ratio level).
"""
from __future__ import annotations

import math
from dataclasses import dataclass

import torch

from . import device as dev
from .device import AtlasSpec
from .types import ViewParams, plan_scheme

PLANNED = (128, 256, 512)  # slicemap.py:40


def scheme_of_level(level_shape) -> int:
    """The planned scheme edge for a level: smallest of 128/256/512 holding its largest axis, capped at 512."""
    edge = max(level_shape)
    for s in PLANNED:
        if edge <= s:
            return s
    return PLANNED[-1]


def scheme_pow2(level_shape) -> AtlasSpec:
    """variant "pow2-1024": smallest power-of-two scheme (grid 8, or 4096 // s for s > 512) holding every axis."""
    edge = max(level_shape)
    s = 128
    while s < edge:
        s *= 2
    if s <= 512:
        return AtlasSpec(s, 8 * s, 8, -(-s // 64))
    grid = 4096 // s
    if grid < 1:
        raise ValueError(f"level {level_shape} larger than one 4096^2 atlas cell")
    return AtlasSpec(s, grid * s, grid, -(-s // (grid * grid)))


# round 1's name for scheme_pow2
scheme_for = scheme_pow2


@dataclass
class StreamResult:
    hist: torch.Tensor
    flags: torch.Tensor
    atlases: dict       # level -> uint8 (maps, A, A)
    thumbs: torch.Tensor  # (n_views, dim, dim, 4) uint8


class PreviewStream:
    """Reusable per-shape buffers; ``process(vol)`` runs one volume on the current stream."""

    def __init__(self, shape, dtype=torch.uint16, n_levels: int = 4, thumb_dim: int = 512, n_views: int = 36,
                 device=None, variant: str = "scheme"):
        if variant not in ("scheme", "pow2-1024"):
            raise ValueError(f"unknown variant {variant!r}")
        self.shape = tuple(shape)
        self.variant = variant
        self.device = torch.device(device or "cuda")
        nz, ny, nx = self.shape
        self.level_shape = {l: (nz >> l, ny >> l, nx >> l) for l in range(1, n_levels + 1)}
        self.levels, self.targets = {}, {}
        for l, (lz, ly, lx) in self.level_shape.items():
            if variant == "scheme":
                s = scheme_of_level((lz, ly, lx))
                self.levels[l] = AtlasSpec.of(plan_scheme(s))
                self.targets[l] = (min(s, lx), min(s, ly), min(s, lz))   # _scheme_volume, pipeline.py:221-222
            else:
                self.levels[l] = scheme_pow2((lz, ly, lx))
                self.targets[l] = (lx, ly, lz)
        self.thumb_level = next((l for l, sh in self.level_shape.items() if max(sh) <= thumb_dim), n_levels)
        tl = self.thumb_level
        self.thumb_shape = self.level_shape[tl]
        # levels produced dense by the pass: those that must be downscaled, and the thumbnail level
        self.dense = {l for l, (lz, ly, lx) in self.level_shape.items() if self.targets[l] != (lx, ly, lz)} | {tl}
        self.nbins = dev.NBINS_U16 if dtype == torch.uint16 else dev.NBINS_U8
        self.hist = torch.empty(self.nbins, dtype=torch.int64, device=self.device)
        self.dense_bufs = {l: torch.empty(self.level_shape[l], dtype=torch.uint8, device=self.device)
                           for l in self.dense}
        self.atlases = {}  # the pass writes the identity levels' atlases in place; the others are packed per call
        for l, sp in self.levels.items():
            if l not in self.dense:
                tx, ty, tz = self.targets[l]
                self.atlases[l] = dev.alloc_level((tz, ty, tx), sp, self.device)
        n_max = max(self.thumb_shape)
        r = math.sqrt(sum((d / (2.0 * n_max)) ** 2 for d in self.thumb_shape))
        self.steps = math.ceil(4 * r * n_max)  # 0.5-voxel steps over the 2R window (render.py:139)
        self.views = [ViewParams(azimuth_deg=360.0 * k / n_views, image_dim=thumb_dim, steps=self.steps, mode="mip")
                      for k in range(n_views)]
        self.thumbs = torch.empty((n_views, thumb_dim, thumb_dim, 4), dtype=torch.uint8, device=self.device)
        self.trace = None  # a list -> process() appends (phase, CUDA event) after each phase (bench breakdown)

    def _mark(self, name: str) -> None:
        torch.cuda.nvtx.mark(f"stream.{name}")
        if self.trace is not None:
            e = torch.cuda.Event(enable_timing=True)
            e.record()
            self.trace.append((name, e))

    @property
    def product_bytes(self) -> int:
        return sum(sp.map_count * sp.atlas_dim ** 2 for sp in self.levels.values()) + self.thumbs.numel()

    def process(self, vol: torch.Tensor) -> StreamResult:
        self._mark("start")
        outputs = {l: ("xyz" if l in self.dense else sp) for l, sp in self.levels.items()}
        tensors = {l: (self.dense_bufs[l] if l in self.dense else self.atlases[l]) for l in self.levels}
        _, _, lut, flags = dev.preview_step(vol, outputs, 3, 0.0005, hist=self.hist, out_tensors=tensors)
        self._mark("fused_pass")
        for l in sorted(self.dense):
            lz, ly, lx = self.level_shape[l]
            src = self.dense_bufs[l]
            if self.targets[l] != (lx, ly, lz):  # _scheme_volume: the general-ratio box mean (volume.py:277-309)
                src = dev.downscale(src, self.targets[l])
                self._mark(f"downscale_L{l}")
            self.atlases[l] = dev.encode_atlas(src, self.levels[l])     # pack + _pad_to_cube (pipeline.py:226-237)
            self._mark(f"encode_L{l}")
        dev.render(self.dense_bufs[self.thumb_level], self.views, channels=4, fp32=True, out=self.thumbs)
        self._mark("mip_strip")
        return StreamResult(self.hist, flags, self.atlases, self.thumbs)
