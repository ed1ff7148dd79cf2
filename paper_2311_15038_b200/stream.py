"""Config 5: a stream of anisotropic 12-bit volumes, each reduced end to end on
one GPU (one volume per GPU when several are present: replicas, no collective).

Per volume (frozen here -- the reference has no uint16 path):
  * 4096-bin histogram, artifact bins of the top 3 slices, filter o 16->8 rescale
    (the c3 rules);
  * power-of-two pyramid levels L1..L4 of the filtered volume (exact block sums,
    volume.py:306-308 rounding, every level from full resolution);
  * every level packed into the slicemap scheme whose edge is the smallest
    power-of-two scheme >= the level's largest dimension, origin-anchored and
    zero-padded (pipeline.py:226-237): for 1536^2 x 2048, L1 768^2 x 1024 ->
    SlicemapScheme(1024, 4096, 4, 64), L2 -> plan 512, L3 -> plan 256, L4 -> plan 128;
  * a 36-view MIP strip of ``thumb_dim``^2 RGBA8 thumbnails rendered from the
    level whose largest dimension equals ``thumb_dim`` (L2 for 512), 0.5-voxel
    steps of that level.
All of it is one fused pass plus one render batch per volume.
"""
from __future__ import annotations

import math
from dataclasses import dataclass

import torch

from . import device as dev
from .device import AtlasSpec
from .types import ViewParams


def scheme_for(level_shape) -> AtlasSpec:
    """Smallest planned-style scheme (grid 8, or grid 4 for 1024) holding every axis of the level."""
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


@dataclass
class StreamResult:
    hist: torch.Tensor
    flags: torch.Tensor
    atlases: dict       # level -> uint8 (maps, A, A)
    thumbs: torch.Tensor  # (n_views, dim, dim, 4) uint8


class PreviewStream:
    """Reusable per-shape buffers; ``process(vol)`` runs one volume on the current stream."""

    def __init__(self, shape, dtype=torch.uint16, n_levels: int = 4, thumb_dim: int = 512, n_views: int = 36,
                 device=None):
        self.shape = tuple(shape)
        self.device = torch.device(device or "cuda")
        nz, ny, nx = self.shape
        self.levels = {}
        for l in range(1, n_levels + 1):
            self.levels[l] = scheme_for((nz >> l, ny >> l, nx >> l))
        self.thumb_level = next((l for l in self.levels if max(nz >> l, ny >> l, nx >> l) <= thumb_dim),
                                n_levels)
        tl = self.thumb_level
        self.thumb_shape = (nz >> tl, ny >> tl, nx >> tl)
        self.nbins = dev.NBINS_U16 if dtype == torch.uint16 else dev.NBINS_U8
        self.hist = torch.empty(self.nbins, dtype=torch.int64, device=self.device)
        self.atlases = {l: dev.alloc_level((nz >> l, ny >> l, nx >> l), sp, self.device) for l, sp in self.levels.items()}
        self.thumb_vol = torch.empty(self.thumb_shape, dtype=torch.uint8, device=self.device)
        n_max = max(self.thumb_shape)
        r = math.sqrt(sum((d / (2.0 * n_max)) ** 2 for d in self.thumb_shape))
        self.steps = math.ceil(4 * r * n_max)  # 0.5-voxel steps over the 2R window (render.py:139)
        self.views = [ViewParams(azimuth_deg=360.0 * k / n_views, image_dim=thumb_dim, steps=self.steps, mode="mip")
                      for k in range(n_views)]
        self.thumbs = torch.empty((n_views, thumb_dim, thumb_dim, 4), dtype=torch.uint8, device=self.device)

    def process(self, vol: torch.Tensor) -> StreamResult:
        outputs = dict(self.levels)
        outputs[self.thumb_level] = "xyz"       # the thumbnail level dense, its atlas packed from it
        outs, _, lut, flags = dev.preview_step(
            vol, outputs, 3, 0.0005, hist=self.hist,
            out_tensors={l: t for l, t in self.atlases.items() if l != self.thumb_level}
            | {self.thumb_level: self.thumb_vol})
        for l, t in outs.items():
            if l != self.thumb_level:
                self.atlases[l] = t
        self.atlases[self.thumb_level] = dev.encode_atlas(self.thumb_vol, self.levels[self.thumb_level])
        dev.render(self.thumb_vol, self.views, channels=4, fp32=True, out=self.thumbs)
        return StreamResult(self.hist, flags, self.atlases, self.thumbs)
