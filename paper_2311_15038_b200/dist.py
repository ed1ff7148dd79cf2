"""z-slab sharding of one volume across the GPUs of a node.

Rank r owns slices [z0_r, z1_r) with every slab height a multiple of 2^nlev,
so no pyramid cell straddles two ranks (no halo).  One step:

  1. the rank holding the top ``n_top`` slices (mask.py:227: the LAST rank)
     builds the artifact LUT from its top-slab histogram and broadcasts it;
  2. every rank runs the fused pass on its slab (global z offset z_base), writing
     its slices straight into the atlas layout;
  3. the 256/4096-bin histograms are summed with an all-reduce (int64);
  4. each rank's atlas byte range -- contiguous because slab heights at every
     level are multiples of the scheme grid (whole cell rows) -- is sent to rank 0.

The compute is injected (``SlabCompute``) so the collective/host logic is the
same code under NCCL on GPUs and under gloo on the CPU in the tests; the
product binds it to the CUDA kernels (``DeviceSlabCompute``).
"""
from __future__ import annotations

from dataclasses import dataclass

import torch
import torch.distributed as dist

from .device import AtlasSpec


def slab_bounds(nz: int, world: int, rank: int, align: int) -> tuple[int, int]:
    """Balanced split of [0, nz) into ``world`` slabs whose heights are multiples of ``align``."""
    if nz % align:
        raise ValueError(f"nz={nz} not a multiple of the slab alignment {align}")
    units = nz // align
    base, extra = divmod(units, world)
    start = rank * base + min(rank, extra)
    count = base + (1 if rank < extra else 0)
    return start * align, (start + count) * align


def slab_alignment(schemes: dict, nlev_of: dict) -> int:
    """Slab height alignment: 2^nlev, and whole atlas cell rows at every level."""
    a = 1 << max(nlev_of.values(), default=0)
    for s, l in nlev_of.items():
        spec = schemes[s]
        a = max(a, spec.grid << l)  # grid slices at level l == grid << l source slices
    return a


def atlas_byte_range(spec: AtlasSpec, k0: int, k1: int) -> tuple[int, int]:
    """Bytes of the atlas set holding level slices [k0, k1) when k0, k1 are cell-row aligned."""
    per = spec.grid * spec.grid

    def off(k):
        m, w = divmod(k, per)
        return m * spec.atlas_dim * spec.atlas_dim + (w // spec.grid) * spec.s * spec.atlas_dim

    if k0 % spec.grid or (k1 % spec.grid and k1 != spec.s):
        raise ValueError(f"slices [{k0}, {k1}) are not whole cell rows of grid {spec.grid}")
    end = off(k1) if k1 % spec.grid == 0 else off(k1 - 1) + spec.s * spec.atlas_dim
    return off(k0), end


class SlabCompute:
    """Interface of the per-rank compute (device kernels in production)."""

    nbins: int

    def artifact_lut(self, top_slab, n_top: int, frac: float) -> torch.Tensor:  # pragma: no cover
        raise NotImplementedError

    def fused(self, slab, lut, z_base: int, full_nz: int, hist, atlases: dict) -> None:  # pragma: no cover
        raise NotImplementedError


class DeviceSlabCompute(SlabCompute):
    """The CUDA kernels behind the C ABI (fused pass per slab)."""

    def __init__(self, dtype, fused_levels: dict):
        from . import device as dev
        self.dev = dev
        self.nbins = dev.NBINS_U8 if dtype == torch.uint8 else dev.NBINS_U16
        self.fused_levels = fused_levels  # level -> AtlasSpec

    def artifact_lut(self, top_slab, n_top, frac, zero_hist=None):
        # one launch: top-slab histogram + LUT (+ zeroing the step's histogram)
        self._lut, _ = self.dev.artifact_lut_fused(top_slab, n_top, frac, zero_hist=zero_hist,
                                                   lut=getattr(self, "_lut", None))
        return self._lut

    def fused(self, slab, lut, z_base, full_nz, hist, atlases):
        self.dev.preview(slab, lut, self.fused_levels, hist=hist, z_base=z_base, full_nz=full_nz,
                         out_tensors=atlases)


@dataclass
class ShardedPreview:
    """One rank's view of a z-slab-sharded preview step."""

    shape: tuple                 # full volume (nz, ny, nx)
    schemes: dict                # s -> AtlasSpec
    level_of: dict               # s -> level (power-of-two ratios only)
    compute: SlabCompute
    rank: int
    world: int
    device: torch.device
    n_top: int = 3
    frac: float = 0.0005
    group: object = None

    def __post_init__(self):
        self.fused_events = None  # optional (start, end) CUDA events around the fused pass (bench)
        nz, ny, nx = self.shape
        for s, l in self.level_of.items():  # scheme s must be exactly level l (pipeline.py:221-222)
            if (nx >> l, ny >> l, nz >> l) != (min(s, nx), min(s, ny), min(s, nz)) or (nx | ny | nz) % (1 << l):
                raise ValueError(f"scheme {s} is not the power-of-two level {l} of {self.shape}")
        self.align = slab_alignment(self.schemes, self.level_of)
        self.z0, self.z1 = slab_bounds(nz, self.world, self.rank, self.align)
        last0, last1 = slab_bounds(nz, self.world, self.world - 1, self.align)
        if last1 - last0 < self.n_top:
            raise ValueError("the last slab must hold the n_top top slices")
        self.hist = torch.zeros(self.compute.nbins, dtype=torch.int64, device=self.device)
        self.atlases = {}
        for s, l in self.level_of.items():
            spec = self.schemes[s]
            self.atlases[l] = torch.zeros((spec.map_count, spec.atlas_dim, spec.atlas_dim), dtype=torch.uint8,
                                          device=self.device)

    def ranges(self, rank: int) -> dict:
        z0, z1 = slab_bounds(self.shape[0], self.world, rank, self.align)
        return {l: atlas_byte_range(self.schemes[s], z0 >> l, z1 >> l) for s, l in self.level_of.items()}

    def step(self, slab: torch.Tensor, gather: bool = True) -> dict:
        """slab: this rank's [z0, z1) voxels on ``device``.  Returns {hist, lut, atlases} (complete on rank 0)."""
        nz = self.shape[0]
        owner = self.world - 1
        if self.world == 1 and isinstance(self.compute, DeviceSlabCompute):
            # a single rank holds the whole volume: LUT step + fused pass in one cooperative launch
            if self.fused_events is not None:
                self.fused_events[0].record()
            _, _, lut, _ = self.compute.dev.preview_step(
                slab, self.compute.fused_levels, self.n_top, self.frac, hist=self.hist,
                lut=getattr(self, "_lut_buf", None), out_tensors=self.atlases)
            if self.fused_events is not None:
                self.fused_events[1].record()
            self._lut_buf = lut
            return {"hist": self.hist, "lut": lut, "atlases": self.atlases}
        zeroed = False
        if self.rank == owner:
            top = slab[slab.shape[0] - self.n_top:]
            if isinstance(self.compute, DeviceSlabCompute):
                lut = self.compute.artifact_lut(top, self.n_top, self.frac, zero_hist=self.hist)
                zeroed = True
            else:
                lut = self.compute.artifact_lut(top, self.n_top, self.frac)
        else:
            lut = torch.empty(self.compute.nbins, dtype=torch.uint8, device=self.device)
        if self.world > 1:
            dist.broadcast(lut, src=owner, group=self.group)
        if not zeroed:
            self.hist.zero_()
        if self.fused_events is not None:
            self.fused_events[0].record()
        self.compute.fused(slab, lut, self.z0, nz, self.hist, self.atlases)
        if self.fused_events is not None:
            self.fused_events[1].record()
        if self.world > 1:
            dist.all_reduce(self.hist, group=self.group)
            if gather:
                self._gather()
        return {"hist": self.hist, "lut": lut, "atlases": self.atlases}

    def _gather(self) -> None:
        if self.rank == 0:
            ops = []
            for r in range(1, self.world):
                for l, (a, b) in self.ranges(r).items():
                    ops.append(dist.P2POp(dist.irecv, self.atlases[l].view(-1)[a:b], r, group=self.group))
            for w in dist.batch_isend_irecv(ops):
                w.wait()
        else:
            ops = [dist.P2POp(dist.isend, self.atlases[l].view(-1)[a:b].contiguous(), 0, group=self.group)
                   for l, (a, b) in self.ranges(self.rank).items()]
            for w in dist.batch_isend_irecv(ops):
                w.wait()
