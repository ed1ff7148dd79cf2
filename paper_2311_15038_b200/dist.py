"""z-slab sharding of one volume across the GPUs of a node:
the preview step (``ShardedPreview``) and sort-last rendering (``ShardedRender``).

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

import math
from dataclasses import dataclass

import numpy as np
import torch
import torch.distributed as dist

from . import trace
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


class PeerBuffer:
    """A device buffer of another process of the node, mapped through CUDA IPC
    (``ctp_ipc_import``); usable wherever the kernels take a destination pointer."""

    is_peer = True  # kernels storing here end with a system-scope fence (CTP_OUT_PEER)

    def __init__(self, handle: bytes, offset: int, shape, dtype=torch.uint8):
        import ctypes as C
        from . import _lib
        self._lib = _lib
        self.offset = int(offset)
        self.shape = tuple(shape)
        self.dtype = dtype
        p = C.c_void_p()
        _lib.call("ctp_ipc_import", C.create_string_buffer(bytes(handle), len(handle)), self.offset, C.byref(p))
        self.ptr = int(p.value)

    def data_ptr(self) -> int:
        return self.ptr

    def numel(self) -> int:
        return int(np.prod(self.shape))

    def close(self) -> None:
        import ctypes as C
        if self.ptr:
            self._lib.call("ctp_ipc_close", C.c_void_p(self.ptr), self.offset)
            self.ptr = 0


def export_buffer(t: torch.Tensor) -> tuple[bytes, int]:
    """(IPC handle, offset) of a CUDA tensor's storage for ``PeerBuffer`` in another process."""
    import ctypes as C
    from . import _lib
    h = C.create_string_buffer(64)
    off = C.c_int64()
    _lib.call("ctp_ipc_export", C.c_void_p(t.data_ptr()), h, C.byref(off))
    return h.raw, int(off.value)


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
    peer_atlases: bool = False   # ranks > 0 store straight into rank 0's atlases (CUDA IPC over NVLink)

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
        self.peer = self.peer_atlases and self.world > 1
        for s, l in self.level_of.items():
            spec = self.schemes[s]
            if self.peer and self.rank != 0:
                continue
            self.atlases[l] = torch.zeros((spec.map_count, spec.atlas_dim, spec.atlas_dim), dtype=torch.uint8,
                                          device=self.device)
        if self.peer:
            # the gather fused into the pass: rank 0 exports its atlases, every other rank maps
            # them and its kernel stores its slab's cell rows there directly (no gather step)
            torch.cuda.synchronize(self.device)
            handles = [{l: export_buffer(t) for l, t in self.atlases.items()} if self.rank == 0 else None]
            dist.broadcast_object_list(handles, src=0, group=self.group)
            if self.rank != 0:
                for s, l in self.level_of.items():
                    spec = self.schemes[s]
                    h, off = handles[0][l]
                    self.atlases[l] = PeerBuffer(h, off, (spec.map_count, spec.atlas_dim, spec.atlas_dim))

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
            lut = torch.zeros(self.compute.nbins, dtype=torch.uint8, device=self.device)
        if self.world > 1:
            with trace.range("sharded.lut_exchange"):
                if self.peer:
                    # peer mode: every rank's pass stores into rank 0's atlases, which are reused by
                    # every step -- so the LUT is distributed by an all-reduce (MAX over the owner's
                    # LUT and zeros) instead of a broadcast: no rank can start its pass before rank 0
                    # has entered this step, i.e. finished with the previous step's atlases
                    dist.all_reduce(lut, op=dist.ReduceOp.MAX, group=self.group)
                else:
                    dist.broadcast(lut, src=owner, group=self.group)
        if not zeroed:
            self.hist.zero_()
        if self.fused_events is not None:
            self.fused_events[0].record()
        with trace.range("sharded.fused_pass"):
            self.compute.fused(slab, lut, self.z0, nz, self.hist, self.atlases)
        if self.fused_events is not None:
            self.fused_events[1].record()
        if self.world > 1:
            # stream-ordered after every rank's pass: when rank 0's all-reduce completes, every
            # rank's kernel -- and, in peer mode, its stores into rank 0's atlases -- is done
            with trace.range("sharded.hist_allreduce"):
                dist.all_reduce(self.hist, group=self.group)
            if gather and not self.peer:
                with trace.range("sharded.atlas_gather"):
                    self._gather()
        return {"hist": self.hist, "lut": lut, "atlases": self.atlases}

    def close(self) -> None:
        for t in self.atlases.values():
            if isinstance(t, PeerBuffer):
                t.close()

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


# ---------------------------------------------------------------------------
# Sort-last rendering of a z-slab-sharded volume.
#
# The reference camera has elevation 0 (render.py:131-140): pixel row j's rays
# all lie in the plane z = wy(j), so row j samples only the slices around
# uz(j).  The per-slab partial images of a sort-last renderer are therefore
# disjoint row bands and the composite is a row-band gather: rank r renders the
# rows whose clamped floor(uz) lies in its core slices [z0, z1), from its core
# plus a halo of the slices those rows read (the trilinear pair, the surface
# gradient's +-1 and one slice of margin -- ``row_slices``, the same rule the
# library enforces in ctp_render_slab_u8).

def render_geometry(shape, image_dim: int) -> tuple[float, float, float]:
    """(big_r, px_size, n_max) of render.py:212-223 for a (nz, ny, nx) volume."""
    nz, ny, nx = shape
    n_max = float(max(nz, ny, nx))
    hx, hy, hz = nx / (2.0 * n_max), ny / (2.0 * n_max), nz / (2.0 * n_max)
    big_r = math.sqrt(hx * hx + hy * hy + hz * hz)
    return big_r, 2.0 * big_r / image_dim, n_max


def row_uz(shape, image_dim: int) -> np.ndarray:
    """Voxel-space z of every image row (render.py:131-137, 114-118), fp64 in the kernel's order."""
    nz = shape[0]
    big_r, px, n_max = render_geometry(shape, image_dim)
    j = np.arange(image_dim, dtype=np.float64)
    return (big_r - (j + 0.5) * px) * n_max + (nz - 1) * 0.5


def row_slices(shape, image_dim: int) -> tuple[np.ndarray, np.ndarray]:
    """Per row, the inclusive slice window [lo, hi] it reads (lo > hi: none)."""
    nz = shape[0]
    uz = row_uz(shape, image_dim)
    inside = (uz >= -0.51) & (uz <= nz - 0.49)
    zf = np.floor(uz).astype(np.int64)
    lo = np.where(inside, np.clip(zf - 2, 0, nz - 1), 1)
    hi = np.where(inside, np.clip(zf + 3, 0, nz - 1), 0)
    return lo, hi


def row_band(shape, image_dim: int, z0: int, z1: int) -> tuple[int, int]:
    """Rows whose clamped floor(uz) lies in [z0, z1): contiguous, since uz falls with j."""
    nz = shape[0]
    owner = np.clip(np.floor(row_uz(shape, image_dim)), 0, nz - 1).astype(np.int64)
    rows = np.flatnonzero((owner >= z0) & (owner < z1))
    if rows.size == 0:
        return 0, 0
    r0, r1 = int(rows[0]), int(rows[-1]) + 1
    assert rows.size == r1 - r0
    return r0, r1


def held_slices(shape, image_dim: int, z0: int, z1: int) -> tuple[int, int]:
    """Slices a rank must hold to render its row band: its core plus the halo the band reads."""
    r0, r1 = row_band(shape, image_dim, z0, z1)
    lo, hi = row_slices(shape, image_dim)
    h0, h1 = z0, z1
    for j in range(r0, r1):
        if lo[j] <= hi[j]:
            h0, h1 = min(h0, int(lo[j])), max(h1, int(hi[j]) + 1)
    return h0, h1


class RenderCompute:
    """Interface of the per-rank renderer (device kernels in production)."""

    def render(self, slab, z_base: int, full_nz: int, views, rows, channels: int, fp32: bool):  # pragma: no cover
        raise NotImplementedError


class DeviceRenderCompute(RenderCompute):
    def __init__(self):
        from . import device as dev
        self.dev = dev

    def render(self, slab, z_base, full_nz, views, rows, channels, fp32):
        return self.dev.render(slab, views, channels=channels, fp32=fp32, rows=rows, z_base=z_base, full_nz=full_nz)

    def render_into(self, slab, z_base, full_nz, views, rows, channels, fp32, out_ptr: int, view_stride: int,
                    peer: bool = True):
        """Write each view's row band straight into full images at ``out_ptr`` (row 0 of view 0)."""
        d = int(views[0].image_dim)
        self.dev.render(slab, views, channels=channels, fp32=fp32, rows=rows, z_base=z_base, full_nz=full_nz,
                        out_ptr=out_ptr + rows[0] * d * channels, out_view_stride=view_stride, out_peer=peer)


@dataclass
class ShardedRender:
    """One rank's share of a batch of views, volume z-slab-sharded (sort-last) or
    replicated (image rows split evenly).  ``render`` returns the full images on
    rank 0 (``gather``) and this rank's row band everywhere else."""

    shape: tuple                 # full volume (nz, ny, nx)
    image_dim: int
    compute: RenderCompute
    rank: int
    world: int
    device: torch.device
    replicated: bool = False
    align: int = 1               # core slab alignment (the preview's, to share its slabs)
    group: object = None
    peer_images: bool = False    # ranks render their bands straight into rank 0's images (CUDA IPC)

    def __post_init__(self):
        nz = self.shape[0]
        self._peer_out = {}
        self.cores, self.bands, self.held = [], [], []
        for r in range(self.world):
            if self.replicated:
                d = self.image_dim
                self.cores.append((0, nz))
                self.bands.append((r * d // self.world, (r + 1) * d // self.world))
                self.held.append((0, nz))
            else:
                z0, z1 = slab_bounds(nz, self.world, r, self.align)
                self.cores.append((z0, z1))
                self.bands.append(row_band(self.shape, self.image_dim, z0, z1))
                self.held.append(held_slices(self.shape, self.image_dim, z0, z1))
        cover = sorted(b for b in self.bands if b[1] > b[0])
        if cover[0][0] != 0 or cover[-1][1] != self.image_dim or any(p[1] != q[0] for p, q in zip(cover, cover[1:])):
            raise AssertionError(f"row bands {self.bands} do not partition [0, {self.image_dim})")
        self.z0, self.z1 = self.cores[self.rank]
        self.h0, self.h1 = self.held[self.rank]
        self.r0, self.r1 = self.bands[self.rank]

    def _peer_images(self, n: int, channels: int):
        """Rank 0's (n, dim, dim[, ch]) image buffer, mapped on every rank (set up once per shape)."""
        key = (n, channels)
        if key not in self._peer_out:
            d = self.image_dim
            shape = (n, d, d) if channels == 1 else (n, d, d, channels)
            buf = torch.empty(shape, dtype=torch.uint8, device=self.device) if self.rank == 0 else None
            handle = [export_buffer(buf) if self.rank == 0 else None]
            dist.broadcast_object_list(handle, src=0, group=self.group)
            self._peer_out[key] = buf if self.rank == 0 else PeerBuffer(handle[0][0], handle[0][1], shape)
        return self._peer_out[key]

    def close(self) -> None:
        for t in self._peer_out.values():
            if isinstance(t, PeerBuffer):
                t.close()
        self._peer_out.clear()

    def render(self, local: torch.Tensor, views, channels: int = 1, fp32: bool = False, gather: bool = True):
        """local: slices [h0, h1) of the volume on ``device`` (the whole volume when replicated)."""
        views = list(views)
        n, d = len(views), self.image_dim
        tail = (d,) if channels == 1 else (d, channels)
        if self.peer_images and self.world > 1 and gather:
            # sort-last composite fused into the render: every rank's kernel stores its row band
            # into rank 0's images over NVLink; the all-reduce after it (stream order) completes it
            out = self._peer_images(n, channels)
            # rank 0's images are reused by every call: no rank may store this batch's band
            # before rank 0 has entered the call, i.e. finished with the previous batch
            # (its host or stream-ordered consumers come before this call)
            ready = torch.ones(1, dtype=torch.int32, device=self.device)
            dist.all_reduce(ready, group=self.group)
            if self.r1 > self.r0:
                self.compute.render_into(local, self.h0, self.shape[0], views, (self.r0, self.r1), channels, fp32,
                                         out.data_ptr(), d * d * channels, peer=self.rank != 0)
            flag = torch.ones(1, dtype=torch.int32, device=self.device)
            dist.all_reduce(flag, group=self.group)
            return out if self.rank == 0 else None
        band = None
        if self.r1 > self.r0:
            band = self.compute.render(local, self.h0, self.shape[0], views, (self.r0, self.r1), channels, fp32)
        if self.world == 1 or not gather:
            return band
        if self.rank == 0:
            out = torch.empty((n, d) + tail, dtype=torch.uint8, device=self.device)
            if band is not None:
                out[:, self.r0:self.r1] = band
            bufs, ops = {}, []
            for r in range(1, self.world):
                a, b = self.bands[r]
                if b > a:
                    bufs[r] = torch.empty((n, b - a) + tail, dtype=torch.uint8, device=self.device)
                    ops.append(dist.P2POp(dist.irecv, bufs[r], r, group=self.group))
            if ops:
                for w in dist.batch_isend_irecv(ops):
                    w.wait()
            for r, t in bufs.items():
                a, b = self.bands[r]
                out[:, a:b] = t
            return out
        if band is not None:
            for w in dist.batch_isend_irecv([dist.P2POp(dist.isend, band.contiguous(), 0, group=self.group)]):
                w.wait()
        return band
