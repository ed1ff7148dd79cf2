"""Device-side orchestration of the preview data-reduction path.

The composition the BASELINE configs run, equal to the
reference functions called in this order:

    hist  = volume_histogram(v)                                volume.py:252-262
    bins  = artifact_bins(v, n_top, frac)                      mask.py:215-231
    f     = filter_histogram_bins(v, bins)                     mask.py:234-246
    L_s   = _scheme_volume(f, s)  (direct from f, per scheme)  pipeline.py:215-223, 275
    maps  = encode_slicemaps(_pad_to_cube(L_s, s), scheme_s)   slicemap.py:120-142, pipeline.py:226-237

mapped onto at most THREE launches for power-of-two level ratios: the
top-slab histogram (n_top slices), the LUT build, and ONE fused pass that
reads every voxel once and writes the histogram, every level's atlases
and (optionally) the dense levels.  Levels whose ratio is not a power of two
(e.g. 768 -> 512) fall back to the general device downscale + atlas packer.
uint16 (12-bit) volumes use the 4096-bin / filter-o-rescale extension.
"""
from __future__ import annotations

from dataclasses import dataclass, field

import torch

from . import device as dev
from . import trace
from .device import AtlasSpec


def check_top(n_top: int, frac: float, nz: int) -> None:
    """mask.py:223-226: the artifact-bin arguments, checked before any read or launch."""
    from .errors import RangeOutOfBounds
    if not 1 <= n_top <= nz:
        raise RangeOutOfBounds(f"n_top {n_top} outside [1, {nz}]")
    if frac < 0:
        raise RangeOutOfBounds(f"frac {frac} must be non-negative")


def level_for_target(shape, target) -> int | None:
    """Return l if target == shape >> l on every axis with exact division (l <= 4)."""
    nz, ny, nx = shape
    tx, ty, tz = target
    for l in range(0, 5):
        b = 1 << l
        if nx % b or ny % b or nz % b:
            break
        if (nx >> l, ny >> l, nz >> l) == (tx, ty, tz):
            return l
    return None


@dataclass
class PreviewPlan:
    """Which product comes from where."""

    shape: tuple
    schemes: dict                          # s -> AtlasSpec
    fused: dict = field(default_factory=dict)     # level -> AtlasSpec | "xyz"
    scheme_level: dict = field(default_factory=dict)  # s -> fused level (or None)
    general: list = field(default_factory=list)   # s needing the general path
    keep_filtered: bool = False

    @property
    def nlev(self) -> int:
        return max(self.fused) if self.fused else 0


def plan_preview(shape, schemes: dict, keep_filtered: bool = False, keep_levels: bool = False) -> PreviewPlan:
    nz, ny, nx = shape
    plan = PreviewPlan(tuple(shape), dict(schemes), keep_filtered=keep_filtered)
    vec_ok = nx % 16 == 0
    for s, spec in schemes.items():
        target = (min(s, nx), min(s, ny), min(s, nz))  # pipeline.py:221-222
        l = level_for_target(shape, target) if vec_ok else None
        if l is not None and l not in plan.fused and not keep_levels:
            plan.fused[l] = spec
            plan.scheme_level[s] = l
        else:
            plan.general.append(s)
            plan.scheme_level[s] = None
    if plan.general or keep_filtered:
        plan.fused.setdefault(0, "xyz")
        if plan.fused[0] != "xyz":  # level 0 is an atlas AND needed dense: general-pack the atlas
            s0 = [s for s, l in plan.scheme_level.items() if l == 0][0]
            plan.general.append(s0)
            plan.scheme_level[s0] = None
            plan.fused[0] = "xyz"
    return plan


@dataclass
class DevicePreview:
    hist: torch.Tensor                   # int64[256] or [4096]
    lut: torch.Tensor                    # uint8[nbins]
    flags: torch.Tensor                  # uint8[nbins], 1 = artifact bin
    atlases: dict                        # s -> uint8 (maps, A, A)
    levels: dict                         # s -> dense uint8 level (only when materialised)
    filtered: torch.Tensor | None


def run_preview(vol: torch.Tensor, plan: PreviewPlan, n_top: int = 3, frac: float = 0.0005,
                hist: torch.Tensor | None = None) -> DevicePreview:
    """All device work for one volume on the current stream (no sync).  ``hist``
    (optional buffer to reuse) is zeroed and receives the histogram of ``vol``."""
    nbins = dev.NBINS_U8 if vol.dtype == torch.uint8 else dev.NBINS_U16
    if hist is None:
        hist = torch.empty(nbins, dtype=torch.int64, device=vol.device)
    nz, ny, nx = vol.shape
    if nx % (16 // vol.element_size()) and set(plan.fused) == {0}:
        # rows not 16-byte vectorisable: filter (+ rescale) + histogram with the any-size LUT kernels
        with trace.range("preview.lut_apply"):
            lut, flags = dev.artifact_lut_fused(vol, n_top, frac, zero_hist=hist)
            apply = dev.lut_apply_u8 if vol.dtype == torch.uint8 else dev.lut_apply_u16
            outs = {0: apply(vol, lut, hist=hist)}
    else:
        # the whole step (artifact LUT + fused pass) in one cooperative launch
        with trace.range("preview.fused_step"):
            outs, hist, lut, flags = dev.preview_step(vol, plan.fused, n_top, frac, hist=hist)
    atlases, levels = {}, {}
    filtered = outs.get(0) if plan.fused.get(0) == "xyz" else None
    for s, l in plan.scheme_level.items():
        if l is not None:
            atlases[s] = outs[l]
    for s in plan.general:
        spec = plan.schemes[s]
        with trace.range(f"preview.general_level_{s}"):
            lv = dev.downscale(filtered, (min(s, nx), min(s, ny), min(s, nz)))
            levels[s] = lv
            atlases[s] = dev.encode_atlas(lv, spec)
    return DevicePreview(hist, lut, flags, atlases, levels, filtered)


def _cell_row_offset(spec: AtlasSpec, k: int) -> int:
    """Byte offset of the first cell row holding slice k (slicemap.py:79-85 layout)."""
    per = spec.grid * spec.grid
    m, w = divmod(k, per)
    cy = w // spec.grid
    return m * spec.atlas_dim * spec.atlas_dim + cy * spec.s * spec.atlas_dim


class PreviewSession:
    """Host-buffer end-to-end path: pinned host volume in -> pinned host atlases out.

    The volume streams through the GPU in z-chunks: chunk c+1's H2D copy, chunk
    c's fused pass and chunk c-1's atlas D2H overlap on three CUDA streams, so
    the end-to-end time approaches the PCIe transfer time.  Chunk heights are a
    multiple of 2^nlev, so every chunk is a halo-free z-slab (like a multi-GPU
    shard), and the histogram accumulates across chunks.  Only power-of-two
    level ratios stream; plans with general-ratio levels run whole-volume.
    """

    def __init__(self, shape, dtype, schemes: dict, n_top: int = 3, frac: float = 0.0005,
                 chunk_slices: int = 64, ring: int = 3, device=None):
        self.shape = tuple(shape)
        self.dtype = dtype
        check_top(n_top, frac, self.shape[0])
        self.n_top, self.frac = n_top, frac
        self.device = torch.device(device or "cuda")
        self.plan = plan_preview(self.shape, schemes)
        nz, ny, nx = self.shape
        self.streaming = not self.plan.general
        self.nlev = self.plan.nlev
        blk = 1 << self.nlev
        c = max(blk, (chunk_slices // blk) * blk)
        self.chunk = min(c, nz)
        self.nbins = dev.NBINS_U8 if dtype == torch.uint8 else dev.NBINS_U16
        self.hist = torch.zeros(self.nbins, dtype=torch.int64, device=self.device)
        self.atlases = {}
        for s, l in self.plan.scheme_level.items():
            spec = self.plan.schemes[s]
            if l is not None:
                self.atlases[s] = dev.alloc_level((nz >> l, ny >> l, nx >> l), spec, self.device)
        self.host_atlases = {s: torch.empty(t.shape, dtype=torch.uint8, pin_memory=True)
                             for s, t in self.atlases.items()}
        self.host_hist = torch.empty(self.nbins, dtype=torch.int64, pin_memory=True)
        self.host_flags = torch.empty(self.nbins, dtype=torch.uint8, pin_memory=True)
        if self.streaming:
            self.ring = [torch.empty((self.chunk, ny, nx), dtype=dtype, device=self.device) for _ in range(ring)]
            self.top = torch.empty((n_top, ny, nx), dtype=dtype, device=self.device)
        else:
            self.full = torch.empty(self.shape, dtype=dtype, device=self.device)
        self.s_h2d = torch.cuda.Stream(self.device)
        self.s_cmp = torch.cuda.Stream(self.device)
        self.s_d2h = torch.cuda.Stream(self.device)
        self.h2d_bytes = nz * ny * nx * (1 if dtype == torch.uint8 else 2)
        self.d2h_bytes = sum(t.numel() for t in self.host_atlases.values()) + self.nbins * 8 * 1 + self.nbins

    def run(self, host_vol: torch.Tensor) -> dict:
        """host_vol: pinned CPU tensor of ``shape``.  Returns host tensors (pinned, reused)."""
        assert host_vol.shape == self.shape and host_vol.dtype == self.dtype
        if not self.streaming:
            return self._run_whole(host_vol)
        return self._stream(lambda z0, z1, slot: host_vol[z0:z1], lambda slot, evt: None)

    def run_reader(self, read) -> dict:
        """Volume from a reader instead of host memory: ``read(z0, z1, out)`` fills the
        pinned numpy array ``out`` (z1 - z0, ny, nx) with slices [z0, z1) (e.g. straight
        from a .raw file).  Reading chunk c+1 overlaps chunk c's copy and pass; only
        ``ring`` chunks of host memory are ever held."""
        nz, ny, nx = self.shape
        if not self.streaming:
            full = torch.empty(self.shape, dtype=self.dtype, pin_memory=True)
            read(0, nz, full.numpy())
            return self._run_whole(full)
        if not hasattr(self, "host_ring"):
            self.host_ring = [torch.empty((self.chunk, ny, nx), dtype=self.dtype, pin_memory=True)
                              for _ in range(len(self.ring))]
            self.host_top = torch.empty((self.n_top, ny, nx), dtype=self.dtype, pin_memory=True)
        freed = [None] * len(self.host_ring)
        top_freed = getattr(self, "_top_freed", None)
        if top_freed is not None:
            top_freed.synchronize()  # the previous run's top-slab H2D is done

        def src(z0, z1, slot):
            if slot < 0:  # the top slab
                read(z0, z1, self.host_top.numpy())
                return self.host_top
            if freed[slot] is not None:
                freed[slot].synchronize()  # the previous H2D out of this host slot is done
            v = self.host_ring[slot][: z1 - z0]
            read(z0, z1, v.numpy())
            return v

        def done(slot, evt):
            if slot >= 0:
                freed[slot] = evt
            else:
                self._top_freed = evt

        return self._stream(src, done)

    def _stream(self, src, h2d_done) -> dict:
        nz, ny, nx = self.shape
        cur = torch.cuda.current_stream(self.device)
        for s in (self.s_h2d, self.s_cmp, self.s_d2h):
            s.wait_stream(cur)
        with torch.cuda.stream(self.s_h2d):
            top_src = src(nz - self.n_top, nz, -1)
            self.top.copy_(top_src, non_blocking=True)
            top_ready = torch.cuda.Event()
            top_ready.record(self.s_h2d)
        h2d_done(-1, top_ready)
        with torch.cuda.stream(self.s_cmp):
            self.s_cmp.wait_event(top_ready)
            lut, flags = dev.artifact_lut_fused(self.top, self.n_top, self.frac, zero_hist=self.hist)
        n_chunks = (nz + self.chunk - 1) // self.chunk
        free = [None] * len(self.ring)
        for c in range(n_chunks):
            z0 = c * self.chunk
            z1 = min(nz, z0 + self.chunk)
            slot = c % len(self.ring)
            buf = self.ring[slot][: z1 - z0]
            host = src(z0, z1, slot)
            with torch.cuda.stream(self.s_h2d):
                if free[slot] is not None:
                    self.s_h2d.wait_event(free[slot])
                buf.copy_(host, non_blocking=True)
                landed = torch.cuda.Event()
                landed.record(self.s_h2d)
            h2d_done(slot, landed)
            with torch.cuda.stream(self.s_cmp):
                self.s_cmp.wait_event(landed)
                outs = {l: self.atlases[s] for s, l in self.plan.scheme_level.items()}
                dev.preview(buf, lut, self.plan.fused, hist=self.hist, z_base=z0, full_nz=nz, out_tensors=outs)
                done = torch.cuda.Event()
                done.record(self.s_cmp)
                free[slot] = done
            with torch.cuda.stream(self.s_d2h):
                self.s_d2h.wait_event(done)
                last = c == n_chunks - 1
                for s, l in self.plan.scheme_level.items():
                    spec = self.plan.schemes[s]
                    k0, k1 = z0 >> l, z1 >> l
                    a = _cell_row_offset(spec, k0)
                    b = self.atlases[s].numel() if last else min(
                        self.atlases[s].numel(), _cell_row_offset(spec, k1 - 1) + spec.s * spec.atlas_dim)
                    if b > a:
                        self.host_atlases[s].view(-1)[a:b].copy_(self.atlases[s].view(-1)[a:b], non_blocking=True)
        with torch.cuda.stream(self.s_d2h):
            self.s_d2h.wait_stream(self.s_cmp)
            self.host_hist.copy_(self.hist, non_blocking=True)
            self.host_flags.copy_(flags, non_blocking=True)
        self.s_d2h.synchronize()
        return {"hist": self.host_hist, "flags": self.host_flags, "atlases": self.host_atlases}

    def _run_whole(self, host_vol):
        with torch.cuda.stream(self.s_cmp):
            self.full.copy_(host_vol, non_blocking=True)
            res = run_preview(self.full, self.plan, self.n_top, self.frac)
            for s, t in res.atlases.items():
                if s not in self.host_atlases:
                    self.host_atlases[s] = torch.empty(t.shape, dtype=torch.uint8, pin_memory=True)
                self.host_atlases[s].copy_(t, non_blocking=True)
            self.host_hist.copy_(res.hist, non_blocking=True)
            self.host_flags.copy_(res.flags, non_blocking=True)
        self.s_cmp.synchronize()
        return {"hist": self.host_hist, "flags": self.host_flags, "atlases": self.host_atlases}
