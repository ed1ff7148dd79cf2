"""Device-resident API: torch CUDA tensors in, torch CUDA tensors out.

Thin wrappers over the C ABI (``_lib``) that allocate outputs with the torch
caching allocator and launch on torch's current stream.  Nothing here
synchronises; nothing here has a CPU path -- a CPU tensor is an error.
This is what ``bench.py`` times (inputs resident in HBM) and what the
host-array drop-ins in ``ops.py`` call after their H2D copy.
"""
from __future__ import annotations

import ctypes as C
import math
from dataclasses import dataclass

import torch

from . import _lib
from ._lib import LevelOut, View

NBINS_U8 = 256
NBINS_U16 = 4096
VMAX_U16 = 4095


def _ptr(t: torch.Tensor | None):
    return C.c_void_p(t.data_ptr()) if t is not None else None


def _stream():
    return C.c_void_p(torch.cuda.current_stream().cuda_stream)


def _check_dev(t: torch.Tensor, dtype, name: str, ndim: int | None = 3):
    if not isinstance(t, torch.Tensor) or not t.is_cuda:
        raise _lib.NativeUnavailable(f"{name}: expected a CUDA tensor (there is no CPU path)")
    if t.dtype != dtype:
        raise TypeError(f"{name}: expected {dtype}, got {t.dtype}")
    if ndim is not None and t.dim() != ndim:
        raise ValueError(f"{name}: expected {ndim}-d tensor, got shape {tuple(t.shape)}")
    if not t.is_contiguous():
        raise ValueError(f"{name}: tensor must be contiguous")


# ---------------------------------------------------------------------------
# histogram / LUT

def hist_u8(vol: torch.Tensor, z_range=None, out: torch.Tensor | None = None) -> torch.Tensor:
    """volume.py:252-262 on the device; returns (or accumulates into) int64[256]."""
    _check_dev(vol, torch.uint8, "hist_u8")
    nz, ny, nx = vol.shape
    z0, z1 = (0, nz) if z_range is None else z_range
    if out is None:
        out = torch.zeros(NBINS_U8, dtype=torch.int64, device=vol.device)
    _lib.call("ctp_hist_u8", _ptr(vol), nz, ny, nx, z0, z1, _ptr(out), _stream())
    return out


def hist_u16(vol: torch.Tensor, z_range=None, nbins: int = NBINS_U16, out: torch.Tensor | None = None):
    _check_dev(vol, torch.uint16, "hist_u16")
    nz, ny, nx = vol.shape
    z0, z1 = (0, nz) if z_range is None else z_range
    if out is None:
        out = torch.zeros(nbins, dtype=torch.int64, device=vol.device)
    _lib.call("ctp_hist_u16", _ptr(vol), nz, ny, nx, z0, z1, nbins, _ptr(out), _stream())
    return out


def cutoff_floor(frac: float, top_size: int) -> int:
    """mask.py:229-230: ``count > frac * top.size`` in float64 <=> count > floor(cutoff)."""
    cutoff = frac * top_size
    if cutoff >= 2.0 ** 63:
        return 2 ** 63 - 1
    return int(math.floor(cutoff))


def lut_from_hist(top_hist: torch.Tensor, top_size: int, frac: float, rescale_vmax: int = 0):
    """mask.py:229-231 + 241-245 on the device: (lut uint8[nbins], flags uint8[nbins])."""
    nbins = top_hist.numel()
    lut = torch.empty(nbins, dtype=torch.uint8, device=top_hist.device)
    flags = torch.empty(nbins, dtype=torch.uint8, device=top_hist.device)
    _lib.call("ctp_lut_build", _ptr(top_hist), nbins, cutoff_floor(frac, top_size), rescale_vmax,
              _ptr(lut), _ptr(flags), _stream())
    return lut, flags


def artifact_lut(vol: torch.Tensor, n_top: int = 3, frac: float = 0.0005):
    """Top-slab histogram (mask.py:227-228) -> LUT; u8 or 12-bit u16 input
    (u16: filter fused with the frozen 16->8 rescale)."""
    nz = vol.shape[0]
    top_size = n_top * vol.shape[1] * vol.shape[2]
    if vol.dtype == torch.uint8:
        th = hist_u8(vol, (nz - n_top, nz))
        return lut_from_hist(th, top_size, frac, 0)
    th = hist_u16(vol, (nz - n_top, nz))
    return lut_from_hist(th, top_size, frac, VMAX_U16)


_WORKSPACES: dict = {}


def _workspace(device) -> torch.Tensor:
    """Zero-initialised uint64[4097] per (device, stream) for ctp_artifact_lut (kept zero by the kernel)."""
    key = (device.index if isinstance(device, torch.device) else device, torch.cuda.current_stream().cuda_stream)
    ws = _WORKSPACES.get(key)
    if ws is None:
        ws = torch.zeros(4097, dtype=torch.int64, device=device)
        _WORKSPACES[key] = ws
    return ws


def artifact_lut_fused(vol: torch.Tensor, n_top: int = 3, frac: float = 0.0005,
                       zero_hist: torch.Tensor | None = None, lut: torch.Tensor | None = None,
                       flags: torch.Tensor | None = None):
    """The artifact-LUT step in ONE launch (top-slab histogram + LUT + flags), also
    zeroing ``zero_hist`` for the fused pass that follows."""
    is16 = vol.dtype == torch.uint16
    _check_dev(vol, torch.uint16 if is16 else torch.uint8, "artifact_lut_fused")
    nz, ny, nx = vol.shape
    nbins = NBINS_U16 if is16 else NBINS_U8
    if lut is None:
        lut = torch.empty(nbins, dtype=torch.uint8, device=vol.device)
    if flags is None:
        flags = torch.empty(nbins, dtype=torch.uint8, device=vol.device)
    _lib.call("ctp_artifact_lut", _ptr(vol), 2 if is16 else 1, nz, ny, nx, n_top,
              cutoff_floor(frac, n_top * ny * nx), VMAX_U16 if is16 else 0, _ptr(lut), _ptr(flags), _ptr(zero_hist),
              _ptr(_workspace(vol.device)), _stream())
    return lut, flags


def lut_apply_u8(src: torch.Tensor, lut: torch.Tensor | None, out: torch.Tensor | None = None,
                 hist: torch.Tensor | None = None) -> torch.Tensor:
    """mask.py:246 on the device (any shape); optionally accumulates the raw histogram."""
    _check_dev(src, torch.uint8, "lut_apply_u8", ndim=None)
    if out is None:
        out = torch.empty_like(src)
    _lib.call("ctp_lut_apply_u8", _ptr(src), _ptr(out), src.numel(), _ptr(lut), _ptr(hist), _stream())
    return out


def lut_apply_u16(src: torch.Tensor, lut: torch.Tensor, out: torch.Tensor | None = None,
                  hist: torch.Tensor | None = None) -> torch.Tensor:
    """Extension: uint16 (12-bit) -> uint8 through the 4096-entry filter o rescale LUT
    (any shape, any row length); optionally accumulates the raw 4096-bin histogram."""
    _check_dev(src, torch.uint16, "lut_apply_u16", ndim=None)
    _check_dev(lut, torch.uint8, "lut_apply_u16 lut", ndim=1)
    if lut.numel() != NBINS_U16:
        raise ValueError("lut_apply_u16: the LUT must have 4096 entries")
    if out is None:
        out = torch.empty(src.shape, dtype=torch.uint8, device=src.device)
    _lib.call("ctp_lut_apply_u16", _ptr(src), _ptr(out), src.numel(), _ptr(lut), _ptr(hist), _stream())
    return out


# ---------------------------------------------------------------------------
# fused pass

@dataclass(frozen=True)
class AtlasSpec:
    """A slicemap scheme as plain ints (slicemap.py:43-61)."""

    s: int
    atlas_dim: int
    grid: int
    map_count: int

    @classmethod
    def of(cls, scheme) -> "AtlasSpec":
        return cls(int(scheme.s), int(scheme.atlas_dim), int(scheme.grid), int(scheme.map_count))


def alloc_level(level_shape, spec, device, zero_pad: bool = True):
    """Allocate the output of one level: dense (nz, ny, nx) or (maps, A, A) atlases."""
    if spec is None or spec == "xyz":
        return torch.empty(level_shape, dtype=torch.uint8, device=device)
    lz, ly, lx = level_shape
    shape = (spec.map_count, spec.atlas_dim, spec.atlas_dim)
    per = spec.grid * spec.grid
    fills_all = (lx == spec.s and ly == spec.s and lz == spec.s and spec.s % per == 0)
    if fills_all or not zero_pad:
        return torch.empty(shape, dtype=torch.uint8, device=device)
    return torch.zeros(shape, dtype=torch.uint8, device=device)


def _out_flags(t) -> int:
    """OUT_PEER for a destination mapped from another GPU (``dist.PeerBuffer``)."""
    return _lib.OUT_PEER if getattr(t, "is_peer", False) else 0


def preview(vol: torch.Tensor, lut: torch.Tensor | None, outputs: dict, hist: torch.Tensor | None = None,
            z_base: int = 0, full_nz: int | None = None, out_tensors: dict | None = None):
    """ONE pass: hist(vol) += ..., f = lut[vol], levels l in ``outputs`` (l -> "xyz" | AtlasSpec).

    Returns {level: tensor}.  For slab-sharded runs pass z_base / full_nz; atlas
    tensors then cover the whole volume (slices outside the slab untouched)."""
    is16 = vol.dtype == torch.uint16
    _check_dev(vol, torch.uint16 if is16 else torch.uint8, "preview")
    nz, ny, nx = vol.shape
    full_nz = full_nz if full_nz is not None else z_base + nz
    nlev = max(outputs) if outputs else 0
    levels = [None] * _lib.MAX_LEVELS
    res = {}
    for l, spec in outputs.items():
        shape = (nz >> l, ny >> l, nx >> l) if (spec is None or spec == "xyz") else (full_nz >> l, ny >> l, nx >> l)
        t = out_tensors.get(l) if out_tensors else None
        if t is None:
            t = alloc_level(shape, spec, vol.device)
        res[l] = t
        if spec is None or spec == "xyz":
            levels[l] = LevelOut(t.data_ptr(), _lib.LAYOUT_XYZ, 0, 0, 0, 0, _out_flags(t))
        else:
            levels[l] = LevelOut(t.data_ptr(), _lib.LAYOUT_ATLAS, spec.s, spec.grid, spec.atlas_dim,
                                 spec.map_count, _out_flags(t))
    arr = _lib.levels_array(levels)
    fn = "ctp_preview_u16" if is16 else "ctp_preview_u8"
    _lib.call(fn, _ptr(vol), nz, ny, nx, z_base, _ptr(lut), nlev, arr, _ptr(hist), _stream())
    return res


# ---------------------------------------------------------------------------
# general resampling / atlases

def downscale(vol: torch.Tensor, target) -> torch.Tensor:
    """volume.py:277-309 (any ratio).  target = (tx, ty, tz)."""
    _check_dev(vol, torch.uint8, "downscale")
    tx, ty, tz = (int(t) for t in target)
    nz, ny, nx = vol.shape
    out = torch.empty((max(tz, 1), max(ty, 1), max(tx, 1)), dtype=torch.uint8, device=vol.device)
    _lib.call("ctp_downscale_u8", _ptr(vol), nz, ny, nx, tz, ty, tx, _ptr(out), _stream())
    return out


def encode_atlas(cube: torch.Tensor, spec: AtlasSpec) -> torch.Tensor:
    """slicemap.py:130-142 packing (+ _pad_to_cube) of an at-most-s^3 volume."""
    _check_dev(cube, torch.uint8, "encode_atlas")
    nz, ny, nx = cube.shape
    out = torch.empty((spec.map_count, spec.atlas_dim, spec.atlas_dim), dtype=torch.uint8, device=cube.device)
    _lib.call("ctp_encode_atlas_u8", _ptr(cube), nz, ny, nx, spec.s, spec.grid, spec.atlas_dim,
              spec.map_count, _ptr(out), _stream())
    return out


def decode_atlas(atlases: torch.Tensor, spec: AtlasSpec) -> torch.Tensor:
    _check_dev(atlases, torch.uint8, "decode_atlas")
    out = torch.empty((spec.s, spec.s, spec.s), dtype=torch.uint8, device=atlases.device)
    _lib.call("ctp_decode_atlas_u8", _ptr(atlases), spec.s, spec.grid, spec.atlas_dim, spec.map_count,
              _ptr(out), _stream())
    return out


# ---------------------------------------------------------------------------
# rendering

_MODES = {"surface": _lib.MODE_SURFACE, "additive": _lib.MODE_ADDITIVE, "mip": _lib.MODE_MIP,
          "alpha": _lib.MODE_ALPHA}


def make_view(p, channels: int = 1, fp32: bool = False) -> View:
    v = View()
    v.azimuth_deg = float(p.azimuth_deg) % 360.0
    v.image_dim = int(p.image_dim)
    v.steps = int(p.steps)
    v.mode = _MODES[p.mode]
    v.threshold = int(p.threshold)
    v.gain = float(p.gain)
    tf = getattr(p, "tf", None)
    if tf is not None:
        for a in range(4):
            for b in range(5):
                v.tf[a][b] = float(tf[a][b])
    v.early_stop = float(getattr(p, "early_stop", 0.99))
    v.channels = channels
    v.fp32 = 1 if fp32 else 0
    return v


def render(vol: torch.Tensor, params_list, channels: int = 1, fp32: bool = False, rows=None,
           out: torch.Tensor | None = None, z_base: int = 0, full_nz: int | None = None,
           out_ptr: int | None = None, out_view_stride: int = 0, out_peer: bool = False) -> torch.Tensor | None:
    """render.py:205-236, batched over views (<= 64 per launch).
    Returns uint8 (n, rows, dim) or (n, rows, dim, 4).

    ``vol`` may be a z-slab (slices [z_base, z_base + vol.shape[0]) of a volume
    ``full_nz`` deep): the geometry is the full volume's and every requested row
    must read only held slices (``dist.row_slices``), else the library refuses.
    ``out_ptr`` / ``out_view_stride``: write view q's band at out_ptr + q * stride
    instead (e.g. into rank 0's full images through a peer mapping, ``out_peer``:
    the kernels then end with a system-scope fence); returns None."""
    _check_dev(vol, torch.uint8, "render")
    snz, ny, nx = vol.shape
    nz = snz if full_nz is None else int(full_nz)
    params_list = list(params_list)
    n = len(params_list)
    dim = int(params_list[0].image_dim)
    r0, r1 = (0, dim) if rows is None else rows
    band = (r1 - r0) * dim * channels
    if out_ptr is None:
        shape = (n, r1 - r0, dim) if channels == 1 else (n, r1 - r0, dim, channels)
        if out is None:
            out = torch.empty(shape, dtype=torch.uint8, device=vol.device)
        base, stride = out.data_ptr(), band
    else:
        base, stride = int(out_ptr), int(out_view_stride or band)
    for b in range(0, n, 64):
        chunk = params_list[b:b + 64]
        arr = (View * len(chunk))(*[make_view(p, channels, fp32) for p in chunk])
        dst = C.c_void_p(base + b * stride)
        if z_base == 0 and snz == nz and stride == band and not out_peer:
            _lib.call("ctp_render_u8", _ptr(vol), nz, ny, nx, arr, len(chunk), r0, r1, dst, _stream())
        else:
            _lib.call("ctp_render_slab_u8", _ptr(vol), z_base, snz, nz, ny, nx, arr, len(chunk), r0, r1, dst,
                      stride, _lib.OUT_PEER if out_peer else 0, _stream())
    return out if out_ptr is None else None


def render_release() -> None:
    """Free the row planes the fp32 MIP/alpha path keeps between calls."""
    _lib.call("ctp_render_release")


def image_hist(imgs: torch.Tensor) -> torch.Tensor:
    """Per-image 256-bin histograms, (n, 256) int64."""
    _check_dev(imgs, torch.uint8, "image_hist", ndim=None)
    n = imgs.shape[0]
    out = torch.zeros((n, 256), dtype=torch.int64, device=imgs.device)
    _lib.call("ctp_image_hist_u8", _ptr(imgs), n, imgs[0].numel(), _ptr(out), _stream())
    return out


# ---------------------------------------------------------------------------
# synthetic inputs

def synth(shape, dtype, seed: int, bg_mean: float, bg_sd: float, shells, speckle_p: float,
          vmax: int | None = None, z_base: int = 0, full_nz: int | None = None, device=None,
          out: torch.Tensor | None = None, speckle_lambda: float = 0.0) -> torch.Tensor:
    nz, ny, nx = shape
    full_nz = full_nz if full_nz is not None else z_base + nz
    elem = 1 if dtype == torch.uint8 else 2
    vmax = vmax if vmax is not None else (255 if elem == 1 else VMAX_U16)
    if out is None:
        out = torch.empty(shape, dtype=dtype, device=device or "cuda")
    arr = (_lib.Shell * max(1, len(shells)))()
    for i, s in enumerate(shells):
        arr[i] = _lib.Shell(*[float(x) for x in s], 0.0)
    _lib.call("ctp_synth_volume", _ptr(out), elem, nz, ny, nx, z_base, full_nz, seed, bg_mean, bg_sd, vmax,
              arr, len(shells), speckle_p, speckle_lambda, _stream())
    return out


def preview_step(vol: torch.Tensor, outputs: dict, n_top: int = 3, frac: float = 0.0005,
                 hist: torch.Tensor | None = None, lut: torch.Tensor | None = None, flags: torch.Tensor | None = None,
                 out_tensors: dict | None = None):
    """The whole step of a full volume in ONE cooperative launch: artifact LUT of the
    top ``n_top`` slices (mask.py:215-231) + the fused pass (``preview``).
    Returns (outputs dict, hist, lut, flags); hist is zeroed by the launch."""
    is16 = vol.dtype == torch.uint16
    _check_dev(vol, torch.uint16 if is16 else torch.uint8, "preview_step")
    nz, ny, nx = vol.shape
    nbins = NBINS_U16 if is16 else NBINS_U8
    if hist is None:
        hist = torch.empty(nbins, dtype=torch.int64, device=vol.device)
    if lut is None:
        lut = torch.empty(nbins, dtype=torch.uint8, device=vol.device)
    if flags is None:
        flags = torch.empty(nbins, dtype=torch.uint8, device=vol.device)
    nlev = max(outputs) if outputs else 0
    levels = [None] * _lib.MAX_LEVELS
    res = {}
    for l, spec in outputs.items():
        shape = (nz >> l, ny >> l, nx >> l)
        t = out_tensors.get(l) if out_tensors else None
        if t is None:
            t = alloc_level(shape, spec, vol.device)
        res[l] = t
        if spec is None or spec == "xyz":
            levels[l] = LevelOut(t.data_ptr(), _lib.LAYOUT_XYZ, 0, 0, 0, 0, 0)
        else:
            levels[l] = LevelOut(t.data_ptr(), _lib.LAYOUT_ATLAS, spec.s, spec.grid, spec.atlas_dim,
                                 spec.map_count, 0)
    fn = "ctp_preview_step_u16" if is16 else "ctp_preview_step_u8"
    _lib.call(fn, _ptr(vol), nz, ny, nx, n_top, cutoff_floor(frac, n_top * ny * nx), nlev,
              _lib.levels_array(levels), _ptr(hist), _ptr(lut), _ptr(flags), _ptr(_workspace(vol.device)),
              _stream())
    return res, hist, lut, flags


def circle_mask(vol: torch.Tensor, cx: float, cy: float, r_eff_sq: float, out: torch.Tensor | None = None):
    """mask.py:208-211 on the device (every slice)."""
    _check_dev(vol, torch.uint8, "circle_mask")
    nz, ny, nx = vol.shape
    if out is None:
        out = torch.empty_like(vol)
    _lib.call("ctp_circle_mask_u8", _ptr(vol), nz, ny, nx, float(cx), float(cy), float(r_eff_sq), _ptr(out),
              _stream())
    return out


def png_filter(images: torch.Tensor, out: torch.Tensor | None = None, filter: int = -1) -> torch.Tensor:
    """PNG-filtered scanlines of (n, H, W) u8 images -> (n, H, W + 1) (ctp_png_filter_u8);
    ``filter`` 0..4 fixes the PNG filter type, -1 picks per row (lowest residual entropy)."""
    _check_dev(images, torch.uint8, "png_filter")
    n, h, w = images.shape
    if out is None:
        out = torch.empty((n, h, w + 1), dtype=torch.uint8, device=images.device)
    _lib.call("ctp_png_filter_u8", _ptr(images), n, h, w, filter, _ptr(out), _stream())
    return out
