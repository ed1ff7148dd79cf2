"""Host-array drop-ins for the reference's hot-path entry points.

Same names, signatures, validation order and error classes as the reference
(ctprev/__init__.py:29-88 re-exports); numpy in, fresh numpy out, with the
H2D / D2H copies inside and the arithmetic in the sm_100a kernels.

    volume_histogram       volume.py:252-262
    Histogram256.of        volume.py:117-122
    artifact_bins          mask.py:215-231
    filter_histogram_bins  mask.py:234-246
    downscale_volume       volume.py:277-309
    encode_slicemaps       slicemap.py:120-142
    decode_slicemaps       slicemap.py:145-155
    render_view            render.py:205-236
    image_entropy          render.py:248-262
    optimal_snapshot       render.py:273-314

plus the fused ``preview_pipeline`` (one HBM pass for hist + filter + levels
+ atlases) and ``render_views`` (batched, incl. the MIP / alpha extensions).
"""
from __future__ import annotations

from dataclasses import dataclass

import numpy as np
import torch

from . import _lib
from . import device as dev
from . import hostio
from .device import AtlasSpec
from .errors import InvalidTarget, RangeOutOfBounds, UnsupportedPixelFormat, DimensionMismatch
from .pipeline import plan_preview, run_preview
from .types import FACTORY, STAGES_DATA, ViewParams, plan_scheme

__all__ = [
    "volume_histogram", "histogram_of", "artifact_bins", "filter_histogram_bins", "downscale_volume",
    "encode_slicemaps", "decode_slicemaps", "render_view", "render_views", "image_entropy",
    "optimal_snapshot", "preview_pipeline", "PreviewResult", "build_data_preview", "to_device", "cuda_device",
]


def cuda_device() -> torch.device:
    if not torch.cuda.is_available():
        raise _lib.NativeUnavailable("no CUDA device visible: the B200 path has no CPU fallback")
    _lib.load()
    return torch.device("cuda", torch.cuda.current_device())


def to_device(arr: np.ndarray) -> torch.Tensor:
    """The device copy of a host array: from the device cache when this frozen array
    was uploaded or produced before (``hostio.DeviceCache``), else a staged H2D copy
    (cached if the array is frozen).  The result is never written by the callers."""
    dev_ = cuda_device()
    t = hostio.CACHE.get(arr, dev_)
    if t is None:
        t = hostio.h2d(arr, dev_)
        hostio.CACHE.put(arr, t)
    return t


def _host(t: torch.Tensor) -> np.ndarray:
    return hostio.d2h(t)


def _host_volume(t: torch.Tensor) -> np.ndarray:
    """Voxels of a result Volume: frozen (as Volume would, volume.py:60-62), device copy kept."""
    return hostio.d2h_frozen(t)


def _voxels(volume) -> np.ndarray:
    return volume.voxels


# ---------------------------------------------------------------------------
# histogram / filter

def histogram_of(values: np.ndarray, cls=None):
    """Histogram256.of (volume.py:117-122) of any uint8 array."""
    cls = cls or FACTORY.Histogram256
    if values.dtype != np.uint8:
        raise UnsupportedPixelFormat(f"expected uint8 values, got {values.dtype}")
    flat = np.ascontiguousarray(values).reshape(1, 1, -1) if values.size else None
    if flat is None:
        return cls(np.zeros(256, dtype=np.int64))
    h = dev.hist_u8(to_device(flat))
    return cls(_host(h))


def volume_histogram(volume, z_range: tuple[int, int] | None = None):
    """volume.py:252-262."""
    vox = _voxels(volume)
    if z_range is None:
        return FACTORY.Histogram256(_host(dev.hist_u8(to_device(vox))))
    z0, z1 = z_range
    if not (0 <= z0 < z1 <= vox.shape[0]):
        raise RangeOutOfBounds(f"z_range {z_range} outside [0, {vox.shape[0]}]")
    # only the slab crosses PCIe
    return FACTORY.Histogram256(_host(dev.hist_u8(to_device(vox[z0:z1]))))


def artifact_bins(volume, n_top: int = 3, frac: float = 0.0005) -> frozenset:
    """mask.py:215-231: the top-slab histogram and the cutoff test on the GPU."""
    vox = _voxels(volume)
    nz = vox.shape[0]
    if not 1 <= n_top <= nz:
        raise RangeOutOfBounds(f"n_top {n_top} outside [1, {nz}]")
    if frac < 0:
        raise RangeOutOfBounds(f"frac {frac} must be non-negative")
    top = to_device(vox[nz - n_top:])
    th = dev.hist_u8(top)
    _, flags = dev.lut_from_hist(th, top.numel(), frac, 0)
    f = _host(flags)
    return frozenset(int(b) for b in np.nonzero(f)[0])


def _lut_from_bins(bins) -> np.ndarray:
    lut = np.arange(256, dtype=np.uint8)  # mask.py:241-245
    for b in bins:
        if not 0 <= int(b) <= 255:
            raise RangeOutOfBounds(f"bin {b} outside [0, 255]")
        lut[int(b)] = 0
    return lut


def filter_histogram_bins(volume, bins):
    """mask.py:234-246: one pass of the LUT kernel."""
    lut = _lut_from_bins(bins)
    vox = _voxels(volume)
    out = dev.lut_apply_u8(to_device(vox), to_device(lut))
    return FACTORY.Volume(_host_volume(out), getattr(volume, "voxel_size_um", None))


# ---------------------------------------------------------------------------
# downscale / slicemaps

def _check_target(target, dims):
    tx, ty, tz = (int(t) for t in target)
    nx, ny, nz = dims
    for t, n, ax in ((tx, nx, "x"), (ty, ny, "y"), (tz, nz, "z")):  # volume.py:287-289
        if not 1 <= t <= n:
            raise InvalidTarget(f"target {ax}={t} outside [1, {n}]")
    return tx, ty, tz


def downscale_volume(volume, target):
    """volume.py:277-309 (identity returns the same voxels, volume.py:290-291)."""
    vox = _voxels(volume)
    nz, ny, nx = vox.shape
    tx, ty, tz = _check_target(target, (nx, ny, nz))
    vs = getattr(volume, "voxel_size_um", None)
    if (tx, ty, tz) == (nx, ny, nz):
        return FACTORY.Volume(vox, vs)
    return FACTORY.Volume(_host_volume(_downscale_dev(to_device(vox), (tx, ty, tz))), vs)


def _downscale_dev(t: torch.Tensor, target) -> torch.Tensor:
    """Power-of-two ratios go through the fused pyramid kernel, others the general one."""
    from .pipeline import level_for_target
    nz, ny, nx = t.shape
    l = level_for_target((nz, ny, nx), target) if nx % 16 == 0 else None
    if l is not None and l >= 1:
        return dev.preview(t, None, {l: "xyz"})[l]
    return dev.downscale(t, target)


def _scheme_levels(t: torch.Tensor, sizes) -> dict:
    """``_scheme_volume(v, s)`` (pipeline.py:215-223) for several schemes at once: every
    level that is a power-of-two ratio of the volume comes out of ONE fused pass (dense,
    each straight from full resolution: exact block sums, volume.py:306-308 rounding);
    identity targets are the volume itself; any other ratio takes the general kernel."""
    from .pipeline import level_for_target
    nz, ny, nx = t.shape
    targets = {s: (min(s, nx), min(s, ny), min(s, nz)) for s in sizes}
    out, fused = {}, {}
    for s, tg in targets.items():
        if tg == (nx, ny, nz):
            out[s] = t
        elif nx % 16 == 0:
            l = level_for_target((nz, ny, nx), tg)
            if l is not None and l >= 1:
                fused[s] = l
    if fused:
        res = dev.preview(t, None, {l: "xyz" for l in set(fused.values())})
        for s, l in fused.items():
            out[s] = res[l]
    for s, tg in targets.items():
        if s not in out:
            out[s] = _downscale_dev(t, tg)
    return out


def encode_slicemaps(volume, scheme):
    """slicemap.py:120-142: downscale to s^3 (errors propagate), then pack."""
    if isinstance(scheme, int):
        scheme = plan_scheme(scheme)
    s = scheme.s
    vox = _voxels(volume)
    nz, ny, nx = vox.shape
    _check_target((s, s, s), (nx, ny, nz))  # slicemap.py:130 -> volume.py:287-289
    spec = AtlasSpec.of(scheme)
    t = to_device(vox)
    cube = t if (nx, ny, nz) == (s, s, s) else _downscale_dev(t, (s, s, s))
    atl = _host(dev.encode_atlas(cube, spec))
    return FACTORY.SlicemapSet(scheme=scheme, atlases=tuple(atl[m] for m in range(spec.map_count)))


def decode_slicemaps(sset):
    """slicemap.py:145-155."""
    sc = sset.scheme
    spec = AtlasSpec.of(sc)
    atl = to_device(np.stack([np.asarray(a) for a in sset.atlases]))
    return FACTORY.Volume(_host_volume(dev.decode_atlas(atl, spec)))


# ---------------------------------------------------------------------------
# rendering

def _view_of(params) -> ViewParams:
    if isinstance(params, ViewParams):
        return params
    return ViewParams(azimuth_deg=params.azimuth_deg, image_dim=params.image_dim, steps=params.steps,
                      mode=params.mode, threshold=params.threshold, gain=params.gain)


def render_view(volume, params) -> np.ndarray:
    """render.py:205-236 (fp64, bit-identical to the numba kernels)."""
    p = _view_of(params)
    img = dev.render(to_device(_voxels(volume)), [p], channels=4 if p.mode == "alpha" else 1)
    return _host(img[0])


def render_views(volume, params_list, channels: int = 1, fp32: bool = False) -> np.ndarray:
    """Batched views of one volume in one launch (per 64 views)."""
    ps = [_view_of(p) for p in params_list]
    return _host(dev.render(to_device(_voxels(volume)), ps, channels=channels, fp32=fp32))


def _entropy_from_counts(counts: np.ndarray, size: int):
    """render.py:256-262 on a histogram (same numpy operations, same bits)."""
    p = counts / size
    nzp = p[p > 0]
    entropy = float(-(nzp * np.log2(nzp)).sum())
    if entropy == 0.0:
        entropy = 0.0
    return entropy, p


def image_entropy(image: np.ndarray):
    """render.py:248-262: histogram on the GPU, the 256-term sum on the host."""
    if image.ndim != 2 or image.dtype != np.uint8:
        raise RangeOutOfBounds("entropy expects a 2-d uint8 image")
    counts = _host(dev.image_hist(to_device(image[None])))[0]
    h, p = _entropy_from_counts(counts, image.size)
    return FACTORY.EntropyResult(entropy=h, probabilities=p)


def optimal_snapshot(volume, n_views: int = 36, params=None):
    """render.py:273-314: all views rendered in one batched launch, per-view
    histograms on the device, the argmax (strict '>', smallest azimuth wins) on the host."""
    if n_views < 1:
        raise RangeOutOfBounds(f"n_views {n_views} must be positive")
    template = _view_of(params) if params is not None else ViewParams()
    return _snapshot_dev(to_device(_voxels(volume)), n_views, template)


def _snapshot_dev(vol_t: torch.Tensor, n_views: int, template):
    step = 360.0 / n_views
    views = [ViewParams(azimuth_deg=k * step, image_dim=template.image_dim, steps=template.steps,
                        mode=template.mode, threshold=template.threshold, gain=template.gain)
             for k in range(n_views)]
    imgs = dev.render(vol_t, views, channels=1)
    counts = _host(dev.image_hist(imgs))
    size = template.image_dim * template.image_dim
    best_k, best_h, per_view = 0, -1.0, []
    for k in range(n_views):
        h, _ = _entropy_from_counts(counts[k], size)
        per_view.append((k * step, h))
        if h > best_h:
            best_k, best_h = k, h
    return FACTORY.SnapshotResult(azimuth_deg=best_k * step, image=_host(imgs[best_k]), entropy=best_h,
                                  per_view=tuple(per_view))


# ---------------------------------------------------------------------------
# fused pipeline

@dataclass
class PreviewResult:
    histogram: np.ndarray          # int64[256] (u8) or int64[4096] (u16)
    bins: frozenset                # artifact bins (incl. 0)
    slicemaps: dict                # s -> SlicemapSet
    levels: dict                   # s -> Volume (only when materialised)
    filtered: object | None        # Volume of the filtered (and rescaled) full-res voxels, if kept


def preview_pipeline(volume, schemes=(512, 256, 128), n_top: int = 3, frac: float = 0.0005,
                     keep_filtered: bool = False) -> PreviewResult:
    """hist + artifact bins + filter (+ 16->8 rescale for uint16) + per-scheme
    levels (direct from the filtered volume) + atlases in one device pass.

    ``volume``: a Volume, or a (nz, ny, nx) uint8 / uint16 (12-bit) array.
    ``schemes``: iterable of ints (plan_scheme) or SlicemapScheme objects."""
    vox = volume if isinstance(volume, np.ndarray) else _voxels(volume)
    if vox.ndim != 3 or min(vox.shape) < 1:
        raise DimensionMismatch("voxels must be a 3-d array (nz, ny, nx)")
    if vox.dtype not in (np.uint8, np.uint16):
        raise UnsupportedPixelFormat(f"voxels must be uint8 or uint16, got {vox.dtype}")
    nz = vox.shape[0]
    if not 1 <= n_top <= nz:
        raise RangeOutOfBounds(f"n_top {n_top} outside [1, {nz}]")
    if frac < 0:
        raise RangeOutOfBounds(f"frac {frac} must be non-negative")
    sch = {}
    for sc in schemes:
        sc = plan_scheme(sc) if isinstance(sc, int) else sc
        sch[sc.s] = sc
    plan = plan_preview(vox.shape, {s: AtlasSpec.of(sc) for s, sc in sch.items()}, keep_filtered=keep_filtered)
    res = run_preview(to_device(vox), plan, n_top, frac)
    slicemaps = {}
    for s, sc in sch.items():
        a = _host(res.atlases[s])
        slicemaps[s] = FACTORY.SlicemapSet(scheme=sc, atlases=tuple(a[m] for m in range(sc.map_count)))
    levels = {s: FACTORY.Volume(_host_volume(t)) for s, t in res.levels.items()}
    flags = _host(res.flags)
    filtered = FACTORY.Volume(_host_volume(res.filtered)) if (keep_filtered and res.filtered is not None) else None
    return PreviewResult(_host(res.hist), frozenset(int(b) for b in np.nonzero(flags)[0]), slicemaps, levels,
                         filtered)


# ---------------------------------------------------------------------------
# preview builders

DATA_SCHEME = 256  # pipeline.py:87


def build_data_preview(volume):
    """pipeline.py:240-257 on the device: the 256-scheme level (_scheme_volume,
    direct from full resolution), its zero-padded atlases, artifact bins from the
    level's top slices, and the filter.  decode -> filter -> encode of the
    reference equals the LUT applied to the atlas bytes themselves (the padding
    is 0 and LUT(0) = 0), so the filter is ONE lut_apply pass over 16 MB."""
    vox = _voxels(volume)
    nz, ny, nx = vox.shape
    s = DATA_SCHEME
    scheme = plan_scheme(s)
    spec = AtlasSpec.of(scheme)
    t = to_device(vox)
    target = (min(s, nx), min(s, ny), min(s, nz))                     # pipeline.py:221-222
    down = t if target == (nx, ny, nz) else _downscale_dev(t, target)
    atl = dev.encode_atlas(down, spec)                                # pipeline.py:249 (+ _pad_to_cube)
    n_top = 3
    dz = down.shape[0]
    if not 1 <= n_top <= dz:                                          # mask.py:223-224
        raise RangeOutOfBounds(f"n_top {n_top} outside [1, {dz}]")
    lut, flags = dev.artifact_lut(down, n_top, 0.0005)                # pipeline.py:250
    fatl = dev.lut_apply_u8(atl, lut)                                 # pipeline.py:251-252
    a = _host(fatl)
    bins = tuple(int(b) for b in np.nonzero(_host(flags))[0])
    sset = FACTORY.SlicemapSet(scheme=scheme, atlases=tuple(a[m] for m in range(spec.map_count)))
    return FACTORY.DataPreview(slicemaps=sset, filtered_bins=bins, stages=STAGES_DATA)


def apply_circle_mask(volume, circle, margin: float = 0.02):
    """mask.py:194-212: zero every voxel outside the circle shrunk by ``margin``."""
    from .errors import CircleOutOfBounds
    vox = _voxels(volume)
    nz, ny, nx = vox.shape
    if not (0 <= circle.cx < nx and 0 <= circle.cy < ny):                   # mask.py:202-205
        raise CircleOutOfBounds(f"center ({circle.cx:.1f}, {circle.cy:.1f}) outside {nx}x{ny} slice")
    if not 0.0 <= margin < 1.0:                                              # mask.py:206-207
        raise RangeOutOfBounds(f"margin {margin} outside [0, 1)")
    r_eff = circle.r * (1.0 - margin)                                        # mask.py:208
    out = dev.circle_mask(to_device(vox), circle.cx, circle.cy, r_eff ** 2)
    return FACTORY.Volume(_host_volume(out), getattr(volume, "voxel_size_um", None))


def _host_helper(module: str, name: str):
    """A host-side reference function that is not on the device path (circle
    Hough transform, Otsu sweep): taken from the installed ctprev."""
    try:
        import importlib
        return getattr(importlib.import_module(f"ctprev.{module}"), name)
    except Exception as e:  # pragma: no cover - depends on the environment
        raise RuntimeError(f"build_interactive_preview: ctprev.{module}.{name} (host, off the device path) is not "
                           f"importable; pass it explicitly") from e


def build_list_preview(volume, n_views: int = 36, full_res: bool = False, detect=None, threshold=None):
    """pipeline.py:157-212 with the volume resident on the device: working copy
    (``_working_copy``, pipeline.py:142-154), container circle found by the HOST
    detector on its top slice and masked on the device, the histogram on the
    device for the host Otsu ``threshold``, then the batched snapshot
    (``optimal_snapshot``); a missing circle or a single-value histogram degrade
    the product as the reference does."""
    from .errors import CircleOutOfBounds, DegenerateHistogram, EmptyVolume, NoCircleFound
    from .types import STAGES_LIST, THUMBNAIL_DIM, WORKING_EDGE
    detect = detect or _host_helper("mask", "detect_container_circle")
    threshold = threshold or _host_helper("threshold", "otsu_threshold")
    vox = _voxels(volume)
    if vox.size == 0:
        raise EmptyVolume("volume has no nonzero voxels")
    t = to_device(vox)
    if int(_host(dev.hist_u8(t))[1:].sum()) == 0:                              # pipeline.py:172-173
        raise EmptyVolume("volume has no nonzero voxels")
    nz, ny, nx = vox.shape
    working = t
    if not full_res and max(nx, ny, nz) > WORKING_EDGE:                       # _working_copy
        k = -(-max(nx, ny, nz) // WORKING_EDGE)
        working = _downscale_dev(t, (-(-nx // k), -(-ny // k), -(-nz // k)))
    warnings_: list[str] = []
    circle = None
    masked = working
    try:
        circle = detect(_host(working[-1]))                                     # top_slice
        wz, wy, wx = working.shape
        if not (0 <= circle.cx < wx and 0 <= circle.cy < wy):                 # mask.py:202-205
            raise CircleOutOfBounds(f"center ({circle.cx:.1f}, {circle.cy:.1f}) outside {wx}x{wy} slice")
        masked = dev.circle_mask(working, circle.cx, circle.cy, (circle.r * (1.0 - 0.02)) ** 2)
    except NoCircleFound:
        warnings_.append("no_container_circle")
    thr, mode = None, "surface"
    try:
        thr = threshold(FACTORY.Histogram256(_host(dev.hist_u8(masked)))).value
    except DegenerateHistogram:
        warnings_.append("degenerate_histogram")
        mode = "additive"
    params = ViewParams(image_dim=THUMBNAIL_DIM, steps=THUMBNAIL_DIM, mode=mode, threshold=thr if thr is not None else 1)
    snap = _snapshot_dev(masked, n_views, params)
    if circle is not None and working is not t:                               # _rescale_circle to raw pixels
        fx, fy = nx / working.shape[2], ny / working.shape[1]
        circle = FACTORY.Circle(circle.cx * fx, circle.cy * fy, circle.r * min(fx, fy), circle.votes)
    return FACTORY.ListPreview(image=snap.image, azimuth_deg=snap.azimuth_deg, entropy=snap.entropy, threshold=thr,
                               circle=circle, mode=mode, warnings=tuple(warnings_), stages=STAGES_LIST)


def build_interactive_preview(volume, detect=None, threshold=None, margin: float = 0.02):
    """pipeline.py:267-309 with the volume resident on the device.

    Each scheme's level comes straight from full resolution (``_scheme_volume``,
    pipeline.py:215-223); the container circle is found once on the 512-scheme
    level's top slice by the HOST detector (``detect``, default
    ctprev.mask.detect_container_circle -- one 2-D slice, scipy) and rescaled per
    scheme (pipeline.py:260-264); then per scheme on the device: circle mask
    (mask.py:194-212), 256-bin histogram, zero-padded atlases (pipeline.py:226-237);
    the host ``threshold`` (default ctprev.threshold.otsu_threshold) reads the
    histogram.  Only the top slice and the 256-bin histograms cross PCIe before
    the atlases come back."""
    from .errors import DegenerateHistogram, NoCircleFound
    from .types import INTERACTIVE_SCHEMES, STAGES_INTERACTIVE
    detect = detect or _host_helper("mask", "detect_container_circle")
    threshold = threshold or _host_helper("threshold", "otsu_threshold")
    vox = _voxels(volume)
    t = to_device(vox)
    downs = _scheme_levels(t, INTERACTIVE_SCHEMES)                               # pipeline.py:215-223, 286
    warnings_: list[str] = []
    circle = None
    try:
        circle = detect(_host(downs[512][-1]))                                   # Volume.top_slice (volume.py:92-95)
    except NoCircleFound:
        warnings_.append("no_container_circle")
    slicemaps, thresholds = {}, {}
    for s in INTERACTIVE_SCHEMES:
        down = downs[s]
        if circle is not None:
            ref = downs[512]
            fx, fy = down.shape[2] / ref.shape[2], down.shape[1] / ref.shape[1]  # _rescale_circle, pipeline.py:260-264
            c = FACTORY.Circle(circle.cx * fx, circle.cy * fy, circle.r * min(fx, fy), circle.votes)
            if not (0 <= c.cx < down.shape[2] and 0 <= c.cy < down.shape[1]):   # mask.py:202-205
                from .errors import CircleOutOfBounds
                raise CircleOutOfBounds(f"center ({c.cx:.1f}, {c.cy:.1f}) outside {down.shape[2]}x{down.shape[1]} slice")
            down = dev.circle_mask(down, c.cx, c.cy, (c.r * (1.0 - margin)) ** 2)
        hist = FACTORY.Histogram256(_host(dev.hist_u8(down)))
        try:
            thresholds[s] = threshold(hist).value
        except DegenerateHistogram:
            if "degenerate_histogram" not in warnings_:
                warnings_.append("degenerate_histogram")
            thresholds[s] = None
        scheme = plan_scheme(s)
        spec = AtlasSpec.of(scheme)
        a = _host(dev.encode_atlas(down, spec))                                  # pipeline.py:298 (+ _pad_to_cube)
        slicemaps[s] = FACTORY.SlicemapSet(scheme=scheme, atlases=tuple(a[m] for m in range(spec.map_count)))
    return FACTORY.InteractivePreview(slicemaps=slicemaps, circle=circle, thresholds=thresholds,
                                      warnings=tuple(warnings_), stages=STAGES_INTERACTIVE)


from .png import save_slicemaps  # noqa: E402,F401  (slicemap.py:158-166, device filter + parallel deflate)


def load_volume(header_path, threads: int = 8):
    """volume.py:229-249 drop-in: the header checked exactly as load_volume does
    (same order, error classes and messages), the raw bytes read by ``threads``
    concurrent preadv calls into one (nz, ny, nx) uint8 array, returned as the
    reference's Volume with its voxel size.  Host I/O only -- the device path
    streams a raw volume with ``ingest.preview_from_raw`` instead."""
    from .ingest import RawReader, read_header
    shape, raw, voxel_size = read_header(header_path)
    arr = np.empty(shape, dtype=np.uint8)
    with RawReader(raw, shape, threads=threads) as rd:
        rd(0, shape[0], arr)
    return FACTORY.Volume(arr, voxel_size)


def load_slice_stack(manifest_path, threads: int = 8):
    """volume.py:167-202 drop-in: the same manifest checks and error classes, the
    slices decoded by a thread pool (Pillow releases the GIL while decoding) into
    one C-contiguous (nz, ny, nx) uint8 array, returned as the reference's Volume.
    Host I/O only -- the device path streams a stack with
    ``ingest.preview_from_slice_stack`` instead of materialising it."""
    from .ingest import SliceStackReader, read_manifest
    paths, shape = read_manifest(manifest_path)
    stack = np.empty(shape, dtype=np.uint8)
    with SliceStackReader(paths, shape, threads=threads) as rd:
        rd(0, shape[0], stack)
    return FACTORY.Volume(stack)
