"""Mirrors of the reference's value types, with the same validation.

  Volume          ctprev/volume.py:38-95
  Histogram256    ctprev/volume.py:98-122
  SlicemapScheme  ctprev/slicemap.py:43-68
  SlicemapSet     ctprev/slicemap.py:88-117
  ViewParams      ctprev/render.py:39-65 (+ the MIP / alpha extension modes)
  EntropyResult   ctprev/render.py:239-245
  SnapshotResult  ctprev/render.py:265-270
  Circle          ctprev/mask.py:35-56
  DataPreview / InteractivePreview   ctprev/pipeline.py:116-133

The drop-in functions accept the reference's own objects (duck typed on the
same attributes) and build their results through ``FACTORY``, which
``install()`` points at the reference classes so callers inside ctprev get
exactly the types they check for (slicemap.py:95-110).
"""
from __future__ import annotations

from dataclasses import dataclass, field

import numpy as np

from .errors import (CircleOutOfBounds, DimensionMismatch, ManifestMismatch, RangeOutOfBounds, UnsupportedPixelFormat,
                     UnsupportedScheme, IndexOutOfRange)

SURFACE = "surface"
ADDITIVE = "additive"
MIP = "mip"          # extension
ALPHA = "alpha"      # extension
_PLANNED: dict[int, int] = {128: 1024, 256: 2048, 512: 4096}  # slicemap.py:40


@dataclass(eq=False)
class Volume:
    """Dense 8-bit grid, (nz, ny, nx) C-contiguous, frozen (volume.py:38-62)."""

    voxels: np.ndarray
    voxel_size_um: float | None = None

    def __post_init__(self) -> None:
        v = self.voxels
        if not isinstance(v, np.ndarray) or v.ndim != 3:
            raise DimensionMismatch("voxels must be a 3-d array (nz, ny, nx)")
        if v.dtype != np.uint8:
            raise UnsupportedPixelFormat(f"voxels must be uint8, got {v.dtype}")
        if min(v.shape) < 1:
            raise DimensionMismatch(f"degenerate volume shape {v.shape}")
        v = np.ascontiguousarray(v)
        v.setflags(write=False)
        self.voxels = v

    @property
    def dims(self) -> tuple[int, int, int]:
        nz, ny, nx = self.voxels.shape
        return nx, ny, nz

    @property
    def nx(self) -> int:
        return self.voxels.shape[2]

    @property
    def ny(self) -> int:
        return self.voxels.shape[1]

    @property
    def nz(self) -> int:
        return self.voxels.shape[0]

    @property
    def raw_bytes(self) -> int:
        return self.voxels.size

    def slice_xy(self, z: int) -> np.ndarray:
        if not 0 <= z < self.nz:
            raise RangeOutOfBounds(f"z={z} outside [0, {self.nz})")
        return self.voxels[z]

    def top_slice(self) -> np.ndarray:
        return self.voxels[-1]


@dataclass(eq=False)
class Histogram256:
    """Counts over 256 bins (volume.py:98-122)."""

    bins: np.ndarray

    def __post_init__(self) -> None:
        b = np.asarray(self.bins, dtype=np.int64)
        if b.shape != (256,):
            raise DimensionMismatch(f"histogram must have 256 bins, got {b.shape}")
        if (b < 0).any():
            raise RangeOutOfBounds("histogram counts must be non-negative")
        b.setflags(write=False)
        self.bins = b

    @property
    def total(self) -> int:
        return int(self.bins.sum())

    @classmethod
    def of(cls, values: np.ndarray) -> "Histogram256":
        """Histogram of any uint8 array -- computed on the GPU."""
        from .ops import histogram_of
        return histogram_of(values, cls)


@dataclass(frozen=True)
class SlicemapScheme:
    """Atlas layout (slicemap.py:43-68)."""

    s: int
    atlas_dim: int
    grid: int
    map_count: int

    def __post_init__(self) -> None:
        if self.grid * self.s != self.atlas_dim:
            raise UnsupportedScheme(f"grid {self.grid} x slice {self.s} != atlas {self.atlas_dim}")
        per_map = self.grid * self.grid
        if self.map_count != -(-self.s // per_map):
            raise UnsupportedScheme(f"{self.map_count} maps cannot hold {self.s} slices at {per_map}/map")

    @property
    def slices_per_map(self) -> int:
        return self.grid * self.grid

    def atlas_names(self, ext: str = "png") -> list[str]:
        return [f"sm_{self.s}_{i}.{ext}" for i in range(self.map_count)]


def plan_scheme(s: int) -> SlicemapScheme:
    """slicemap.py:71-76."""
    if s not in _PLANNED:
        raise UnsupportedScheme(f"no planned layout for s={s}, expected one of {sorted(_PLANNED)}")
    return FACTORY.SlicemapScheme(s=s, atlas_dim=_PLANNED[s], grid=8, map_count=-(-s // 64))


def slice_cell(index: int, scheme) -> tuple[int, int, int]:
    """slicemap.py:79-85."""
    if not 0 <= index < scheme.s:
        raise IndexOutOfRange(f"slice index {index} outside [0, {scheme.s})")
    m, within = divmod(index, scheme.grid * scheme.grid)
    cell_y, cell_x = divmod(within, scheme.grid)
    return m, cell_x, cell_y


@dataclass(eq=False)
class SlicemapSet:
    """Encoded atlases plus their layout (slicemap.py:88-117)."""

    scheme: SlicemapScheme
    atlases: tuple

    def __post_init__(self) -> None:
        if len(self.atlases) != self.scheme.map_count:
            raise ManifestMismatch(f"{len(self.atlases)} atlases for a {self.scheme.map_count}-map scheme")
        frozen = []
        for i, a in enumerate(self.atlases):
            if a.shape != (self.scheme.atlas_dim, self.scheme.atlas_dim) or a.dtype != np.uint8:
                raise ManifestMismatch(
                    f"atlas {i}: shape {a.shape} dtype {a.dtype}, expected "
                    f"({self.scheme.atlas_dim}, {self.scheme.atlas_dim}) uint8")
            a = np.ascontiguousarray(a)
            a.setflags(write=False)
            frozen.append(a)
        self.atlases = tuple(frozen)

    def manifest(self) -> dict:
        sc = self.scheme
        return {"scheme": {"s": sc.s, "atlas": sc.atlas_dim, "grid": sc.grid, "maps": sc.map_count},
                "atlases": sc.atlas_names()}


def _default_tf() -> tuple:
    # (value, r, g, b, a): transparent air, soft tissue, dense material
    return ((0.0, 0.0, 0.0, 0.0, 0.0), (60.0, 0.8, 0.3, 0.2, 0.0),
            (140.0, 1.0, 0.8, 0.6, 0.05), (255.0, 1.0, 1.0, 1.0, 0.3))


@dataclass(frozen=True)
class ViewParams:
    """render.py:39-65, plus the extension modes ``mip`` and ``alpha``
    (1D RGBA transfer function with 4 control points, early termination)."""

    azimuth_deg: float = 0.0
    image_dim: int = 512
    steps: int = 512
    mode: str = SURFACE
    threshold: int = 1
    gain: float = 4.0
    tf: tuple = field(default_factory=_default_tf)
    early_stop: float = 0.99

    def __post_init__(self) -> None:
        object.__setattr__(self, "azimuth_deg", float(self.azimuth_deg) % 360.0)
        if self.image_dim < 16:
            raise RangeOutOfBounds(f"image_dim {self.image_dim} below minimum 16")
        if self.steps < 32:
            raise RangeOutOfBounds(f"steps {self.steps} below minimum 32")
        if self.mode not in (SURFACE, ADDITIVE, MIP, ALPHA):
            raise RangeOutOfBounds(f"mode {self.mode!r} not one of ({SURFACE!r}, {ADDITIVE!r}, {MIP!r}, {ALPHA!r})")
        if not 0 <= self.threshold <= 255:
            raise RangeOutOfBounds(f"threshold {self.threshold} outside [0, 255]")
        if self.gain <= 0:
            raise RangeOutOfBounds(f"gain {self.gain} must be positive")
        tf = np.asarray(self.tf, dtype=np.float64)
        if tf.shape != (4, 5) or not np.all(np.diff(tf[:, 0]) > 0):
            raise RangeOutOfBounds("tf must be 4 control points (value, r, g, b, a) with ascending values")
        if not (0.0 < self.early_stop <= 1.0):
            raise RangeOutOfBounds(f"early_stop {self.early_stop} outside (0, 1]")


@dataclass(frozen=True)
class EntropyResult:
    entropy: float
    probabilities: np.ndarray
    bins: int = 256


@dataclass(frozen=True)
class SnapshotResult:
    azimuth_deg: float
    image: np.ndarray
    entropy: float
    per_view: tuple


STAGES_DATA = ("slicemaps_conversion", "histogram_filtering")  # pipeline.py:82


@dataclass(frozen=True)
class DataPreview:
    """pipeline.py:116-122."""

    slicemaps: SlicemapSet
    filtered_bins: tuple
    stages: tuple


STAGES_LIST = ("3d_conversion", "thresholding_container_removal", "server_side_rendering")  # pipeline.py:81
STAGES_INTERACTIVE = ("slicemaps_conversion", "thresholding_container_removal")  # pipeline.py:83
THUMBNAIL_DIM = 512                                                                    # pipeline.py:88
WORKING_EDGE = 256                                                                     # pipeline.py:89


@dataclass(frozen=True)
class ListPreview:
    """pipeline.py:92-113."""

    image: np.ndarray
    azimuth_deg: float
    entropy: float
    threshold: object
    circle: object
    mode: str
    warnings: tuple
    stages: tuple

    def sidecar(self) -> dict:
        c = self.circle
        return {"azimuth": self.azimuth_deg, "entropy": self.entropy, "threshold": self.threshold,
                "circle": None if c is None else {"cx": c.cx, "cy": c.cy, "r": c.r, "votes": c.votes},
                "mode": self.mode, "warnings": list(self.warnings)}
INTERACTIVE_SCHEMES = (128, 256, 512)                                          # pipeline.py:85


@dataclass(frozen=True)
class InteractivePreview:
    """pipeline.py:125-133."""

    slicemaps: dict
    circle: object
    thresholds: dict
    warnings: tuple
    stages: tuple


@dataclass(frozen=True)
class Circle:
    """mask.py:35-56: a container circle in pixel coordinates."""

    cx: float
    cy: float
    r: float
    votes: float = 1.0

    def __post_init__(self) -> None:
        if self.r <= 0:
            raise CircleOutOfBounds(f"radius {self.r} must be positive")
        if not 0.0 <= self.votes <= 1.0:
            raise RangeOutOfBounds(f"votes {self.votes} outside [0, 1]")

    def scaled(self, factor: float) -> "Circle":
        return type(self)(self.cx * factor, self.cy * factor, self.r * factor, self.votes)


class _Factory:
    """Where result objects come from (switched by ``install()``)."""

    def __init__(self) -> None:
        self.reset()

    def reset(self) -> None:
        self.Volume = Volume
        self.Histogram256 = Histogram256
        self.SlicemapScheme = SlicemapScheme
        self.SlicemapSet = SlicemapSet
        self.EntropyResult = EntropyResult
        self.SnapshotResult = SnapshotResult
        self.DataPreview = DataPreview
        self.InteractivePreview = InteractivePreview
        self.ListPreview = ListPreview
        self.Circle = Circle


FACTORY = _Factory()
