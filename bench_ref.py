"""The reference arm of ``bench.py`` (``--impl reference``) and the shared
headline ``config`` of both arms.

This module imports numpy and the REFERENCE only -- never
``paper_2311_15038_b200`` and never its shared library -- so the reference arm
measures ctprev's own CPU code path:

* ctprev itself, from ``baseline/_ref`` (installed there by ``pip install
  --no-deps --target baseline/_ref /root/reference/pkg``; ``kind: "reference"``),
  or, when that is absent, the numpy restatement in ``oracle/`` (``kind: "port"``);
* the config-2 composition of SURVEY.md s8(d), exactly as the GPU arm runs it:
      bins  = artifact_bins(v)                                  mask.py:215-231
      hist  = volume_histogram(v)                               volume.py:252-262
      f     = filter_histogram_bins(v, bins)                    mask.py:234-246
      L_s   = downscale_volume(f, (s, s, s)), s = 512/256/128   volume.py:277-309
      maps  = encode_slicemaps(L_s, plan_scheme(s))             slicemap.py:120-142
  fanned out over z-slabs on every host core (exact, since
  histograms of slabs sum, the filter is per voxel and the power-of-two
  downscales are separable on slabs of whole level-3 cells), and once "as is"
  (one process, the functions called on one volume) on a bounded sample;
* ``render_view`` in the reference's additive mode on the config-4 volume
  (render.py:125-146; numba, all host threads).

Inputs come from a numpy generator with the GPU arm's SynthSpec parameters
(BASELINE.json configs; the bytes differ from the device generator's, the
CPU cost of this path does not depend on them).
"""
from __future__ import annotations

import json
import math
import mmap
import os
import sys
import time
from pathlib import Path

import numpy as np

ROOT = Path(__file__).resolve().parent
METRIC = "pipeline GVoxel/s (hist+filter+slicemaps) & MIP frames/s, % of HBM roofline"
SCHEMES = (512, 256, 128)

# the GPU arm's synth.config("c2") / ("c4") parameters (tests/test_host_logic.py checks they agree)
GEN = {
    "c2": dict(shape=(1024, 1024, 1024), seed=0, n_shells=12, bg=(20.0, 6.0), shell=(160.0, 20.0),
               axes=(40.0, 110.0), thickness=(3.0, 6.0), speckle_p=0.01, vmax=255),
    "c4": dict(shape=(1024, 1024, 1024), seed=0, n_shells=3, bg=(20.0, 6.0), shell=(160.0, 20.0),
               axes=(40.0, 110.0), thickness=(3.0, 6.0), speckle_p=0.0, vmax=255),
}


def headline_config(world: int) -> dict:
    """The ``config`` of the headline line -- the SAME dict in both arms."""
    return {"workload": "c2: 1024^3 u8 (one volume), volume_histogram + artifact_bins + filter_histogram_bins + "
                        "512/256/128 levels (downscale_volume, each direct from the filtered volume) + "
                        "encode_slicemaps atlases (8x4096^2, 4x2048^2, 2x1024^2)",
            "voxels_per_step": 1024 ** 3,
            "parallelism": "1 GPU" if world == 1 else f"z-slab sharded x{world} (one volume)",
            "l2": "input 1 GiB per step > 126 MB L2 (no flush needed)"}


# ---------------------------------------------------------------------------
# numpy generator (same spec as paper_2311_15038_b200.synth; independent bytes)

def shells(p: dict):
    """(cx, cy, cz, ax, ay, az, thickness, mean, sd) per shell -- SynthSpec.shells' draw order."""
    rng = np.random.default_rng(p["seed"])
    nz, ny, nx = p["shape"]
    out = []
    for _ in range(p["n_shells"]):
        ax, ay, az = rng.uniform(p["axes"][0], p["axes"][1], size=3)
        cx = rng.uniform(0.25, 0.75) * nx
        cy = rng.uniform(0.25, 0.75) * ny
        cz = rng.uniform(0.25, 0.75) * nz
        th = rng.uniform(p["thickness"][0], p["thickness"][1])
        mean = rng.normal(p["shell"][0], p["shell"][1] * 0.25)
        out.append((cx, cy, cz, ax, ay, az, th, mean, p["shell"][1]))
    return out


def gen_slab(p: dict, z0: int, z1: int, out: np.ndarray) -> None:
    """Slices [z0, z1) of the volume into ``out`` (uint8)."""
    nz, ny, nx = p["shape"]
    rng = np.random.default_rng([p["seed"], z0])
    v = rng.standard_normal((z1 - z0, ny, nx), dtype=np.float32)
    v *= np.float32(p["bg"][1])
    v += np.float32(p["bg"][0])
    for (cx, cy, cz, ax, ay, az, th, mean, sd) in shells(p):
        za, zb = max(z0, int(cz - az) - 1), min(z1, int(cz + az) + 2)
        if za >= zb:
            continue
        ya, yb = max(0, int(cy - ay) - 1), min(ny, int(cy + ay) + 2)
        xa, xb = max(0, int(cx - ax) - 1), min(nx, int(cx + ax) + 2)
        z = (np.arange(za, zb, dtype=np.float32) + 0.5 - cz)[:, None, None]
        y = (np.arange(ya, yb, dtype=np.float32) + 0.5 - cy)[None, :, None]
        x = (np.arange(xa, xb, dtype=np.float32) + 0.5 - cx)[None, None, :]
        qo = x * x / (ax * ax) + y * y / (ay * ay) + z * z / (az * az)
        ix, iy, iz = max(ax - th, 0.5), max(ay - th, 0.5), max(az - th, 0.5)
        qi = x * x / (ix * ix) + y * y / (iy * iy) + z * z / (iz * iz)
        m = (qo <= 1.0) & (qi >= 1.0)
        blk = v[za - z0:zb - z0, ya:yb, xa:xb]
        blk[m] = mean + sd * rng.standard_normal(int(m.sum()), dtype=np.float32)
    if p["speckle_p"] > 0:
        m = rng.random(v.shape, dtype=np.float32) < p["speckle_p"]
        v[m] = rng.random(int(m.sum()), dtype=np.float32) * (p["vmax"] + 1) - 0.5
    np.rint(v, out=v)
    np.clip(v, 0, p["vmax"], out=v)
    out[...] = v.astype(np.uint8)


_GEN_BUF = None
_GEN_P = None


def _gen_task(zr):
    z0, z1 = zr
    gen_slab(_GEN_P, z0, z1, _GEN_BUF[z0:z1])
    return z1 - z0


def generate(p: dict, workers: int) -> np.ndarray:
    """The whole volume, generated by ``workers`` forked processes into shared memory."""
    global _GEN_BUF, _GEN_P
    import multiprocessing as mp
    nz, ny, nx = p["shape"]
    mm = mmap.mmap(-1, nz * ny * nx)  # MAP_SHARED | MAP_ANONYMOUS: the children's writes land here
    buf = np.frombuffer(mm, dtype=np.uint8).reshape(nz, ny, nx)
    _GEN_BUF, _GEN_P = buf, p
    step = 16
    with mp.get_context("fork").Pool(workers) as pool:
        pool.map(_gen_task, [(z, min(nz, z + step)) for z in range(0, nz, step)])
    _GEN_BUF = None
    return np.array(buf)  # private, C-contiguous copy (the mmap is released)


# ---------------------------------------------------------------------------
# the reference's functions, or the oracle port when ctprev is not installed

class Ref:
    """ctprev's own entry points (``kind = "reference"``) or the oracle port (``"port"``)."""

    def __init__(self):
        ref_dir = ROOT / "baseline" / "_ref"
        os.environ.setdefault("NUMBA_CACHE_DIR", "/tmp/ctp_ref_numba_cache")
        self.kind = "port"
        self.where = "oracle/ctp_oracle.py (numpy restatement of ctprev)"
        try:
            if ref_dir.is_dir() and str(ref_dir) not in sys.path:
                sys.path.insert(0, str(ref_dir))
            import ctprev  # noqa: F401
            from ctprev import mask, render, slicemap, volume
            self.m = {"volume": volume, "mask": mask, "slicemap": slicemap, "render": render}
            self.kind = "reference"
            self.where = f"ctprev {getattr(ctprev, '__version__', '')} from {Path(ctprev.__file__).parent}"
        except Exception as e:  # pragma: no cover - depends on the box
            self.import_error = repr(e)[:200]
            from oracle import ctp_oracle as O
            self.O = O

    # Volume wrapping
    def vol(self, arr):
        return self.m["volume"].Volume(arr) if self.kind == "reference" else arr

    def arr(self, v):
        return v.voxels if self.kind == "reference" else v

    def volume_histogram(self, v, z_range=None):
        if self.kind == "reference":
            return self.m["volume"].volume_histogram(v, z_range).bins
        return self.O.histogram(v, z_range)

    def artifact_bins(self, v):
        return self.m["mask"].artifact_bins(v) if self.kind == "reference" else self.O.artifact_bins(v)

    def filter_histogram_bins(self, v, bins):
        if self.kind == "reference":
            return self.m["mask"].filter_histogram_bins(v, bins)
        return self.O.filter_histogram_bins(v, bins)

    def downscale_volume(self, v, target):
        if self.kind == "reference":
            return self.m["volume"].downscale_volume(v, target)
        return self.O.downscale(v, target)

    def encode_slicemaps(self, v, s):
        if self.kind == "reference":
            sm = self.m["slicemap"]
            return sm.encode_slicemaps(v, sm.plan_scheme(s)).atlases
        return self.O.encode_slicemaps(v, self.O.plan_scheme(s))

    def render_additive(self, v, azimuth, dim, steps):
        if self.kind == "reference":
            r = self.m["render"]
            return r.render_view(v, r.ViewParams(azimuth_deg=azimuth, image_dim=dim, steps=steps, mode="additive"))
        return self.O.render_view(v, azimuth, dim, steps, "additive")

    def threads(self) -> int:
        if self.kind == "reference":
            import numba
            return int(numba.get_num_threads())
        return 1


REF: Ref | None = None
VOL = None  # the whole c2 volume (a ctprev Volume), inherited by the forked workers


def _slab_task(args):
    """One z-slab [z0, z1) through the reference functions: its histogram, its
    filtered voxels and its share of each level (whole level-3 cells)."""
    z0, z1, bins = args
    nz, ny, nx = REF.arr(VOL).shape
    h = REF.volume_histogram(VOL, (z0, z1))                                   # volume.py:252-262 (z_range)
    f = REF.filter_histogram_bins(REF.vol(REF.arr(VOL)[z0:z1]), bins)          # mask.py:234-246
    lv = []
    for s in SCHEMES:                                                         # volume.py:277-309 per slab
        r = nz // s                                                           # isotropic 1024^3: r on every axis
        lv.append(REF.arr(REF.downscale_volume(f, (nx // r, ny // r, (z1 - z0) // r))))
    return z0, np.asarray(h), lv


def _pack_cells(level_slices: np.ndarray, s: int, k0: int) -> None:
    """encode_slicemaps' packing (slicemap.py:132-141) of the atlas maps that level slices
    [k0, k0 + n) fall in -- used only for a step that samples part of the volume, where
    encode_slicemaps itself (which needs the whole s^3 level) cannot run; 0.1% of the work."""
    g = 8
    per = g * g
    n = level_slices.shape[0]
    for m in range(k0 // per, -(-(k0 + n) // per)):
        blk = np.zeros((per, s, s), dtype=np.uint8)
        a0, a1 = max(m * per, k0), min((m + 1) * per, k0 + n)
        blk[a0 - m * per:a1 - m * per] = level_slices[a0 - k0:a1 - k0]
        blk.reshape(g, g, s, s).transpose(0, 2, 1, 3).reshape(g * s, g * s).copy()


def cpu_baseline(vol_u8: np.ndarray, n_slices: int = 512) -> dict:
    """The GPU arm's ``cpu_baseline``: the fanned-out composition on ``n_slices`` slices of
    the GPU arm's own volume (copied to the host), all host cores."""
    global REF, VOL
    import multiprocessing as mp
    REF = Ref()
    VOL = REF.vol(vol_u8)
    workers = os.cpu_count() or 1
    task = max(8, n_slices // (2 * workers) // 8 * 8)
    with mp.get_context("fork").Pool(workers) as pool:
        fanned_step(pool, 0, 64, 8)
        t = time.perf_counter()
        n = fanned_step(pool, 0, n_slices, task)
        sec = time.perf_counter() - t
    VOL = None
    return {"value": n / sec / 1e9, "unit": "GVoxel/s", "cores": workers, "kind": REF.kind,
            "sample": f"{n_slices} of 1024 z-slices of the GPU arm's c2 volume: artifact_bins + volume_histogram + "
                      f"filter_histogram_bins + downscale_volume x3 per {task}-slice slab on a {workers}-process pool "
                      f"+ atlas packing ({REF.where})", "seconds": sec}


def fanned_step(pool, z_lo: int, z_hi: int, task_slices: int):
    """The c2 composition over slices [z_lo, z_hi) on the pool.  Returns voxels processed."""
    nz, ny, nx = REF.arr(VOL).shape
    bins = REF.artifact_bins(VOL)                                             # mask.py:215-231 (top 3 slices)
    tasks = [(z, min(z + task_slices, z_hi), bins) for z in range(z_lo, z_hi, task_slices)]
    res = pool.map(_slab_task, tasks)
    hist = np.zeros(256, dtype=np.int64)
    levels = {s: np.empty(((z_hi - z_lo) * s // nz, s, s), dtype=np.uint8) for s in SCHEMES}
    for z0, h, lv in res:
        hist += h
        for s, l in zip(SCHEMES, lv):
            k = (z0 - z_lo) * s // nz
            levels[s][k:k + l.shape[0]] = l
    for s in SCHEMES:
        if z_lo == 0 and z_hi == nz:
            REF.encode_slicemaps(REF.vol(levels[s]), s)                       # slicemap.py:120-142
        else:
            _pack_cells(levels[s], s, z_lo * s // nz)
    assert int(hist.sum()) == (z_hi - z_lo) * ny * nx
    return (z_hi - z_lo) * ny * nx


def as_is_pass(n_slices: int) -> float:
    """The composition called exactly as the oracle composes it, in ONE process, on a
    volume of the first ``n_slices`` slices (numpy is single-threaded).  GVoxel/s."""
    arr = np.ascontiguousarray(REF.arr(VOL)[:n_slices])
    v = REF.vol(arr)
    nz, ny, nx = arr.shape
    t = time.perf_counter()
    REF.volume_histogram(v)
    bins = REF.artifact_bins(v)
    f = REF.filter_histogram_bins(v, bins)
    for s in SCHEMES:
        r = 1024 // s
        lv = REF.downscale_volume(f, (nx // r, ny // r, nz // r))
        if REF.arr(lv).shape == (s, s, s):
            REF.encode_slicemaps(lv, s)
    return nz * ny * nx / (time.perf_counter() - t) / 1e9


def render_reference(workers: int) -> dict:
    """render_view additive (render.py:125-146) on the config-4 volume: 1024^2, 0.5-voxel
    steps (3548), numba on all host threads.  One frame after a JIT warm-up."""
    global VOL
    p = GEN["c4"]
    v = REF.vol(generate(p, workers))
    steps = math.ceil(4 * math.sqrt(3.0) / 2.0 * p["shape"][0])
    t = time.perf_counter()
    REF.render_additive(REF.vol(np.zeros((32, 32, 32), np.uint8)), 0.0, 16, 32)   # numba compile / cache load
    t_compile = time.perf_counter() - t
    t = time.perf_counter()
    REF.render_additive(v, 0.0, 1024, steps)
    s = time.perf_counter() - t
    return {"workload": f"render_view(v, ViewParams(0, 1024, {steps}, 'additive')) on the 1024^3 config-4 volume "
                        "(render.py:125-146), one frame", "s_per_frame": s, "frames_per_s": 1.0 / s,
            "threads": REF.threads(), "kind": REF.kind, "jit_or_cache_load_s": t_compile}


def run_reference(args) -> int:
    """--impl reference: rank 0 only (the others exit 0), all host cores, bounded samples."""
    global REF, VOL
    if int(os.environ.get("RANK", "0")) != 0:
        return 0
    import multiprocessing as mp
    world = int(os.environ.get("WORLD_SIZE", "1"))
    workers = os.cpu_count() or 1
    REF = Ref()
    p = GEN["c2"]
    nz = p["shape"][0]
    VOL = REF.vol(generate(p, workers))
    with mp.get_context("fork").Pool(workers) as pool:
        # calibration on 64 slices, then the per-step sample: the whole volume when the run fits
        # ~150 s, else fewer slices (multiples of 64: whole level-3 cells, 8 slices per task)
        fanned_step(pool, 0, 64, 8)
        t = time.perf_counter()
        fanned_step(pool, 0, 128, 8)
        per_slice = (time.perf_counter() - t) / 128
        budget = 150.0 / max(1, args.steps + args.warmup)
        sample = int(min(nz, max(64, budget / max(per_slice, 1e-9))) // 64 * 64)
        task = max(8, sample // (2 * workers) // 8 * 8)
        for _ in range(args.warmup):
            fanned_step(pool, 0, sample, task)
        t0 = time.perf_counter()
        vox = 0
        for i in range(args.steps):
            z0 = min((i * sample) % nz, nz - sample)
            vox += fanned_step(pool, z0, z0 + sample, task)
        dt = time.perf_counter() - t0
    value = vox / dt / 1e9
    as_is_n = 128
    as_is = {"value": as_is_pass(as_is_n), "unit": "GVoxel/s", "cores": 1, "kind": REF.kind,
             "sample": f"the composition on the first {as_is_n} slices as one {as_is_n}x1024x1024 volume, "
                       "one process (BASELINE.md s3.1)"}
    try:
        render = render_reference(workers)
    except Exception as e:  # pragma: no cover - reported in the line
        render = {"error": repr(e)[:200]}
    sample_txt = (f"{sample} of {nz} z-slices per step ({'the whole volume' if sample == nz else 'bounded sample'}): "
                  f"artifact_bins + volume_histogram(z_range) + filter_histogram_bins + downscale_volume x3 per "
                  f"slab of {task} slices on a {workers}-process pool, encode_slicemaps of the assembled levels "
                  f"({REF.where})")
    line = {"metric": METRIC, "value": value, "unit": "GVoxel/s", "n_gpus": world, "steps": args.steps,
            "warmup": args.warmup, "ms_per_step": dt / args.steps * 1e3, "higher_is_better": True,
            "scaling": "strong", "vs_baseline": None, "dtype": "u8",
            "data": "synthetic (config-2 generator, numpy)", "impl": "reference",
            "config": headline_config(world),
            "cpu_baseline": {"value": value, "unit": "GVoxel/s", "cores": workers, "kind": REF.kind,
                             "sample": sample_txt},
            "e2e": {"value": value, "unit": "GVoxel/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
            "as_is": as_is, "c4_additive": render}
    if REF.kind == "port":
        line["reference_import_error"] = getattr(REF, "import_error", None)
    print(json.dumps(line))
    return 0
