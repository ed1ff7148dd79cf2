"""Host-side logic of the drop-in (CPU only): type validation mirroring the
reference, planning of fused vs general levels, the float64 cutoff rule, the
install() rebinding, and that the product never imports the oracle."""
from __future__ import annotations

import importlib
import math
import os
import re
import sys
from pathlib import Path

import numpy as np
import pytest

import paper_2311_15038_b200 as P
from paper_2311_15038_b200 import device as dev
from paper_2311_15038_b200.device import AtlasSpec
from paper_2311_15038_b200.pipeline import level_for_target, plan_preview

ROOT = Path(__file__).resolve().parents[1]


def test_product_does_not_import_the_oracle():
    for f in (ROOT / "paper_2311_15038_b200").rglob("*.py"):
        text = f.read_text()
        assert not re.search(r"^\s*(from|import)\s+oracle", text, re.M), f
        assert "ctp_oracle" not in text, f


def test_volume_mirror_validation():
    with pytest.raises(P.UnsupportedPixelFormat):
        P.Volume(np.zeros((2, 2, 2), np.uint16))
    with pytest.raises(P.DimensionMismatch):
        P.Volume(np.zeros((2, 2), np.uint8))
    with pytest.raises(P.DimensionMismatch):
        P.Volume(np.zeros((0, 2, 2), np.uint8))
    v = P.Volume(np.zeros((3, 4, 5), np.uint8))
    assert v.dims == (5, 4, 3) and not v.voxels.flags.writeable
    with pytest.raises(P.RangeOutOfBounds):
        v.slice_xy(3)


def test_histogram_mirror_validation():
    with pytest.raises(P.DimensionMismatch):
        P.Histogram256(np.zeros(255))
    with pytest.raises(P.RangeOutOfBounds):
        P.Histogram256(-np.ones(256))
    assert P.Histogram256(np.ones(256)).total == 256


def test_scheme_mirror_validation():
    for s, atlas, maps in ((128, 1024, 2), (256, 2048, 4), (512, 4096, 8)):  # test_slicemap.py:35-41
        sc = P.plan_scheme(s)
        assert (sc.s, sc.atlas_dim, sc.grid, sc.map_count) == (s, atlas, 8, maps)
    for s in (64, 100, 1024, 0):
        with pytest.raises(P.UnsupportedScheme):
            P.plan_scheme(s)
    with pytest.raises(P.UnsupportedScheme):
        P.SlicemapScheme(s=128, atlas_dim=1000, grid=8, map_count=2)
    with pytest.raises(P.UnsupportedScheme):
        P.SlicemapScheme(s=128, atlas_dim=1024, grid=8, map_count=3)
    assert P.slice_cell(9, P.plan_scheme(128)) == (0, 1, 1)
    assert P.slice_cell(511, P.plan_scheme(512)) == (7, 7, 7)
    with pytest.raises(P.IndexOutOfRange):
        P.slice_cell(128, P.plan_scheme(128))
    assert P.plan_scheme(256).atlas_names()[3] == "sm_256_3.png"


def test_view_params_mirror():
    assert P.ViewParams(azimuth_deg=370.0).azimuth_deg == 10.0
    assert P.ViewParams(azimuth_deg=-45.0).azimuth_deg == 315.0
    for kw in ({"image_dim": 15}, {"steps": 31}, {"mode": "volumetric"}, {"threshold": 256}, {"gain": 0.0},
               {"tf": ((0, 0, 0, 0, 0),) * 4}, {"early_stop": 0.0}):
        with pytest.raises(P.RangeOutOfBounds):
            P.ViewParams(**kw)
    P.ViewParams(mode="mip")
    P.ViewParams(mode="alpha")


def test_cutoff_floor_matches_float_comparison():
    # mask.py:229-230: count > frac * size (float64) <=> count > floor(cutoff)
    rng = np.random.default_rng(0)
    for _ in range(2000):
        frac = float(rng.choice([0.0005, 0.0, 0.01, 1e-7, 0.123456, 1.0]))
        size = int(rng.integers(1, 10 ** 7))
        cutoff = frac * size
        t = dev.cutoff_floor(frac, size)
        for count in (t - 1, t, t + 1, t + 2):
            if count >= 0:
                assert (count > cutoff) == (count > t)
    assert dev.cutoff_floor(0.0005, 3 * 1024 * 1024) == 1572  # config 2: flag counts >= 1573


def test_level_for_target_and_plan():
    assert level_for_target((1024, 1024, 1024), (512, 512, 512)) == 1
    assert level_for_target((1024, 1024, 1024), (128, 128, 128)) == 3
    assert level_for_target((96, 160, 160), (128, 128, 96)) is None
    assert level_for_target((10, 10, 10), (5, 5, 5)) == 1
    sch = {s: AtlasSpec.of(P.plan_scheme(s)) for s in (512, 256, 128)}
    p = plan_preview((1024, 1024, 1024), sch)
    assert p.fused == {1: sch[512], 2: sch[256], 3: sch[128]} and not p.general and p.nlev == 3
    p = plan_preview((96, 160, 160), {128: AtlasSpec.of(P.plan_scheme(128))})
    assert p.general == [128] and p.fused == {0: "xyz"}
    c1 = {256: AtlasSpec(256, 4096, 16, 1)}
    p = plan_preview((256, 256, 256), c1)
    assert p.fused == {0: c1[256]}
    p = plan_preview((256, 256, 256), c1, keep_filtered=True)  # level 0 needed dense AND as an atlas
    assert p.fused == {0: "xyz"} and p.general == [256]
    p = plan_preview((64, 64, 72), {64: AtlasSpec(64, 512, 8, 1)})  # nx % 16 != 0 -> general
    assert p.general == [64]


def test_errors_share_one_base():
    for name in ("InvalidTarget", "RangeOutOfBounds", "UnsupportedScheme", "ManifestMismatch", "IndexOutOfRange"):
        assert issubclass(getattr(P, name), P.CTPrevError)


def test_no_cuda_means_loud_failure(monkeypatch):
    import torch
    if torch.cuda.is_available():
        pytest.skip("a CUDA device is present")
    from paper_2311_15038_b200 import _lib
    with pytest.raises(_lib.NativeUnavailable):
        P.volume_histogram(P.Volume(np.zeros((2, 2, 2), np.uint8)))


@pytest.mark.skipif(not Path("/root/reference/pkg/src/ctprev").exists(), reason="reference not mounted")
def test_install_rebinds_every_site(monkeypatch, tmp_path):
    import os
    monkeypatch.setenv("NUMBA_CACHE_DIR", str(tmp_path))
    monkeypatch.setattr(sys, "dont_write_bytecode", True)
    monkeypatch.syspath_prepend("/root/reference/pkg/src")
    ctprev = importlib.import_module("ctprev")
    inst = importlib.import_module("paper_2311_15038_b200.install")
    try:
        patched = inst.install()
        assert "ctprev.pipeline.encode_slicemaps" in patched and "ctprev.slicemap.downscale_volume" in patched
        import ctprev.cli, ctprev.mask, ctprev.pipeline, ctprev.render, ctprev.slicemap, ctprev.volume  # noqa: E401
        assert ctprev.pipeline.volume_histogram is P.volume_histogram
        assert ctprev.slicemap.downscale_volume is P.downscale_volume
        assert ctprev.render.render_view is P.render_view
        assert ctprev.volume_histogram is P.volume_histogram
        assert ctprev.pipeline.load_slice_stack is P.load_slice_stack
        assert ctprev.cli.load_volume is P.load_volume
        from paper_2311_15038_b200.types import FACTORY
        assert FACTORY.Volume is ctprev.volume.Volume and FACTORY.SlicemapSet is ctprev.slicemap.SlicemapSet
    finally:
        inst.uninstall()
    import ctprev.volume
    assert ctprev.volume.volume_histogram is not P.volume_histogram


def test_reference_arm_is_independent_of_the_package():
    """bench_ref (the --impl reference arm) imports numpy + ctprev only: importing it and
    generating a slab must not import paper_2311_15038_b200 (nor load its .so), and its
    generator parameters are the GPU arm's synth.config c2 / c4."""
    import subprocess
    code = ("import sys; sys.path.insert(0, %r); import bench_ref, numpy as np\n"
            "out = np.empty((2, 64, 64), np.uint8); p = dict(bench_ref.GEN['c2'], shape=(8, 64, 64))\n"
            "bench_ref.gen_slab(p, 0, 2, out); bench_ref.headline_config(1)\n"
            "assert not any(m.startswith('paper_2311_15038_b200') for m in sys.modules), 'package imported'\n"
            "print('ok', int(out.max()))\n") % str(ROOT)
    r = subprocess.run([sys.executable, "-c", code], capture_output=True, text=True, timeout=120)
    assert r.returncode == 0 and r.stdout.startswith("ok"), r.stderr
    import bench_ref
    from paper_2311_15038_b200 import synth
    for name in ("c2", "c4"):
        sp, p = synth.config(name), bench_ref.GEN[name]
        assert (sp.shape, sp.seed, sp.n_shells, (sp.bg_mean, sp.bg_sd), (sp.shell_mean, sp.shell_sd), sp.axes,
                sp.thickness, sp.speckle_p) == (p["shape"], p["seed"], p["n_shells"], p["bg"], p["shell"], p["axes"],
                                                p["thickness"], p["speckle_p"]), name
        assert [tuple(s) for s in sp.shells()] == [tuple(s) for s in bench_ref.shells(p)], name


def test_install_binds_reference_error_classes_when_imported_later():
    """ctprev imported AFTER this package: install() rebinds the error classes everywhere in
    the package, so the drop-in builders catch ctprev's own NoCircleFound / DegenerateHistogram
    (raised by its host circle detector / Otsu) and raise what ctprev's callers catch."""
    import subprocess
    ref = next((d for d in (ROOT / "baseline" / "_ref", Path("/root/reference/pkg/src")) if (d / "ctprev").is_dir()),
               None)
    if ref is None:
        pytest.skip("ctprev not installed nor mounted")
    code = ("import sys; sys.path.insert(0, %r)\n"
            "import paper_2311_15038_b200 as P\n"
            "from paper_2311_15038_b200 import errors, ingest, ops, types\n"
            "assert not errors.FROM_REFERENCE\n"
            "sys.path.insert(0, %r)\n"
            "import ctprev.errors as E\n"
            "P.install()\n"
            "assert ops.RangeOutOfBounds is E.RangeOutOfBounds and ingest.MissingSlice is E.MissingSlice\n"
            "assert types.DimensionMismatch is E.DimensionMismatch and P.NoCircleFound is E.NoCircleFound\n"
            "from paper_2311_15038_b200.errors import NoCircleFound\n"
            "assert NoCircleFound is E.NoCircleFound\n"
            "print('ok')\n") % (str(ROOT), str(ref))
    r = subprocess.run([sys.executable, "-c", code], capture_output=True, text=True, timeout=120,
                       env={**os.environ, "NUMBA_CACHE_DIR": "/tmp/ctp_numba_err_test"})
    assert r.returncode == 0 and r.stdout.strip() == "ok", r.stderr


def test_device_cache_only_tracks_arrays_frozen_all_the_way_down():
    """The device-copy cache of the host drop-ins (hostio.DeviceCache) must never serve a
    stale copy: a read-only view of an array the caller can still write through is not
    cached (Volume freezes only the view it is given, volume.py:60-62), a view whose base
    nobody else refers to (Volume(data.reshape(...)), volume.py:249) is."""
    from paper_2311_15038_b200.hostio import DeviceCache

    def loaded():
        data = np.zeros(4 << 20, np.uint8)
        v = data.reshape(4, 1 << 10, 1 << 10)
        v.setflags(write=False)
        return v

    v = loaded()
    assert DeviceCache.cacheable(v)
    base = v.base                      # the caller got hold of the writeable owner
    assert not DeviceCache.cacheable(v)
    del base
    assert DeviceCache.cacheable(v)
    big = np.zeros((4, 1 << 20), np.uint8)
    w = big[1:3]
    w.setflags(write=False)
    assert not DeviceCache.cacheable(w)  # big[...] = x would change w
    big.setflags(write=False)
    assert DeviceCache.cacheable(w)
    own = np.zeros(4 << 20, np.uint8)
    assert not DeviceCache.cacheable(own)
    own.setflags(write=False)
    assert DeviceCache.cacheable(own)
    assert not DeviceCache.cacheable(np.zeros(16, np.uint8))  # too small to track
