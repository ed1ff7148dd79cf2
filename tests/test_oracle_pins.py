"""Pin the CPU oracle before trusting it (CPU only).

1. Against the golden vectors produced by running the reference itself
   (tests/golden/make_golden.py -> ref_golden.npz).
2. Against the known answers in the reference's own tests
   (pkg/tests/test_volume.py, test_mask.py, test_slicemap.py, test_render.py).
"""
from __future__ import annotations

import math
from pathlib import Path

import numpy as np
import pytest

from oracle import ctp_oracle as O

ROOT = Path(__file__).resolve().parents[1]


# ---------------------------------------------------------------- golden vectors

def test_histogram_golden(golden):
    for i in range(int(golden["hist_n"])):
        zr = tuple(int(x) for x in golden[f"hist{i}_z"])
        zr = None if zr == (-1, -1) else zr
        assert np.array_equal(O.histogram(golden[f"hist{i}_in"], zr), golden[f"hist{i}_out"])


def test_artifact_bins_and_filter_golden(golden):
    for i in range(int(golden["art_n"])):
        v = golden[f"art{i}_in"]
        bins = O.artifact_bins(v, int(golden[f"art{i}_ntop"]), float(golden[f"art{i}_frac"]))
        assert sorted(bins) == golden[f"art{i}_bins"].tolist()
        assert np.array_equal(O.filter_histogram_bins(v, bins), golden[f"art{i}_filtered"])


def test_downscale_golden(golden):
    for i in range(int(golden["ds_n"])):
        out = O.downscale(golden[f"ds{i}_in"], tuple(golden[f"ds{i}_target"]))
        assert np.array_equal(out, golden[f"ds{i}_out"]), i


def test_encode_golden(golden):
    for i in range(int(golden["enc_n"])):
        sc = tuple(int(x) for x in golden[f"enc{i}_scheme"])
        atl = np.stack(O.encode_slicemaps(golden[f"enc{i}_in"], sc))
        assert np.array_equal(atl, golden[f"enc{i}_out"]), i


def _render_vol(golden, i):
    return golden[bytes(golden[f"rv{i}_vol"]).decode()]


def test_render_golden_bit_exact(golden):
    for i in range(int(golden["rv_n"])):
        az, dim, steps, add, thr = golden[f"rv{i}_params"]
        img = O.render_view(_render_vol(golden, i), az, int(dim), int(steps), "additive" if add else "surface",
                            int(thr))
        assert np.array_equal(img, golden[f"rv{i}_out"]), i


def test_entropy_golden(golden):
    for i in range(int(golden["ent_n"])):
        assert O.image_entropy(golden[f"ent{i}_in"])[0] == float(golden[f"ent{i}_h"])


def test_snapshot_golden(golden):
    az, img, h, per_view = O.optimal_snapshot(golden["lphantom"], 12, 128, 64, "surface", 60)
    assert az == float(golden["snap_az"]) == 300.0           # test_render.py:178
    assert h == float(golden["snap_h"]) and abs(h - 0.798789) <= 1e-5  # test_render.py:179
    assert np.array_equal(np.array(per_view), golden["snap_per_view"])
    assert np.array_equal(img, golden["snap_img"])


# ------------------------------------------------ reference tests' known answers

def test_hist_known_answers():
    data = np.zeros((2, 2, 2), dtype=np.uint8)          # test_volume.py:70-78
    data.ravel()[:4] = [1, 1, 2, 255]
    h = O.histogram(data)
    assert h.sum() == 8 and h[0] == 4 and h[1] == 2 and h[2] == 1 and h[255] == 1
    data = np.zeros((4, 2, 2), dtype=np.uint8)          # test_volume.py:80-86 (half-open)
    data[1] = 9
    data[2] = 9
    h = O.histogram(data, (1, 3))
    assert h.sum() == 8 and h[9] == 8


def test_artifact_known_answers():
    vox = np.zeros((8, 64, 64), dtype=np.uint8)         # test_mask.py:155-164
    vox[:6] = 90
    vox[6:] = 140
    vox[6:, :8, :8] = 200
    vox[7, 30, 30] = 90
    assert sorted(O.artifact_bins(vox, n_top=2)) == [0, 140, 200]
    assert 90 not in O.artifact_bins(vox, n_top=2)
    with pytest.raises(ValueError):
        O.artifact_bins(vox, n_top=0)
    with pytest.raises(ValueError):
        O.artifact_bins(vox, n_top=9)


def test_filter_known_answers():
    vox = np.arange(256, dtype=np.uint8).reshape(1, 16, 16)  # test_mask.py:187-194
    out = O.filter_histogram_bins(vox, {10, 200})
    assert out[0, 0, 10] == 0 and out[0, 12, 8] == 0
    keep = np.ones(256, dtype=bool)
    keep[[0, 10, 200]] = False
    assert np.array_equal(out.ravel()[keep], vox.ravel()[keep])


def test_downscale_known_answers():
    rng = np.random.default_rng(2)                      # test_volume.py:200-207
    data = rng.integers(0, 256, size=(8, 8, 8), dtype=np.uint8)
    blocks = data.reshape(4, 2, 4, 2, 4, 2).sum(axis=(1, 3, 5), dtype=np.int64)
    assert np.array_equal(O.downscale(data, (4, 4, 4)), ((2 * blocks + 8) // 16).astype(np.uint8))
    data = np.arange(10, dtype=np.uint8).reshape(1, 1, 10).repeat(16, axis=0)  # test_volume.py:209-216
    data = np.ascontiguousarray(data.repeat(16, axis=1))[:16, :16, :]
    assert O.downscale(data, (4, 16, 16))[0, 0].tolist() == [1, 3, 6, 8]
    assert O.cell_starts(10, 4).tolist() == [0, 2, 5, 7, 10]
    v = np.full((7, 9, 11), 137, dtype=np.uint8)       # test_volume.py:218-221
    assert (O.downscale(v, (3, 4, 5)) == 137).all()
    two = np.array([0, 0, 0, 0, 255, 255, 255, 255], dtype=np.uint8).reshape(2, 2, 2)
    assert O.downscale(two, (1, 1, 1))[0, 0, 0] == 128


def test_slicemap_known_answers():
    for s, atlas, maps in ((128, 1024, 2), (256, 2048, 4), (512, 4096, 8)):  # test_slicemap.py:35-41
        assert O.plan_scheme(s) == (s, atlas, 8, maps)
    sc = O.plan_scheme(128)                              # test_slicemap.py:88-97
    vox = np.zeros((128, 128, 128), dtype=np.uint8)
    vox[77, 13, 101] = 251
    atl = O.encode_slicemaps(vox, sc)
    k = 77
    m, w = divmod(k, 64)
    cy, cx = divmod(w, 8)
    assert atl[m][cy * 128 + 13, cx * 128 + 101] == 251
    assert int(np.count_nonzero(np.stack(atl))) == 1
    sc96 = (96, 768, 8, 2)                               # test_slicemap.py:110-121
    v = np.full((96, 96, 96), 9, dtype=np.uint8)
    atl = O.encode_slicemaps(v, sc96)
    tail = atl[1].reshape(8, 96, 8, 96).transpose(0, 2, 1, 3).reshape(64, 96, 96)
    assert (tail[:32] == 9).all() and not tail[32:].any()
    assert np.array_equal(O.decode_slicemaps(atl, sc96), v)
    zs = np.arange(512, dtype=np.uint16).reshape(512, 1, 1)  # test_slicemap.py:129-135
    ys = np.arange(512, dtype=np.uint16).reshape(1, 512, 1)
    xs = np.arange(512, dtype=np.uint16).reshape(1, 1, 512)
    v = ((zs * 7 + ys * 3 + xs * 31) % 256).astype(np.uint8)
    assert np.array_equal(O.decode_slicemaps(O.encode_slicemaps(v, O.plan_scheme(512)), O.plan_scheme(512)), v)


def test_entropy_known_answers():
    assert O.image_entropy(np.full((64, 64), 7, dtype=np.uint8))[0] == 0.0  # test_render.py:140-153
    h = O.image_entropy(np.full((64, 64), 7, dtype=np.uint8))[0]
    assert math.copysign(1.0, h) == 1.0
    img = np.tile(np.arange(256, dtype=np.uint8), 256).reshape(256, 256)
    assert abs(O.image_entropy(img)[0] - 8.0) <= 1e-9
    img = np.zeros((64, 64), dtype=np.uint8)
    img[:32] = 255
    assert abs(O.image_entropy(img)[0] - 1.0) <= 1e-9


def test_sphere_silhouette_known_answer():
    # test_render.py:77-86 at reduced size (64^3 sphere, 128^2): within 3% of analytic
    n = 64
    zz, yy, xx = np.mgrid[0:n, 0:n, 0:n]
    vox = np.zeros((n, n, n), dtype=np.uint8)
    c = (n - 1) / 2
    vox[(xx - c) ** 2 + (yy - c) ** 2 + (zz - c) ** 2 <= 20.0 ** 2] = 200
    img = O.render_view(vox, 0.0, 128, 128, "surface", 100)
    r_px = (20.0 / n) * 128 / math.sqrt(3.0)
    analytic = math.pi * r_px * r_px
    assert abs(int((img > 0).sum()) - analytic) / analytic <= 0.03


def test_extension_rescale_rule():
    v = np.arange(4096)
    r = O.rescale_u16_to_u8(v)
    assert r[0] == 0 and r[4095] == 255 and r.dtype == np.uint8
    # round half up of v*255/4095, exact in integers
    exact = np.floor(v * 255 / 4095 + 0.5).astype(np.int64)
    assert np.array_equal(r.astype(np.int64), exact)
    assert np.all(np.diff(r.astype(int)) >= 0)
    lut = O.lut_u16({0, 5, 4095})
    assert lut[0] == 0 and lut[5] == 0 and lut[4095] == 0 and lut[4094] == r[4094]


def test_data_preview_golden():
    with np.load(Path(__file__).resolve().parent / "golden" / "ref_golden_datapreview.npz") as z:
        g = {k: z[k] for k in z.files}
    for i in range(int(g["dp_n"])):
        bins, atl = O.build_data_preview(g[f"dp{i}_in"])
        assert list(bins) == g[f"dp{i}_bins"].tolist()
        assert np.array_equal(np.stack(atl), g[f"dp{i}_atlases"])


def test_circle_mask_golden():
    with np.load(Path(__file__).resolve().parent / "golden" / "ref_golden_datapreview.npz") as z:
        g = {k: z[k] for k in z.files}
    for i in range(int(g["cm_n"])):
        cx, cy, r, m = g[f"cm{i}_params"]
        assert np.array_equal(O.apply_circle_mask(g["cm_in"], cx, cy, r, m), g[f"cm{i}_out"]), i


def test_otsu_matches_reference_interactive_golden():
    """The oracle's Otsu sweep reproduces the reference thresholds of
    build_interactive_preview from the same (reference-computed) histograms."""
    from pathlib import Path
    g = np.load(Path(__file__).resolve().parent / "golden" / "ref_golden_interactive.npz")
    for i in range(int(g["ip_n"])):
        for s in (128, 256, 512):
            t = O.otsu_threshold(g[f"ip{i}_hist{s}"])
            assert (-1 if t is None else t) == int(g[f"ip{i}_thr{s}"]), (i, s)


def test_oracle_viewer_frames_and_bundle_products():
    """The oracle on the recorded fixture bundle: decode the interactive-128 atlases and
    render the viewer's reference frames (bit-exact); data-preview bins from the volume."""
    import json
    from pathlib import Path
    with np.load(Path(__file__).resolve().parent / "golden" / "ref_golden_bundles.npz") as z:
        atl, fm, ref = z["b0_int128"], json.loads(str(z["frames_params"])), z["frames_img"]
        meta = json.loads(str(z["b0_meta"]))
        vol = z["b0_vol"]
        data = z["b0_data"]
    cube = O.decode_slicemaps(list(atl), (128, 1024, 8, 2))
    for k, fr in enumerate(fm["frames"]):
        img = O.render_view(cube, fr["azimuth"], fm["image_dim"], fm["steps"], fr["mode"], fr["threshold"], fm["gain"])
        assert np.array_equal(img, ref[k]), fr["file"]
    bins, atl_dp = O.build_data_preview(vol)
    assert sorted(bins) == meta["previews"]["data"]["filtered_bins"]
    assert np.array_equal(np.stack(atl_dp), data)


# ------------------------------------------------ the oracle against the LIVE reference (when mounted)

def _live_reference():
    """ctprev itself, from the mount or from baseline/_ref (neither exists on the GPU box)."""
    import importlib
    import os
    import sys
    os.environ.setdefault("NUMBA_CACHE_DIR", "/tmp/ctp_numba_oracle_live")
    for d in (ROOT / "baseline" / "_ref", Path("/root/reference/pkg/src")):
        if (d / "ctprev").is_dir():
            if str(d) not in sys.path:
                sys.path.insert(0, str(d))
            return importlib.import_module("ctprev")
    pytest.skip("ctprev is neither installed (baseline/_ref) nor mounted")


def test_oracle_equals_live_reference_on_the_gpu_sweeps():
    """The seeded sweeps the GPU tests compare against the oracle (test_gpu_parity.py:
    test_downscale_seeded_sweep_every_kernel_path, test_encode_decode_seeded_sweep_custom_schemes,
    test_render_fp64_seeded_sweep_bit_exact) replayed here against ctprev ITSELF: the same
    generators, the same seeds -- so "GPU == oracle" on the box is "GPU == reference"."""
    ct = _live_reference()
    # downscale (volume.py:277-309), a third of the GPU sweep's cases
    rng = np.random.default_rng(2025)
    for case in range(80):
        nx = int(rng.integers(1, 90)) if case % 4 == 3 else 16 * int(rng.integers(1, 40))
        ny, nz = int(rng.integers(1, 48)), int(rng.integers(1, 40))
        pick = lambda n: int(n if rng.random() < 0.15 else rng.integers(1, n + 1))  # noqa: E731
        tx = max(1, nx // int(rng.integers(16, 40))) if case % 5 == 0 else pick(nx)
        target = (tx, pick(ny), pick(nz))
        kind = case % 3
        if kind == 0:
            v = rng.integers(0, 256, size=(nz, ny, nx), dtype=np.uint8)
        elif kind == 1:
            v = np.full((nz, ny, nx), 255, np.uint8)
            v[rng.random((nz, ny, nx)) < 0.1] = 254
        else:
            v = (rng.random((nz, ny, nx)) < 0.07).astype(np.uint8) * rng.integers(1, 256, size=(nz, ny, nx), dtype=np.uint8)
        if target == (nx, ny, nz) or case % 3:
            continue
        assert np.array_equal(O.downscale(v, target), ct.downscale_volume(ct.Volume(v.copy()), target).voxels), case
    # encode / decode with custom schemes (slicemap.py:120-155)
    rng = np.random.default_rng(77)
    for case in range(40):
        g = int(rng.integers(1, 10))
        s = int(rng.choice([8, 12, 16, 20, 24, 32, 33, 40, 48, 64]))
        maps = -(-s // (g * g))
        grow = lambda: int(s if rng.random() < 0.5 else s + rng.integers(1, s + 1))  # noqa: E731
        shape = (grow(), grow(), grow())
        v = rng.integers(0, 256, size=shape, dtype=np.uint8)
        if case % 4:
            continue
        sset = ct.encode_slicemaps(ct.Volume(v.copy()), ct.SlicemapScheme(s, g * s, g, maps))
        ref = O.encode_slicemaps(v, (s, g * s, g, maps))
        assert np.array_equal(np.stack(sset.atlases), np.stack(ref)), case
        assert np.array_equal(ct.decode_slicemaps(sset).voxels, O.decode_slicemaps(ref, (s, g * s, g, maps))), case
    # fp64 renders (render.py:125-236): every case of the GPU sweep
    rng = np.random.default_rng(404)
    for case in range(24):
        shape = tuple(int(x) for x in rng.integers(6, 36, size=3))
        vol = np.clip(np.rint(rng.normal(70, 60, shape)), 0, 255).astype(np.uint8)
        if case % 3 == 0:
            vol[vol < 90] = 0
        az = float(rng.choice([0.0, 90.0, 180.0, 270.0])) if case % 6 == 0 else float(rng.uniform(0, 360))
        dim, steps = int(rng.integers(16, 40)), int(rng.integers(32, 100))
        mode = "surface" if case % 2 == 0 else "additive"
        thr, gain = int(rng.integers(1, 200)), float(rng.choice([1.0, 4.0, 7.5]))
        ref = ct.render_view(ct.Volume(vol.copy()), ct.ViewParams(azimuth_deg=az, image_dim=dim, steps=steps, mode=mode,
                                                                  threshold=thr, gain=gain))
        assert np.array_equal(O.render_view(vol, az, dim, steps, mode, thr, gain), ref), (case, shape, az, mode)


def test_oracle_composition_equals_live_reference_on_the_fused_sweep():
    """The u8 cases of test_gpu_parity.py::test_preview_random_sweep (same generator, same seeds)
    through ctprev's own functions, composed as SURVEY s8(d) / pipeline.py:215-237, 275 compose
    them -- volume_histogram, artifact_bins, filter_histogram_bins, _scheme_volume +
    _pad_to_cube, encode_slicemaps -- against the oracle's ``preview_pipeline``, which is what the
    fused GPU pass is compared with."""
    ct = _live_reference()
    from ctprev.pipeline import _pad_to_cube, _scheme_volume
    import importlib.util
    spec = importlib.util.spec_from_file_location("_gpu_parity", ROOT / "tests" / "test_gpu_parity.py")
    mod = importlib.util.module_from_spec(spec)
    spec.loader.exec_module(mod)  # the GPU sweep's own generator
    _random_volume = mod._random_volume
    for case in range(18):
        rng = np.random.default_rng(1000 + case)
        dtype = np.uint8 if case % 3 else np.uint16
        if case < 12:
            dims = [int(rng.choice([16, 24, 32, 48, 64, 80, 96, 128])) for _ in range(3)]
            if case % 4 == 3:
                dims[2] += int(rng.integers(1, 8))
        else:
            dims = [int(rng.integers(3, 9)), int(rng.integers(1, 9)), int(rng.choice([1, 5, 8, 16, 17]))]
        shape = tuple(dims)
        vox, _ = _random_volume(rng, dtype, shape)
        if dtype != np.uint8:
            continue  # the reference rejects uint16 (volume.py:56-57): the extension stays oracle-only
        big = max(shape)
        sch = []
        sizes = [8, 12, 16, 24, 32, 40, 64, 96, 128] if case < 12 else [1, 2, 3, 4, 6, 8]
        for s in sorted({int(x) for x in rng.choice(sizes, 3)}, reverse=True):
            if s > big:
                continue
            g = int(rng.choice([1, 2, 3, 4, 5, 8]))
            sch.append((s, g * s, g, -(-s // (g * g))))
        if not sch:
            sch = [(1, 2, 2, 1)]
        hist, bins, f, levels, atl = O.preview_pipeline(vox, [s[0] for s in sch], schemes=sch)
        v = ct.Volume(vox.copy())
        assert np.array_equal(ct.volume_histogram(v).bins, hist), case
        rb = ct.artifact_bins(v)
        assert rb == bins, case
        rf = ct.filter_histogram_bins(v, rb)
        assert np.array_equal(rf.voxels, f), case
        for (s, a, g, m), lv, at in zip(sch, levels, atl):
            rl = _scheme_volume(rf, s)
            assert np.array_equal(rl.voxels, lv), (case, s)
            sset = ct.encode_slicemaps(_pad_to_cube(rl, s), ct.SlicemapScheme(s, a, g, m))
            assert np.array_equal(np.stack(sset.atlases), np.stack(at)), (case, s)


def test_slice_cells_equal_the_viewer_parity_fixture():
    """frontend/tests/fixtures/parity.json (every slice -> (map, cx, cy) for the planned schemes
    128 / 256 / 512): the mirror's ``slice_cell`` (slicemap.py:79-85) and the
    oracle's atlas layout agree with every entry.  Read from the mounted reference (skipped where
    it is absent; the fixture is not copied)."""
    import json
    import paper_2311_15038_b200 as P
    fx = Path("/root/reference/pkg/frontend/tests/fixtures/parity.json")
    if not fx.is_file():
        pytest.skip("the reference's frontend fixtures are not mounted")
    table = json.loads(fx.read_text())
    for key, cells in table.items():
        s = int(key)
        scheme = P.plan_scheme(s)
        assert len(cells) == s
        for k, (m, cx, cy) in enumerate(cells):
            assert P.slice_cell(k, scheme) == (m, cx, cy), (s, k)
        sc = O.plan_scheme(s)
        g = sc[2]
        for k in (0, 1, g - 1, g, g * g - 1, g * g, s - 1):
            m, cx, cy = cells[k]
            vol = np.zeros((s, s, s), np.uint8)
            vol[k, 3, 5] = 200
            atl = O.encode_slicemaps(vol, sc)
            # a single voxel of slice k lands in that cell of that map, and nowhere else
            assert atl[m][cy * s + 3, cx * s + 5] == 200 and int(np.stack(atl).astype(np.int64).sum()) == 200, (s, k)
