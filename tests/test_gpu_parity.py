"""Parity of the CUDA path (through the C ABI) against the reference's golden
vectors and the CPU oracle.  Bit-exact for histograms, bins, filtered voxels,
levels, atlases and the fp64 reference render modes; MIP / alpha (fp32
extension path) within max-abs 1 (= 1/255) per channel."""
from __future__ import annotations

import numpy as np
import pytest
import torch

from oracle import ctp_oracle as O

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def P(cuda):
    import paper_2311_15038_b200 as P
    return P


# ---------------------------------------------------------------- golden (reference outputs)

def test_hist_golden(P, golden):
    for i in range(int(golden["hist_n"])):
        zr = tuple(int(x) for x in golden[f"hist{i}_z"])
        zr = None if zr == (-1, -1) else zr
        h = P.volume_histogram(P.Volume(golden[f"hist{i}_in"]), zr)
        assert h.bins.dtype == np.int64 and np.array_equal(h.bins, golden[f"hist{i}_out"]), i


def test_artifact_filter_golden(P, golden):
    for i in range(int(golden["art_n"])):
        v = P.Volume(golden[f"art{i}_in"])
        bins = P.artifact_bins(v, n_top=int(golden[f"art{i}_ntop"]), frac=float(golden[f"art{i}_frac"]))
        assert sorted(bins) == golden[f"art{i}_bins"].tolist(), i
        assert np.array_equal(P.filter_histogram_bins(v, bins).voxels, golden[f"art{i}_filtered"]), i


def test_downscale_golden(P, golden):
    for i in range(int(golden["ds_n"])):
        out = P.downscale_volume(P.Volume(golden[f"ds{i}_in"]), tuple(int(t) for t in golden[f"ds{i}_target"]))
        assert np.array_equal(out.voxels, golden[f"ds{i}_out"]), i


def test_encode_golden(P, golden):
    for i in range(int(golden["enc_n"])):
        s, a, g, m = (int(x) for x in golden[f"enc{i}_scheme"])
        sset = P.encode_slicemaps(P.Volume(golden[f"enc{i}_in"]), P.SlicemapScheme(s, a, g, m))
        assert np.array_equal(np.stack(sset.atlases), golden[f"enc{i}_out"]), i
        back = P.decode_slicemaps(sset)
        assert np.array_equal(np.stack(P.encode_slicemaps(back, sset.scheme).atlases), golden[f"enc{i}_out"])


def test_encode_decode_seeded_sweep_custom_schemes(P):
    """40 seeded custom schemes (slicemap.py:52-61 validates grid * s == atlas_dim and map_count ==
    ceil(s / grid^2); custom schemes are legal, test_slicemap.py:112): grids 1..9 incl. non-powers
    of two, s with and without 16-byte rows, partial last maps, volumes at s^3 and larger on some
    axes (downscale first, slicemap.py:130) -- encode equals the oracle byte for byte, decode
    inverts it, and a volume smaller than s on any axis raises InvalidTarget."""
    rng = np.random.default_rng(77)
    for case in range(40):
        g = int(rng.integers(1, 10))
        s = int(rng.choice([8, 12, 16, 20, 24, 32, 33, 40, 48, 64]))
        maps = -(-s // (g * g))
        scheme = P.SlicemapScheme(s, g * s, g, maps)
        grow = lambda: int(s if rng.random() < 0.5 else s + rng.integers(1, s + 1))  # noqa: E731
        shape = (grow(), grow(), grow())
        v = rng.integers(0, 256, size=shape, dtype=np.uint8)
        sset = P.encode_slicemaps(P.Volume(v), scheme)
        ref = O.encode_slicemaps(v, (s, g * s, g, maps))
        assert len(sset.atlases) == maps
        assert np.array_equal(np.stack(sset.atlases), np.stack(ref)), (case, s, g, shape)
        assert np.array_equal(P.decode_slicemaps(sset).voxels, O.decode_slicemaps(ref, (s, g * s, g, maps))), (case, s, g)
    small = P.Volume(np.zeros((16, 16, 12), np.uint8))
    with pytest.raises(P.InvalidTarget):
        P.encode_slicemaps(small, P.SlicemapScheme(16, 64, 4, 1))


def test_render_golden_bit_exact(P, golden):
    for i in range(int(golden["rv_n"])):
        az, dim, steps, add, thr = golden[f"rv{i}_params"]
        vol = P.Volume(golden[bytes(golden[f"rv{i}_vol"]).decode()])
        img = P.render_view(vol, P.ViewParams(azimuth_deg=az, image_dim=int(dim), steps=int(steps),
                                              mode="additive" if add else "surface", threshold=int(thr)))
        assert img.shape == (int(dim), int(dim)) and img.dtype == np.uint8
        assert np.array_equal(img, golden[f"rv{i}_out"]), (i, int(np.abs(img.astype(int) - golden[f"rv{i}_out"]).max()))


def test_render_fp64_seeded_sweep_bit_exact(P):
    """24 seeded views of random anisotropic volumes in the reference's two modes (render.py:125-202):
    random azimuths incl. the axis-aligned ones, image sizes, step counts, thresholds and gains --
    bit-identical to the oracle's numba-order restatement (which is pinned to the reference's own
    renders), through the byte-load path and the texture-gather path alike."""
    import os
    rng = np.random.default_rng(404)
    for case in range(24):
        shape = tuple(int(x) for x in rng.integers(6, 36, size=3))
        vol = np.clip(np.rint(rng.normal(70, 60, shape)), 0, 255).astype(np.uint8)
        if case % 3 == 0:
            vol[vol < 90] = 0  # sparse: long empty stretches before the first hit
        az = float(rng.choice([0.0, 90.0, 180.0, 270.0])) if case % 6 == 0 else float(rng.uniform(0, 360))
        dim, steps = int(rng.integers(16, 40)), int(rng.integers(32, 100))
        mode = "surface" if case % 2 == 0 else "additive"
        thr, gain = int(rng.integers(1, 200)), float(rng.choice([1.0, 4.0, 7.5]))
        p = P.ViewParams(azimuth_deg=az, image_dim=dim, steps=steps, mode=mode, threshold=thr, gain=gain)
        ref = O.render_view(vol, az, dim, steps, mode, thr, gain)
        for force in ("0", "1"):  # byte loads / texture gathers
            os.environ["CTP_RENDER_FP64_TEX"] = force
            try:
                img = P.render_view(P.Volume(vol), p)
            finally:
                del os.environ["CTP_RENDER_FP64_TEX"]
            assert np.array_equal(img, ref), (case, shape, az, dim, steps, mode, thr, gain, force)


def test_entropy_and_snapshot_golden(P, golden):
    for i in range(int(golden["ent_n"])):
        assert P.image_entropy(golden[f"ent{i}_in"]).entropy == float(golden[f"ent{i}_h"])
    snap = P.optimal_snapshot(P.Volume(golden["lphantom"]), n_views=12,
                              params=P.ViewParams(image_dim=128, steps=64, threshold=60))
    assert snap.azimuth_deg == 300.0 == float(golden["snap_az"])       # test_render.py:178
    assert snap.entropy == float(golden["snap_h"])                       # bit-identical H
    assert np.array_equal(np.array(snap.per_view), golden["snap_per_view"])
    assert np.array_equal(snap.image, golden["snap_img"])


def test_symmetric_cylinder_reports_zero(P, golden):
    snap = P.optimal_snapshot(P.Volume(golden["cylinder"]), n_views=4,
                              params=P.ViewParams(image_dim=128, steps=64, threshold=60))
    ents = [h for _, h in snap.per_view]
    assert max(ents) - min(ents) <= 1e-6 and snap.azimuth_deg == 0.0    # test_render.py:181-193


# ---------------------------------------------------------------- oracle, seeded inputs

@pytest.mark.parametrize("shape", [(1, 1, 1), (2, 3, 5), (17, 33, 65), (64, 64, 64), (3, 1000, 1001)])
def test_hist_random(P, shape):
    rng = np.random.default_rng(sum(shape))
    v = rng.integers(0, 256, size=shape, dtype=np.uint8)
    assert np.array_equal(P.volume_histogram(P.Volume(v)).bins, O.histogram(v))
    if shape[0] > 2:
        assert np.array_equal(P.volume_histogram(P.Volume(v), (1, shape[0] - 1)).bins, O.histogram(v, (1, shape[0] - 1)))


def test_hist_skewed_and_constant(P):
    for v in (np.full((32, 64, 64), 7, np.uint8),
              np.clip(np.rint(np.random.default_rng(1).normal(20, 6, (40, 96, 96))), 0, 255).astype(np.uint8)):
        assert np.array_equal(P.volume_histogram(P.Volume(v)).bins, O.histogram(v))


def test_hist_u16_device(P, cuda):
    from paper_2311_15038_b200 import device as dev
    rng = np.random.default_rng(3)
    v = rng.integers(0, 5000, size=(9, 31, 77)).astype(np.uint16)
    h = dev.hist_u16(torch.from_numpy(v).to(cuda)).cpu().numpy()
    assert np.array_equal(h, O.histogram_u16(v))


def test_lut_apply_u16_any_length(P, cuda):
    """ctp_lut_apply_u16: filter o rescale + 4096-bin histogram for any element count
    and offset (incl. values above 4095, which saturate into the last bin)."""
    from paper_2311_15038_b200 import device as dev
    rng = np.random.default_rng(41)
    bins = frozenset({0, 17, 400, 401, 4095})
    lut = O.lut_u16(bins)
    for n in (1, 7, 8, 9, 1000, 65537):
        v = rng.integers(0, 70000, size=n + 3).astype(np.uint16)[3:]      # odd start offset on the device too
        src = torch.from_numpy(np.ascontiguousarray(v)).to(cuda)
        hist = torch.zeros(4096, dtype=torch.int64, device=cuda)
        out = dev.lut_apply_u16(src, torch.from_numpy(lut).to(cuda), hist=hist).cpu().numpy()
        assert np.array_equal(out, lut[np.minimum(v, 4095)]), n
        assert np.array_equal(hist.cpu().numpy(), O.histogram_u16(v)), n
    full = torch.from_numpy(rng.integers(0, 4096, size=1001).astype(np.uint16)).to(cuda)
    odd = full[1:]                                                         # a 2-byte-aligned view
    out = dev.lut_apply_u16(odd, torch.from_numpy(lut).to(cuda)).cpu().numpy()
    assert np.array_equal(out, lut[odd.cpu().numpy()])


def test_filter_unaligned_lengths(P):
    rng = np.random.default_rng(4)
    for shape in [(1, 1, 17), (3, 7, 11), (5, 64, 65)]:
        v = rng.integers(0, 256, size=shape, dtype=np.uint8)
        bins = {0, 3, 77, 255}
        assert np.array_equal(P.filter_histogram_bins(P.Volume(v), bins).voxels, O.filter_histogram_bins(v, bins))


def test_downscale_random_ratios(P):
    rng = np.random.default_rng(5)
    for shape, target in [((30, 40, 50), (25, 20, 15)), ((64, 64, 64), (32, 32, 32)), ((64, 64, 64), (8, 8, 8)),
                          ((32, 48, 64), (4, 3, 2)), ((96, 160, 160), (128, 128, 96)), ((33, 17, 9), (9, 17, 33))]:
        v = rng.integers(0, 256, size=shape, dtype=np.uint8)
        assert np.array_equal(P.downscale_volume(P.Volume(v), target).voxels, O.downscale(v, target)), (shape, target)


def test_downscale_vector_path_general_ratios(P, cuda):
    """16-byte rows take the column-sum kernel (packed 16-bit lanes); incl. cells of
    up to 16x16 source rows (255 * 256 per lane) and extreme x ratios."""
    from paper_2311_15038_b200 import device as dev
    rng = np.random.default_rng(9)
    # targets are (tx, ty, tz), shapes (nz, ny, nx) as everywhere in the reference
    for shape, target in [((40, 36, 64), (37, 23, 17)), ((64, 48, 160), (128, 7, 5)), ((256, 256, 32), (2, 16, 16)),
                          ((16, 16, 4096), (999, 16, 1)), ((33, 70, 4096), (999, 3, 1)), ((17, 255, 48), (48, 16, 17)),
                          ((8, 8, 16384), (5000, 8, 8)),
                          # the warp-per-row kernel's x-cell classes: <= 2 (1.5:1 / 1.33:1, config 5), <= 4, <= 8
                          ((64, 48, 96), (64, 32, 32)), ((48, 40, 1024), (768, 30, 36)), ((40, 24, 320), (94, 7, 13)),
                          ((24, 20, 256), (37, 20, 24))]:
        v = rng.integers(0, 256, size=shape, dtype=np.uint8)
        v[:, :, :16] = 255  # saturated columns: the packed lanes at their maximum
        got = dev.downscale(torch.from_numpy(v).to(cuda), target).cpu().numpy()
        assert np.array_equal(got, O.downscale(v, target)), (shape, target)


def test_downscale_seeded_sweep_every_kernel_path(P, cuda):
    """80 seeded random (shape, target) pairs through ctp_downscale_u8 against the oracle's
    volume.py:277-309 restatement, bit for bit: rows that are whole 16-byte vectors (the
    warp-per-row kernel with x cells <= 2 / 4 / 8 / 16, and the column-sum kernel beyond) and rows
    that are not (the byte kernel); targets from 1 to n per axis incl. identity axes; random,
    saturated (the packed 16-bit lanes and the magic-multiplier rounding at their maxima) and
    sparse data."""
    from paper_2311_15038_b200 import device as dev
    rng = np.random.default_rng(2025)
    for case in range(80):
        if case % 4 == 3:   # rows that are not whole vectors
            nx = int(rng.integers(1, 90))
        else:
            nx = 16 * int(rng.integers(1, 40))
        ny, nz = int(rng.integers(1, 48)), int(rng.integers(1, 40))
        pick = lambda n: int(n if rng.random() < 0.15 else rng.integers(1, n + 1))  # noqa: E731
        if case % 5 == 0:   # wide x cells (>= 16 columns per output)
            tx = max(1, nx // int(rng.integers(16, 40)))
        else:
            tx = pick(nx)
        target = (tx, pick(ny), pick(nz))
        kind = case % 3
        if kind == 0:
            v = rng.integers(0, 256, size=(nz, ny, nx), dtype=np.uint8)
        elif kind == 1:
            v = np.full((nz, ny, nx), 255, np.uint8)
            v[rng.random((nz, ny, nx)) < 0.1] = 254
        else:
            v = (rng.random((nz, ny, nx)) < 0.07).astype(np.uint8) * rng.integers(1, 256, size=(nz, ny, nx), dtype=np.uint8)
        if target == (nx, ny, nz):
            continue  # identity is the host's shortcut (volume.py:290-291)
        got = dev.downscale(torch.from_numpy(v).to(cuda), target).cpu().numpy()
        assert np.array_equal(got, O.downscale(v, target)), (case, v.shape, target)


def test_errors_match_reference(P):
    v = P.Volume(np.zeros((4, 4, 4), np.uint8))
    with pytest.raises(P.InvalidTarget):
        P.downscale_volume(v, (4, 4, 8))
    with pytest.raises(P.InvalidTarget):
        P.downscale_volume(v, (0, 4, 4))
    with pytest.raises(P.RangeOutOfBounds):
        P.volume_histogram(v, (2, 2))
    with pytest.raises(P.RangeOutOfBounds):
        P.artifact_bins(v, n_top=0)
    with pytest.raises(P.RangeOutOfBounds):
        P.artifact_bins(v, frac=-0.1)
    with pytest.raises(P.RangeOutOfBounds):
        P.filter_histogram_bins(v, {256})
    with pytest.raises(P.InvalidTarget):
        P.encode_slicemaps(v, 128)      # smaller than the scheme (slicemap.py:130)
    with pytest.raises(P.UnsupportedScheme):
        P.encode_slicemaps(v, 100)
    with pytest.raises(P.RangeOutOfBounds):
        P.image_entropy(np.zeros((4, 4, 4), np.uint8))
    with pytest.raises(P.RangeOutOfBounds):
        P.optimal_snapshot(v, n_views=0)


# ---------------------------------------------------------------- fused pipeline (kernels 1-4)

def _synth_host(spec):
    from paper_2311_15038_b200 import synth
    return synth.generate(spec).cpu().numpy()


def _check_preview(P, vox, schemes, keep_filtered=False):
    res = P.preview_pipeline(vox, schemes=schemes, keep_filtered=keep_filtered)
    sch = [(sc.s, sc.atlas_dim, sc.grid, sc.map_count) if not isinstance(sc, int) else O.plan_scheme(sc)
           for sc in schemes]
    hist, bins, f, levels, atl = O.preview_pipeline(vox, [s[0] for s in sch], schemes=sch)
    assert np.array_equal(res.histogram, hist)
    assert res.bins == bins
    for s, a in zip(sch, atl):
        got = np.stack(res.slicemaps[s[0]].atlases)
        assert np.array_equal(got, np.stack(a)), s
    if keep_filtered:
        assert np.array_equal(res.filtered.voxels, f)
    return res


def test_preview_c1_full_size(P):
    """Config 1 exactly: 256^3 u8 seed 0, 3 shells; one 16x16-grid 4096^2 atlas."""
    from paper_2311_15038_b200 import synth
    vox = _synth_host(synth.config("c1"))
    _check_preview(P, vox, [P.SlicemapScheme(256, 4096, 16, 1)], keep_filtered=True)


def test_preview_four_levels_512(P):
    """Levels 1..4 of a 512^3 volume (planned 256/128 + custom 64/32 schemes) in one pass."""
    from paper_2311_15038_b200 import synth
    vox = _synth_host(synth.small((512, 512, 512), seed=7, n_shells=6))
    _check_preview(P, vox, [256, 128, P.SlicemapScheme(64, 512, 8, 1), P.SlicemapScheme(32, 256, 8, 1)])


def test_preview_anisotropic_and_general(P):
    """Non-cubic: power-of-two levels fused; a 1.5:1 level via the general path; padding."""
    from paper_2311_15038_b200 import synth
    vox = _synth_host(synth.small((96, 192, 160), seed=8))       # nz, ny, nx
    _check_preview(P, vox, [128, P.SlicemapScheme(96, 768, 8, 2), P.SlicemapScheme(48, 384, 8, 1)],
                   keep_filtered=True)


def test_preview_u16_extension(P):
    from paper_2311_15038_b200 import synth
    vox = _synth_host(synth.small((64, 128, 128), dtype="u16", seed=9))
    res = _check_preview(P, vox, [128, P.SlicemapScheme(64, 512, 8, 1), P.SlicemapScheme(32, 256, 8, 1)],
                         keep_filtered=True)
    assert res.histogram.shape == (4096,)


def test_preview_c2_full_size(P):
    """Config 2 exactly (1024^3 u8, 12 shells, 1% speckle): hist, bins and all three
    levels' atlases bit-exact against the oracle composition."""
    from paper_2311_15038_b200 import synth
    vox = _synth_host(synth.config("c2"))
    _check_preview(P, vox, [512, 256, 128])


def _random_volume(rng, dtype, shape):
    """Seeded data of one of several shapes of histogram: narrow normal, uniform,
    few distinct values, mostly zero, saturated (u16: incl. values above 4095)."""
    n = int(np.prod(shape))
    kind = int(rng.integers(0, 5))
    top = 255 if dtype == np.uint8 else 4095
    if kind == 0:
        v = rng.normal(top * 0.1, top * 0.03, n)
    elif kind == 1:
        v = rng.integers(0, top + 1, n)
    elif kind == 2:
        v = rng.choice(rng.integers(0, top + 1, 5), n)
    elif kind == 3:
        v = np.where(rng.random(n) < 0.9, 0, rng.integers(1, top + 1, n))
    else:
        v = np.where(rng.random(n) < 0.5, top, rng.integers(0, top + 1, n))
        if dtype == np.uint16:
            v = np.where(rng.random(n) < 0.05, rng.integers(4096, 65536, n), v)
    hi = 255 if dtype == np.uint8 else 65535
    return np.clip(np.rint(v), 0, hi).astype(dtype).reshape(shape), kind


@pytest.mark.parametrize("case", range(18))
def test_preview_random_sweep(P, case):
    """Seeded sweep of the fused pass against the oracle: u8 / u16, shapes with and
    without 16-byte rows and power-of-two dims (fused vs general path), planned and
    custom schemes incl. non-power-of-two grids (division addressing) and partial
    last maps, and five shapes of histogram (artifact bins flag different sets)."""
    rng = np.random.default_rng(1000 + case)
    dtype = np.uint8 if case % 3 else np.uint16
    if case < 12:
        dims = [int(rng.choice([16, 24, 32, 48, 64, 80, 96, 128])) for _ in range(3)]
        if case % 4 == 3:
            dims[2] += int(rng.integers(1, 8))     # rows not a whole number of vectors
    else:                                          # tiny and degenerate extents (n_top = 3 <= nz)
        dims = [int(rng.integers(3, 9)), int(rng.integers(1, 9)), int(rng.choice([1, 5, 8, 16, 17]))]
    shape = tuple(dims)                        # (nz, ny, nx)
    vox, kind = _random_volume(rng, dtype, shape)
    big = max(shape)
    schemes = []
    sizes = [8, 12, 16, 24, 32, 40, 64, 96, 128] if case < 12 else [1, 2, 3, 4, 6, 8]
    for s in sorted({int(x) for x in rng.choice(sizes, 3)}, reverse=True):
        if s > big:
            continue
        g = int(rng.choice([1, 2, 3, 4, 5, 8]))
        schemes.append(P.SlicemapScheme(s, g * s, g, -(-s // (g * g))))
    if not schemes:
        schemes = [P.SlicemapScheme(1, 2, 2, 1)]
    _check_preview(P, vox, schemes, keep_filtered=bool(case % 2))


@pytest.mark.parametrize("nx", [784, 1008, 1296])
@pytest.mark.parametrize("dtype", [np.uint8, np.uint16])
def test_preview_wide_rows_multibox_tiles(P, cuda, nx, dtype):
    """Rows wider than one TMA box (256 bytes) and not a multiple of it: whole-width
    tiles of several boxes, the last one partly outside the volume (zero-filled),
    with 1, 2, 3 and 4 fused dense levels (the tile planner stacks block rows for
    L <= 2); histogram and every level against the oracle."""
    from paper_2311_15038_b200 import device as dev
    rng = np.random.default_rng(nx)
    vox, _ = _random_volume(rng, dtype, (32, 48, nx))
    if dtype == np.uint8:
        lut, h_ref = O.filter_lut({0, 3, 17, 200}), O.histogram(vox)
        f = O.apply_lut(vox, lut)
    else:
        lut, h_ref = O.lut_u16(frozenset({0, 5, 400, 4095})), O.histogram_u16(vox)
        f = lut[np.minimum(vox, 4095)]
    vol = torch.from_numpy(vox).to(cuda)
    for nlev in (1, 2, 3, 4):
        hist = torch.zeros(h_ref.size, dtype=torch.int64, device=cuda)
        outs = dev.preview(vol, torch.from_numpy(lut).to(cuda), {l: "xyz" for l in range(1, nlev + 1)}, hist=hist)
        assert np.array_equal(hist.cpu().numpy(), h_ref), nlev
        for l in range(1, nlev + 1):
            ref = O.downscale(f, (nx >> l, 48 >> l, 32 >> l))
            assert np.array_equal(outs[l].cpu().numpy(), ref), (nlev, l)


@pytest.mark.parametrize("dtype", [np.uint8, np.uint16])
def test_preview_level0_large_tiles(P, cuda, dtype):
    """Level 0 only on a volume above the small-volume threshold (2^26 voxels): four
    one-row units per thread, 64 KB whole-width tiles of several boxes (the last one
    partly outside the rows); the filtered voxels and the histogram against the oracle."""
    from paper_2311_15038_b200 import device as dev
    rng = np.random.default_rng(64)
    vox, _ = _random_volume(rng, dtype, (64, 1024, 1040))
    if dtype == np.uint8:
        lut, h_ref = O.filter_lut({0, 3, 17, 200}), O.histogram(vox)
        f = O.apply_lut(vox, lut)
    else:
        lut, h_ref = O.lut_u16(frozenset({0, 5, 400, 4095})), O.histogram_u16(vox)
        f = lut[np.minimum(vox, 4095)]
    vol = torch.from_numpy(vox).to(cuda)
    hist = torch.zeros(h_ref.size, dtype=torch.int64, device=cuda)
    outs = dev.preview(vol, torch.from_numpy(lut).to(cuda), {0: "xyz"}, hist=hist)
    assert np.array_equal(hist.cpu().numpy(), h_ref)
    assert np.array_equal(outs[0].cpu().numpy(), f)


def test_preview_repeat_bit_identical(P):
    from paper_2311_15038_b200 import synth
    vox = _synth_host(synth.small((128, 128, 128), seed=10))
    a = P.preview_pipeline(vox, schemes=[128, P.SlicemapScheme(64, 512, 8, 1)])
    b = P.preview_pipeline(vox, schemes=[128, P.SlicemapScheme(64, 512, 8, 1)])
    assert np.array_equal(a.histogram, b.histogram)
    for s in (128, 64):
        assert np.array_equal(np.stack(a.slicemaps[s].atlases), np.stack(b.slicemaps[s].atlases))


# ---------------------------------------------------------------- renderer extensions

TF = ((0.0, 0.0, 0.0, 0.0, 0.0), (40.0, 0.9, 0.2, 0.1, 0.02), (150.0, 1.0, 0.8, 0.5, 0.08),
      (255.0, 1.0, 1.0, 1.0, 0.5))


def test_mip_fp64_exact_and_fp32_within_one(P, golden):
    vol = golden["lphantom"]
    for az in (0.0, 33.0, 250.0):
        ref = O.render_mip(vol, az, 64, 96)
        p = P.ViewParams(azimuth_deg=az, image_dim=64, steps=96, mode="mip")
        g64 = P.render_views(P.Volume(vol), [p], channels=1, fp32=False)[0]
        g32 = P.render_views(P.Volume(vol), [p], channels=1, fp32=True)[0]
        assert np.array_equal(g64, ref)
        assert int(np.abs(g32.astype(int) - ref).max()) <= 1


def test_mip_turntable_opposite_views_rendered_once(P):
    """fp32 MIP turntable: a view and the one at azimuth + 180 degrees are rendered ONCE and stored
    mirrored (csrc/render.cu pair_opposite_views).  Every view -- paired or not, RGBA or gray --
    stays within 1/255 of the oracle's independent render of that view, paired and unpaired
    (CTP_RENDER_MIRROR=0) batches agree within 1, and the exact fp64 path is untouched."""
    import os
    rng = np.random.default_rng(23)
    vol = np.clip(np.rint(rng.normal(40, 25, (44, 52, 60))), 0, 255).astype(np.uint8)
    vol[10:30, 20:40, 15:45] = np.clip(vol[10:30, 20:40, 15:45].astype(int) + 120, 0, 255).astype(np.uint8)
    azs = [0.0, 30.0, 45.0, 180.0, 210.0, 300.0, 120.0, 7.5, 187.5]  # pairs (0,180) (30,210) (300,120) (7.5,187.5); 45 alone
    dim, steps = 56, 150
    ps = [P.ViewParams(azimuth_deg=a, image_dim=dim, steps=steps, mode="mip") for a in azs]
    refs = [O.render_mip(vol, a, dim, steps) for a in azs]
    V = P.Volume(vol)
    for ch in (1, 4):
        paired = P.render_views(V, ps, channels=ch, fp32=True)
        os.environ["CTP_RENDER_MIRROR"] = "0"
        try:
            single = P.render_views(V, ps, channels=ch, fp32=True)
        finally:
            del os.environ["CTP_RENDER_MIRROR"]
        for k, ref in enumerate(refs):
            a = paired[k] if ch == 1 else paired[k][..., 0]
            b = single[k] if ch == 1 else single[k][..., 0]
            assert int(np.abs(a.astype(int) - ref.astype(int)).max()) <= 1, (ch, azs[k])
            assert int(np.abs(b.astype(int) - ref.astype(int)).max()) <= 1, (ch, azs[k])
            assert int(np.abs(a.astype(int) - b.astype(int)).max()) <= 1, (ch, azs[k])
            if ch == 4:
                assert np.array_equal(paired[k][..., 1], a) and np.array_equal(paired[k][..., 2], a)
                assert (paired[k][..., 3] == 255).all()
    # a view's opposite really is its mirror image (what the pairing relies on), in the oracle itself
    assert int(np.abs(refs[0].astype(int) - refs[3][:, ::-1].astype(int)).max()) <= 1
    exact = P.render_views(V, ps, channels=1, fp32=False)
    for k, ref in enumerate(refs):
        assert np.array_equal(exact[k], ref)


def test_alpha_fp64_and_fp32_within_one(P):
    rng = np.random.default_rng(11)
    vol = np.clip(np.rint(rng.normal(60, 40, (40, 48, 56))), 0, 255).astype(np.uint8)
    for az in (10.0, 135.0):
        ref = O.render_alpha(vol, az, 48, 80, TF, 0.99)
        p = P.ViewParams(azimuth_deg=az, image_dim=48, steps=80, mode="alpha", tf=TF)
        g64 = P.render_views(P.Volume(vol), [p], channels=4, fp32=False)[0]
        g32 = P.render_views(P.Volume(vol), [p], channels=4, fp32=True)[0]
        assert np.array_equal(g64, ref)
        assert int(np.abs(g32.astype(int) - ref.astype(int)).max()) <= 1


def test_batched_views_equal_single_views(P, golden):
    vol = P.Volume(golden["lphantom"])
    ps = [P.ViewParams(azimuth_deg=10.0 * k, image_dim=48, steps=64, threshold=60) for k in range(5)]
    batch = P.render_views(vol, ps)
    for k, p in enumerate(ps):
        assert np.array_equal(batch[k], O.render_view(golden["lphantom"], p.azimuth_deg, 48, 64, "surface", 60))


# ---------------------------------------------------------------- config 3 at full size (16 GiB)

# Full-size configs 3 and 5 are checked against the oracle on EVERY atlas byte:
# the source is copied to the host once and the oracle runs chunk by chunk on a
# fork pool (levels are separable on slabs of whole 2^L cells, volume.py:265-309;
# histograms of slabs sum), so it never needs the whole filtered volume at once.
_SRC = None   # host copy of the source volume, inherited by the forked workers
_LUT = None


def _chunk_levels(args):
    z0, z1, nlev = args
    v = _SRC[z0:z1]
    h = O.histogram_u16(v)
    f = _LUT[np.minimum(v, 4095)]                                   # filter o rescale (DESIGN s4)
    cz, ny, nx = f.shape
    return z0, h, [O.downscale(f, (nx >> l, ny >> l, cz >> l)) for l in range(1, nlev + 1)]  # volume.py:277-309


def _chunked_oracle(vol_t, nlev: int, chunk: int = 16):
    """(hist, bins, lut, {l: level}) of a 12-bit volume, every level direct from the
    filtered full-resolution voxels (pipeline.py:275), computed in z-chunks."""
    import multiprocessing as mp
    import os
    global _SRC, _LUT
    _SRC = vol_t.cpu().numpy()
    nz, ny, nx = _SRC.shape
    bins = O.artifact_bins_u16(_SRC[nz - 3:])                      # mask.py:215-231 over 4096 bins
    _LUT = O.lut_u16(bins)
    levels = {l: np.empty((nz >> l, ny >> l, nx >> l), np.uint8) for l in range(1, nlev + 1)}
    hist = np.zeros(4096, np.int64)
    try:
        with mp.get_context("fork").Pool(os.cpu_count() or 4) as pool:
            for z0, h, lv in pool.imap_unordered(_chunk_levels, [(z, z + chunk, nlev) for z in range(0, nz, chunk)]):
                hist += h
                for l, a in zip(range(1, nlev + 1), lv):
                    levels[l][z0 >> l:(z0 >> l) + a.shape[0]] = a
    finally:
        _SRC = None
    return hist, bins, _LUT, levels


def test_preview_c3_full_size_every_atlas_byte(P, cuda):
    """Config 3 exactly (2048^3 12-bit u16, 16 GiB): 4096-bin histogram, artifact LUT
    and EVERY byte of all four levels' atlases (1024: 64 maps of 4x4 4096^2; planned
    512/256/128) against the chunked oracle."""
    import torch
    from paper_2311_15038_b200 import synth
    from paper_2311_15038_b200.device import AtlasSpec
    from paper_2311_15038_b200.pipeline import plan_preview, run_preview

    spec = synth.config("c3")
    vol = synth.generate(spec, device=cuda)
    schemes = {1024: AtlasSpec(1024, 4096, 4, 64), 512: AtlasSpec(512, 4096, 8, 8),
               256: AtlasSpec(256, 2048, 8, 4), 128: AtlasSpec(128, 1024, 8, 2)}
    plan = plan_preview(spec.shape, schemes)
    assert not plan.general and plan.nlev == 4
    res = run_preview(vol, plan)
    got = {s: res.atlases[s].cpu().numpy() for s in schemes}
    got_hist, got_lut = res.hist.cpu().numpy(), res.lut.cpu().numpy()
    del res
    hist, bins, lut, levels = _chunked_oracle(vol, 4)
    del vol
    torch.cuda.empty_cache()
    assert np.array_equal(got_hist, hist)
    assert np.array_equal(got_lut, lut)
    for s, l in plan.scheme_level.items():
        sp = schemes[s]
        want = np.stack(O.encode_slicemaps(O.pad_to_cube(levels[l], s), (sp.s, sp.atlas_dim, sp.grid, sp.map_count)))
        assert np.array_equal(got[s], want), s


def test_artifact_lut_single_launch(P, cuda):
    """ctp_artifact_lut == ctp_hist + ctp_lut_build, and leaves its workspace zero
    (repeated calls, u8 and u16, several n_top / frac)."""
    from paper_2311_15038_b200 import device as dev
    rng = np.random.default_rng(12)
    v8 = np.clip(np.rint(rng.normal(20, 6, (12, 96, 80))), 0, 255).astype(np.uint8)
    v8[-2:, :10, :10] = 200
    v16 = np.clip(np.rint(rng.normal(400, 120, (10, 64, 64))), 0, 4095).astype(np.uint16)
    for vox, n_tops in ((v8, (1, 3, 12)), (v16, (1, 3))):
        t = torch.from_numpy(vox).to(cuda)
        for n_top in n_tops:
            for frac in (0.0005, 0.0, 0.01):
                hist = torch.full((256 if vox.dtype == np.uint8 else 4096,), 7, dtype=torch.int64, device=cuda)
                lut, flags = dev.artifact_lut_fused(t, n_top, frac, zero_hist=hist)
                if vox.dtype == np.uint8:
                    bins = O.artifact_bins(vox, n_top, frac)
                    want = O.filter_lut(bins)
                else:
                    bins = O.artifact_bins_u16(vox, n_top, frac)
                    want = O.lut_u16(bins)
                assert np.array_equal(lut.cpu().numpy(), want)
                assert set(np.nonzero(flags.cpu().numpy())[0].tolist()) == set(bins)
                assert int(hist.abs().sum().item()) == 0
    for ws in dev._WORKSPACES.values():
        assert int(ws.abs().sum().item()) == 0


def test_artifact_lut_unaligned_top_slab(P, cuda):
    from paper_2311_15038_b200 import device as dev
    rng = np.random.default_rng(13)
    vox = rng.integers(0, 6, size=(5, 7, 11), dtype=np.uint8)   # 77-byte slices: unaligned top slab
    lut, _ = dev.artifact_lut_fused(torch.from_numpy(vox).to(cuda), 3, 0.01)
    assert np.array_equal(lut.cpu().numpy(), O.filter_lut(O.artifact_bins(vox, 3, 0.01)))
    res = P.preview_pipeline(vox, schemes=[P.SlicemapScheme(8, 32, 4, 1)])
    hist, bins, _, _, atl = O.preview_pipeline(vox, [8], schemes=[(8, 32, 4, 1)])
    assert np.array_equal(res.histogram, hist) and res.bins == bins
    assert np.array_equal(np.stack(res.slicemaps[8].atlases), np.stack(atl[0]))


# ---------------------------------------------------------------- preview builders (SURVEY s8 f)

@pytest.fixture(scope="module")
def golden_dp():
    from pathlib import Path
    with np.load(Path(__file__).resolve().parent / "golden" / "ref_golden_datapreview.npz") as z:
        return {k: z[k] for k in z.files}


def test_build_data_preview_golden(P, golden_dp):
    """pipeline.py:240-257 (reference outputs on two mounted phantoms, incl. a 272->256 general ratio)."""
    for i in range(int(golden_dp["dp_n"])):
        dp = P.build_data_preview(P.Volume(golden_dp[f"dp{i}_in"]))
        assert list(dp.filtered_bins) == golden_dp[f"dp{i}_bins"].tolist(), i
        assert np.array_equal(np.stack(dp.slicemaps.atlases), golden_dp[f"dp{i}_atlases"]), i
        assert dp.stages == ("slicemaps_conversion", "histogram_filtering")


def test_acceptance_snapshot_36_views(P, golden, golden_dp):
    """test_acceptance.py:217-244: 36 views, 256^2, 256 steps -> azimuth 250.0, H = 0.840239."""
    snap = P.optimal_snapshot(P.Volume(golden["lphantom"]), n_views=36,
                              params=P.ViewParams(image_dim=256, steps=256, mode="surface", threshold=60))
    assert snap.azimuth_deg == 250.0 == float(golden_dp["acc_snap_az"])
    assert snap.entropy == float(golden_dp["acc_snap_h"]) and abs(snap.entropy - 0.840239) <= 1e-5
    assert np.array_equal(np.array(snap.per_view), golden_dp["acc_snap_per_view"])
    assert np.array_equal(snap.image, golden_dp["acc_snap_img"])


# ---------------------------------------------------------------- config 5 stream (extension)

def _c5_expected(levels, ps):
    """Per level: _scheme_volume (any ratio) + _pad_to_cube + encode (pipeline.py:215-237,
    slicemap.py:120-142) with the stream's planned scheme."""
    out = {}
    for l, sp in ps.levels.items():
        tx, ty, tz = ps.targets[l]
        src = O.downscale(levels[l], (tx, ty, tz))
        out[l] = np.stack(O.encode_slicemaps(O.pad_to_cube(src, sp.s), (sp.s, sp.atlas_dim, sp.grid, sp.map_count)))
    return out


def test_stream_c5_shape_reduced(P, cuda):
    """Config-5 processing at reduced scale (u16 anisotropic, planned schemes, levels
    -> padded atlases, 6-view MIP strip) against the oracle: histogram, LUT and every
    atlas bit-exact, thumbnails within 1/255; and round 1's pow2-1024 variant."""
    from paper_2311_15038_b200 import synth
    from paper_2311_15038_b200.stream import PreviewStream, scheme_pow2
    spec = synth.small((256, 192, 192), dtype="u16", seed=21, n_shells=4)
    vol = synth.generate(spec, device=cuda)
    vox = vol.cpu().numpy()
    hist, bins, f, _, _ = O.preview_pipeline(vox, [])
    nz, ny, nx = vox.shape
    levels = {l: O.downscale(f, (nx >> l, ny >> l, nz >> l)) for l in range(1, 5)}
    for variant in ("scheme", "pow2-1024"):
        ps = PreviewStream(spec.shape, torch.uint16, thumb_dim=64, n_views=6, device=cuda, variant=variant)
        res = ps.process(vol)
        assert np.array_equal(res.hist.cpu().numpy(), hist)
        assert set(np.nonzero(res.flags.cpu().numpy())[0].tolist()) == set(bins)
        for l, want in _c5_expected(levels, ps).items():
            assert np.array_equal(res.atlases[l].cpu().numpy(), want), (variant, l)
        thumb_src = levels[ps.thumb_level]
        assert ps.thumb_shape == thumb_src.shape
        for k, view in enumerate(ps.views):
            ref = O.render_mip(thumb_src, view.azimuth_deg, view.image_dim, view.steps)
            got = res.thumbs[k].cpu().numpy()
            assert int(np.abs(got[..., 0].astype(int) - ref).max()) <= 1
            assert (got[..., 3] == 255).all()
    sp = scheme_pow2((1024, 768, 768))
    assert (sp.s, sp.atlas_dim, sp.grid, sp.map_count) == (1024, 4096, 4, 64)


def test_stream_c5_full_shape_every_atlas_byte(P, cuda):
    """Config 5 at its real shape (1536^2 x 2048 12-bit u16, 9 GiB) with SURVEY s8(d)'s
    composition: L1 768^2 x 1024 -> 512^3 through the general 1.5:1 / 2:1 downscale,
    L2..L4 identity + zero pad into the planned 512 / 256 / 128 schemes.  Histogram,
    LUT and EVERY atlas byte against the chunked oracle; the MIP strip's first view on
    sampled rows against the oracle within 1/255."""
    import torch
    from paper_2311_15038_b200 import synth
    from paper_2311_15038_b200.stream import PreviewStream
    spec = synth.config("c5")
    vol = synth.generate(spec, device=cuda)
    ps = PreviewStream(spec.shape, torch.uint16, device=cuda)
    assert {l: sp.s for l, sp in ps.levels.items()} == {1: 512, 2: 512, 3: 256, 4: 128}
    assert ps.targets[1] == (512, 512, 512) and ps.targets[2] == (384, 384, 512)
    res = ps.process(vol)
    got = {l: t.cpu().numpy() for l, t in res.atlases.items()}
    got_hist, got_flags = res.hist.cpu().numpy(), res.flags.cpu().numpy()
    thumbs = res.thumbs.cpu().numpy()
    hist, bins, lut, levels = _chunked_oracle(vol, 4)
    del vol, res
    torch.cuda.empty_cache()
    assert np.array_equal(got_hist, hist)
    assert set(np.nonzero(got_flags)[0].tolist()) == set(bins)
    for l, want in _c5_expected(levels, ps).items():
        assert np.array_equal(got[l], want), l
    v0 = ps.views[0]
    for r0 in (100, 300):
        ref = O.render_mip(levels[ps.thumb_level], v0.azimuth_deg, v0.image_dim, v0.steps, rows=(r0, r0 + 2))
        assert int(np.abs(thumbs[0, r0:r0 + 2, :, 0].astype(int) - ref).max()) <= 1, r0


def test_apply_circle_mask_golden(P, golden_dp):
    """mask.py:194-212 (exact fp64 predicate incl. points on the boundary) + its errors."""
    from types import SimpleNamespace as C
    vol = P.Volume(golden_dp["cm_in"])
    for i in range(int(golden_dp["cm_n"])):
        cx, cy, r, m = golden_dp[f"cm{i}_params"]
        out = P.apply_circle_mask(vol, C(cx=float(cx), cy=float(cy), r=float(r)), margin=float(m))
        assert np.array_equal(out.voxels, golden_dp[f"cm{i}_out"]), i
    with pytest.raises(P.CircleOutOfBounds):
        P.apply_circle_mask(vol, C(cx=63.0, cy=1.0, r=5.0))
    with pytest.raises(P.RangeOutOfBounds):
        P.apply_circle_mask(vol, C(cx=3.0, cy=1.0, r=5.0), margin=1.0)


def test_c4_full_size_rows_vs_oracle(P, cuda):
    """Config 4 at full size (1024^3, 1024^2, 3548 steps, 3 azimuths): sampled image
    rows of the fp32 MIP and alpha paths within 1/255 of the ORACLE (render_mip /
    render_alpha restricted to those rows), the fp64 additive path (the reference's
    own mode) bit-exact to the oracle's render_view on the same rows."""
    import math
    from paper_2311_15038_b200 import device as dev, synth
    spec = synth.config("c4")
    vol = synth.generate(spec, device=cuda)
    vox = vol.cpu().numpy()
    steps = math.ceil(4 * math.sqrt(3.0) / 2.0 * spec.shape[0])
    tf = P.ViewParams(mode="alpha").tf
    rows = ((130, 132), (505, 507), (880, 882))
    for mode in ("mip", "alpha", "additive"):
        views = [P.ViewParams(azimuth_deg=a, image_dim=1024, steps=steps, mode=mode) for a in (0.0, 37.0, 250.0)]
        fp32 = mode != "additive"
        img = dev.render(vol, views, channels=4 if fp32 else 1, fp32=fp32).cpu().numpy()
        for k, v in enumerate(views):
            for r in rows:
                if mode == "mip":
                    ref = O.render_mip(vox, v.azimuth_deg, 1024, steps, rows=r)
                    d = np.abs(img[k, r[0]:r[1], :, 0].astype(int) - ref.astype(int))
                elif mode == "alpha":
                    ref = O.render_alpha(vox, v.azimuth_deg, 1024, steps, tf, 0.99, rows=r)
                    d = np.abs(img[k, r[0]:r[1]].astype(int) - ref.astype(int))
                else:
                    ref = O.render_view(vox, v.azimuth_deg, 1024, steps, "additive", rows=r)
                    d = np.abs(img[k, r[0]:r[1]].astype(int) - ref.astype(int))
                assert int(d.max()) <= (0 if mode == "additive" else 1), (mode, v.azimuth_deg, r, int(d.max()))
    del vol
    torch.cuda.empty_cache()


def test_fp64_texture_gathers_identical_to_byte_loads(P, cuda, monkeypatch):
    """The fp64 (reference-mode) renderer reads the eight voxels of a sample through
    two texture gathers (by default for additive / MIP / alpha batches that walk
    much more than the slab copy; forced here for every mode incl. surface with its
    bisection and gradient); the images must equal the byte-load path bit for bit,
    on odd and anisotropic shapes, whole images and row bands."""
    from paper_2311_15038_b200 import device as dev
    rng = np.random.default_rng(91)
    for shape, dim, steps in [((40, 33, 70), 48, 96), ((17, 90, 50), 64, 100), ((64, 64, 64), 40, 64)]:
        vol = torch.from_numpy(_shell_volume(shape, seed=int(rng.integers(0, 99)))).to(cuda)
        for mode in ("surface", "additive", "mip", "alpha"):
            views = [P.ViewParams(azimuth_deg=float(rng.uniform(0, 360)), image_dim=dim, steps=steps, mode=mode,
                                  threshold=int(rng.integers(60, 200))) for _ in range(3)]
            ch = 4 if mode in ("mip", "alpha") else 1
            for rows in (None, (dim // 4, dim // 4 + 5)):
                monkeypatch.setenv("CTP_RENDER_FP64_TEX", "1")
                a = dev.render(vol, views, channels=ch, fp32=False, rows=rows).cpu().numpy()
                monkeypatch.setenv("CTP_RENDER_FP64_TEX", "0")
                b = dev.render(vol, views, channels=ch, fp32=False, rows=rows).cpu().numpy()
                assert np.array_equal(a, b), (shape, mode, rows)


# ---------------------------------------------------------------- z-slab (sort-last) rendering, empty-space skipping

def _shell_volume(shape, seed=3):
    rng = np.random.default_rng(seed)
    nz, ny, nx = shape
    vol = np.clip(np.rint(rng.normal(20, 6, shape)), 0, 255).astype(np.uint8)
    zz, yy, xx = np.mgrid[:nz, :ny, :nx]
    r = np.sqrt(((zz - nz / 2) / (0.4 * nz)) ** 2 + ((yy - ny / 2) / (0.35 * ny)) ** 2 + ((xx - nx / 2) / (0.4 * nx)) ** 2)
    vol[np.abs(r - 1.0) < 0.08] = 190
    return vol


def test_render_slab_bands_equal_whole_volume(P, cuda):
    """Every mode/precision: the row band rendered from a rank's slab + halo equals the
    same rows rendered from the whole volume bit for bit (sort-last = row-band gather)."""
    from paper_2311_15038_b200 import _lib, device as dev, dist as D
    shape = (72, 60, 84)
    nz = shape[0]
    vt = torch.from_numpy(_shell_volume(shape)).to(cuda)
    dim = 112
    cases = [("surface", 1, False), ("additive", 1, False), ("mip", 1, False), ("mip", 4, True), ("alpha", 4, True),
             ("alpha", 4, False)]
    for world in (2, 3, 5):
        for r in range(world):
            z0, z1 = D.slab_bounds(nz, world, r, 1)
            r0, r1 = D.row_band(shape, dim, z0, z1)
            h0, h1 = D.held_slices(shape, dim, z0, z1)
            if r1 <= r0:
                continue
            for mode, ch, fp32 in cases:
                views = [P.ViewParams(azimuth_deg=a, image_dim=dim, steps=128, mode=mode, threshold=100, tf=TF)
                         for a in (0.0, 123.0)]
                whole = dev.render(vt, views, channels=ch, fp32=fp32, rows=(r0, r1)).cpu().numpy()
                part = dev.render(vt[h0:h1].contiguous(), views, channels=ch, fp32=fp32, rows=(r0, r1), z_base=h0,
                                  full_nz=nz).cpu().numpy()
                assert np.array_equal(whole, part), (world, r, mode, fp32)
    # a slab without its halo is refused, not rendered from missing slices
    z0, z1 = D.slab_bounds(nz, 2, 0, 1)
    r0, r1 = D.row_band(shape, dim, z0, z1)
    views = [P.ViewParams(azimuth_deg=0.0, image_dim=dim, steps=128, mode="mip")]
    with pytest.raises(_lib.NativeError):
        dev.render(vt[z0:z1].contiguous(), views, channels=1, fp32=True, rows=(r0, r1), z_base=z0, full_nz=nz)


def test_alpha_empty_space_skipping_is_exact(P, cuda, monkeypatch):
    """fp32 alpha with block skipping (transfer function 0 below 100) equals the
    unskipped fp32 path bit for bit and the fp64 oracle within 1/255."""
    from paper_2311_15038_b200 import device as dev
    vol = _shell_volume((64, 80, 96), seed=5)
    tf = ((0.0, 0.0, 0.0, 0.0, 0.0), (100.0, 0.5, 0.3, 0.2, 0.0), (180.0, 1.0, 0.8, 0.5, 0.3),
          (255.0, 1.0, 1.0, 1.0, 0.9))
    vt = torch.from_numpy(vol).to(cuda)
    views = [P.ViewParams(azimuth_deg=a, image_dim=96, steps=160, mode="alpha", tf=tf) for a in (0.0, 45.0, 200.0)]
    skip = dev.render(vt, views, channels=4, fp32=True).cpu().numpy()
    monkeypatch.setenv("CTP_RENDER_SKIP", "0")
    noskip = dev.render(vt, views, channels=4, fp32=True).cpu().numpy()
    assert np.array_equal(skip, noskip)
    for k, p in enumerate(views):
        ref = O.render_alpha(vol, p.azimuth_deg, 96, 160, tf, 0.99)
        assert int(np.abs(skip[k].astype(int) - ref.astype(int)).max()) <= 1


def test_build_interactive_preview_golden(P, golden_dp):
    """pipeline.py:267-309 on the device vs the reference on two mounted phantoms and a
    constant volume: masked-level histograms (the Otsu input) bit-exact, thresholds,
    warnings, and every scheme's atlas bytes (SHA-256; the 128 scheme byte for byte).
    The host-side circle detector and Otsu sweep are injected (the reference's circle,
    the oracle's pinned Otsu restatement) -- neither is on the device path."""
    import hashlib
    from pathlib import Path
    from paper_2311_15038_b200 import ops
    from paper_2311_15038_b200.errors import DegenerateHistogram, NoCircleFound
    from paper_2311_15038_b200.types import Circle
    with np.load(Path(__file__).resolve().parent / "golden" / "ref_golden_interactive.npz") as z:
        g = {k: z[k] for k in z.files}
    vols = [golden_dp["dp0_in"], golden_dp["dp1_in"], g["ip_const_in"]]
    for i, v in enumerate(vols):
        c = g[f"ip{i}_circle"]

        def detect(top, c=c):
            assert top.shape == v.shape[1:]
            if np.isnan(c[0]):
                raise NoCircleFound("golden: no circle")
            return Circle(*[float(x) for x in c])

        seen = []

        def otsu(h):
            seen.append(np.asarray(h.bins).copy())
            t = O.otsu_threshold(h.bins)
            if t is None:
                raise DegenerateHistogram("all histogram mass in a single bin")
            return type("R", (), {"value": t})()

        ip = ops.build_interactive_preview(P.Volume(v), detect=detect, threshold=otsu)
        assert ",".join(ip.warnings) == str(g[f"ip{i}_warnings"]), i
        for k, s in enumerate((128, 256, 512)):
            assert np.array_equal(seen[k], g[f"ip{i}_hist{s}"]), (i, s)
            t = ip.thresholds[s]
            assert (-1 if t is None else t) == int(g[f"ip{i}_thr{s}"]), (i, s)
            a = np.stack(ip.slicemaps[s].atlases)
            assert a.shape == tuple(g[f"ip{i}_shape{s}"]), (i, s)
            assert hashlib.sha256(a.tobytes()).hexdigest() == str(g[f"ip{i}_sha{s}"]), (i, s)
        assert np.array_equal(np.stack(ip.slicemaps[128].atlases), g[f"ip{i}_atlas128"]), i


def test_bundles_pixel_parity(P, cuda, tmp_path):
    """The reference's two recorded bundles (fixture-128 and demo-scan-01; make_golden
    re-ran ingest_stack + build_bundle and matched all 27/27 mounted checksums of each):
    our list / data / interactive builders on the ingested volume reproduce every
    product pixel for bit -- thumbnail (+ azimuth, entropy, threshold, mode), data
    atlases + filtered bins, interactive atlases per scheme + thresholds + warnings --
    and our save_slicemaps writes the same manifest and losslessly decodable atlases.
    The host helpers (circle Hough transform, Otsu sweep) are injected: the recorded
    circle, the oracle's pinned Otsu."""
    import json
    from pathlib import Path
    from PIL import Image
    from paper_2311_15038_b200 import ops
    from paper_2311_15038_b200.errors import DegenerateHistogram, NoCircleFound
    from paper_2311_15038_b200.types import Circle
    with np.load(Path(__file__).resolve().parent / "golden" / "ref_golden_bundles.npz") as z:
        g = {k: z[k] for k in z.files}

    def otsu(h):
        t = O.otsu_threshold(h.bins)
        if t is None:
            raise DegenerateHistogram("all histogram mass in a single bin")
        return type("R", (), {"value": t})()

    def detector(c):
        def detect(top):
            if c is None:
                raise NoCircleFound("recorded: no circle")
            return Circle(c["cx"], c["cy"], c["r"], c["votes"])
        return detect

    for i in range(int(g["b_n"])):
        vol = P.Volume(g[f"b{i}_vol"])
        meta = json.loads(str(g[f"b{i}_meta"]))
        side = json.loads(str(g[f"b{i}_sidecar"]))
        # list preview (pipeline.py:157-212)
        lp = ops.build_list_preview(vol, n_views=int(g[f"b{i}_nviews"]), detect=detector(side["circle"]),
                                    threshold=otsu)
        assert np.array_equal(lp.image, g[f"b{i}_thumb"]), i
        assert (lp.azimuth_deg, lp.entropy, lp.threshold, lp.mode, list(lp.warnings)) == (
            side["azimuth"], side["entropy"], side["threshold"], side["mode"], side["warnings"]), i
        # data preview (pipeline.py:240-257)
        dp = ops.build_data_preview(vol)
        assert np.array_equal(np.stack(dp.slicemaps.atlases), g[f"b{i}_data"]), i
        assert list(dp.filtered_bins) == meta["previews"]["data"]["filtered_bins"], i
        # interactive preview (pipeline.py:267-309)
        inter = meta["previews"]["interactive"]
        ip = ops.build_interactive_preview(vol, detect=detector(inter["container"]), threshold=otsu)
        for s in (128, 256, 512):
            assert np.array_equal(np.stack(ip.slicemaps[s].atlases), g[f"b{i}_int{s}"]), (i, s)
            assert ip.thresholds[s] == inter["thresholds"][str(s)], (i, s)
        assert list(ip.warnings) == inter["warnings"], i
        # atlas files (slicemap.py:158-166): same manifest, pixels round-trip
        mp = ops.save_slicemaps(dp.slicemaps, tmp_path / f"data{i}")
        man = json.loads(mp.read_text())
        assert man == dp.slicemaps.manifest()
        for m, name in enumerate(man["atlases"]):
            with Image.open(tmp_path / f"data{i}" / name) as im:
                assert np.array_equal(np.asarray(im), g[f"b{i}_data"][m]), (i, name)


def test_viewer_reference_frames(P, golden):
    """frontend/tests/fixtures/frames/params.json: surface (3 azimuths) and additive
    renders of the fixture bundle's decoded interactive-128 scheme -- bit-exact."""
    import json
    from pathlib import Path
    with np.load(Path(__file__).resolve().parent / "golden" / "ref_golden_bundles.npz") as z:
        atl, fm, ref = z["b0_int128"], json.loads(str(z["frames_params"])), z["frames_img"]
    vol = P.decode_slicemaps(P.SlicemapSet(scheme=P.plan_scheme(128), atlases=tuple(atl)))
    for k, fr in enumerate(fm["frames"]):
        vp = P.ViewParams(azimuth_deg=fr["azimuth"], image_dim=fm["image_dim"], steps=fm["steps"], mode=fr["mode"],
                          threshold=fr["threshold"], gain=fm["gain"])
        assert np.array_equal(P.render_view(vol, vp), ref[k]), fr["file"]


def test_circle_mask_spans_random(P, cuda):
    """The span form of the mask (binary search of the exact fp64 predicate per row,
    16-byte copies) equals the oracle per voxel: random circles, centres on and off
    the grid, radii whose boundary passes exactly through lattice points, widths on
    and off the 16-byte path, circles larger than the slice."""
    rng = np.random.default_rng(12)
    cases = [((3, 50, 64), 31.5, 24.5, 20.0, 0.0), ((2, 64, 80), 40.0, 30.0, 5.0 / 0.98, 0.02),  # 3-4-5 boundary
             ((2, 37, 53), 0.0, 0.0, 30.0, 0.1), ((2, 48, 48), 47.9, 47.9, 100.0, 0.0), ((1, 33, 96), 50.2, 16.7, 0.3, 0.0)]
    for _ in range(6):
        nz, ny, nx = int(rng.integers(1, 4)), int(rng.integers(8, 90)), int(rng.choice([16, 48, 64, 70, 128, 131]))
        cases.append(((nz, ny, nx), float(rng.uniform(0, nx)), float(rng.uniform(0, ny)), float(rng.uniform(1, 80)),
                      float(rng.choice([0.0, 0.02, 0.3]))))
    from types import SimpleNamespace as C
    for shape, cx, cy, r, m in cases:
        v = rng.integers(1, 256, size=shape, dtype=np.uint8)
        got = P.apply_circle_mask(P.Volume(v), C(cx=cx, cy=cy, r=r), margin=m).voxels
        assert np.array_equal(got, O.apply_circle_mask(v, cx, cy, r, m)), (shape, cx, cy, r, m)


def test_every_kernel_small_shapes_blocking_launches(P, cuda):
    """tools/sanitize_smoke.py (every kernel on small and ragged shapes: the fused pass u8/u16
    incl. the cooperative step, LUT kernels, general downscale paths, circle mask, PNG filter +
    deflate, atlas encode/decode, every render path, the config-5 processor) with
    CUDA_LAUNCH_BLOCKING=1 in a fresh process: no launch or execution error.  (compute-sanitizer
    is closed on this GPU pool; this is the in-tree stand-in.)"""
    import os
    import subprocess
    import sys
    from pathlib import Path
    root = Path(__file__).resolve().parents[1]
    r = subprocess.run([sys.executable, str(root / "tools" / "sanitize_smoke.py")], capture_output=True, text=True,
                       timeout=600, env={**os.environ, "CUDA_LAUNCH_BLOCKING": "1"})
    assert r.returncode == 0 and "sanitize smoke done" in r.stdout, r.stderr[-2000:]
