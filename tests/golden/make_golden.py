"""Generate the golden fixtures by running the REFERENCE itself (ctprev).

Run in the builder container, where /root/reference exists:

    NUMBA_CACHE_DIR=/tmp/numba_cache PYTHONDONTWRITEBYTECODE=1 \
        python tests/golden/make_golden.py

Writes tests/golden/ref_golden.npz, ref_golden_datapreview.npz,
ref_golden_interactive.npz and ref_golden_bundles.npz (committed).  The GPU box never reads
/root/reference: tests compare the CPU oracle and the CUDA path against these
frozen reference outputs.
"""
from __future__ import annotations

import os
import sys
from pathlib import Path

os.environ.setdefault("NUMBA_CACHE_DIR", "/tmp/numba_cache_ctprev")
os.environ.setdefault("PYTHONDONTWRITEBYTECODE", "1")
sys.dont_write_bytecode = True
sys.path.insert(0, "/root/reference/pkg/src")

import numpy as np  # noqa: E402

from ctprev.mask import artifact_bins, filter_histogram_bins  # noqa: E402
from ctprev.phantom import BoxSpec, CylinderSpec, PhantomSpec, SphereSpec, generate_phantom  # noqa: E402
from ctprev.render import ADDITIVE, SURFACE, ViewParams, image_entropy, optimal_snapshot, render_view  # noqa: E402
from ctprev.slicemap import SlicemapScheme, encode_slicemaps, plan_scheme  # noqa: E402
from ctprev.volume import Volume, downscale_volume, volume_histogram  # noqa: E402

OUT = Path(__file__).resolve().parent / "ref_golden.npz"


def main() -> None:
    g: dict[str, np.ndarray] = {}
    rng = np.random.default_rng(20231115)

    # ---- histogram (volume.py:252-262), incl. degenerate and ragged shapes
    hist_cases = [((1, 1, 1), None), ((3, 5, 7), None), ((7, 9, 33), (2, 5)), ((16, 24, 32), (0, 16)),
                  ((16, 24, 32), (15, 16)), ((5, 16, 48), (1, 4))]
    for i, (shape, zr) in enumerate(hist_cases):
        v = rng.integers(0, 256, size=shape, dtype=np.uint8)
        g[f"hist{i}_in"] = v
        g[f"hist{i}_z"] = np.array(zr if zr else (-1, -1), dtype=np.int64)
        g[f"hist{i}_out"] = volume_histogram(Volume(v), zr).bins.copy()
    g["hist_n"] = np.array(len(hist_cases))

    # ---- artifact bins + filter (mask.py:215-246)
    vox = np.zeros((8, 64, 64), dtype=np.uint8)       # the reference's own test stack (test_mask.py:155-161)
    vox[:6] = 90
    vox[6:] = 140
    vox[6:, :8, :8] = 200
    vox[7, 30, 30] = 90
    art_cases = [(vox, 2, 0.0005), (vox, 3, 0.0005), (vox, 1, 0.01)]
    for n_top, frac in ((3, 0.0005), (2, 0.002), (1, 0.0)):
        bg = np.clip(np.rint(rng.normal(20, 6, size=(12, 40, 48))), 0, 255).astype(np.uint8)
        art_cases.append((bg, n_top, frac))
    for i, (v, n_top, frac) in enumerate(art_cases):
        bins = artifact_bins(Volume(v), n_top=n_top, frac=frac)
        g[f"art{i}_in"] = v
        g[f"art{i}_ntop"] = np.array(n_top)
        g[f"art{i}_frac"] = np.array(frac)
        g[f"art{i}_bins"] = np.array(sorted(bins), dtype=np.int64)
        g[f"art{i}_filtered"] = filter_histogram_bins(Volume(v), bins).voxels.copy()
    g["art_n"] = np.array(len(art_cases))

    # ---- downscale (volume.py:265-309) incl. non-integer ratios
    ds_cases = [((8, 8, 8), (4, 4, 4)), ((16, 16, 10), (4, 16, 16)), ((19, 23, 37), (5, 7, 3)),
                ((24, 40, 40), (32, 32, 20)), ((32, 32, 32), (4, 4, 4)), ((12, 12, 12), (12, 12, 12)),
                ((9, 17, 33), (1, 1, 1)), ((64, 48, 48), (24, 24, 32)), ((16, 32, 64), (16, 8, 4))]
    for i, (shape, target) in enumerate(ds_cases):
        v = rng.integers(0, 256, size=shape, dtype=np.uint8)
        g[f"ds{i}_in"] = v
        g[f"ds{i}_target"] = np.array(target, dtype=np.int64)
        g[f"ds{i}_out"] = downscale_volume(Volume(v), target).voxels.copy()
    g["ds_n"] = np.array(len(ds_cases))

    # ---- slicemaps (slicemap.py:120-142), custom + planned schemes
    enc_cases = [((64, 64, 64), (64, 512, 8, 1)), ((96, 96, 96), (96, 768, 8, 2)), ((100, 90, 80), (64, 512, 8, 1)),
                 ((32, 32, 32), (32, 128, 4, 2)), ((48, 64, 64), (48, 384, 8, 1)), ((128, 128, 128), 128)]
    for i, (shape, sc) in enumerate(enc_cases):
        if isinstance(sc, int):
            zs = np.arange(shape[0]).reshape(-1, 1, 1)
            ys = np.arange(shape[1]).reshape(1, -1, 1)
            xs = np.arange(shape[2]).reshape(1, 1, -1)
            v = ((zs * 7 + ys * 3 + xs * 31) % 256).astype(np.uint8)
            scheme = plan_scheme(sc)
        else:
            v = rng.integers(0, 256, size=shape, dtype=np.uint8)
            scheme = SlicemapScheme(*sc)
        sset = encode_slicemaps(Volume(v), scheme)
        g[f"enc{i}_in"] = v
        g[f"enc{i}_scheme"] = np.array([scheme.s, scheme.atlas_dim, scheme.grid, scheme.map_count], dtype=np.int64)
        g[f"enc{i}_out"] = np.stack(sset.atlases)
    g["enc_n"] = np.array(len(enc_cases))

    # ---- render (render.py:205-236): L-phantom (test_render.py:36-48) and a sphere
    l_ph = generate_phantom(PhantomSpec(
        dims=(96, 96, 96),
        objects=(BoxSpec((8, 40, 8), (88, 56, 24), value=(150, 150)),
                 BoxSpec((8, 40, 24), (24, 56, 88), value=(220, 220)),
                 SphereSpec(70.0, 48.0, 60.0, r=10.0, value=(90, 90))),
        seed=4)).volume
    g["lphantom"] = l_ph.voxels.copy()
    cyl = generate_phantom(PhantomSpec(
        dims=(96, 96, 96),
        container=CylinderSpec(cx=47.5, cy=47.5, r=36.0, wall=36.0, value=(180, 180)), seed=3)).volume
    g["cylinder"] = cyl.voxels.copy()
    aniso = rng.integers(0, 256, size=(20, 28, 36), dtype=np.uint8)
    g["aniso"] = aniso
    rcases = [("lphantom", 17.0, 64, 64, SURFACE, 60), ("lphantom", 0.0, 48, 96, ADDITIVE, 1),
              ("lphantom", 123.4, 64, 64, SURFACE, 1), ("lphantom", 300.0, 32, 128, ADDITIVE, 1),
              ("aniso", 45.0, 32, 64, SURFACE, 100), ("aniso", 200.0, 32, 64, ADDITIVE, 1),
              ("cylinder", 90.0, 40, 40, SURFACE, 60)]
    vols = {"lphantom": l_ph, "cylinder": cyl, "aniso": Volume(aniso)}
    for i, (name, az, dim, steps, mode, thr) in enumerate(rcases):
        img = render_view(vols[name], ViewParams(azimuth_deg=az, image_dim=dim, steps=steps, mode=mode,
                                                 threshold=thr))
        g[f"rv{i}_vol"] = np.frombuffer(name.encode(), dtype=np.uint8)
        g[f"rv{i}_params"] = np.array([az, dim, steps, 1.0 if mode == ADDITIVE else 0.0, thr], dtype=np.float64)
        g[f"rv{i}_out"] = img
    g["rv_n"] = np.array(len(rcases))

    # ---- entropy + snapshot (render.py:248-314); test_render.py:170-179 known answer
    snap = optimal_snapshot(l_ph, n_views=12, params=ViewParams(image_dim=128, steps=64, threshold=60))
    g["snap_az"] = np.array(snap.azimuth_deg)
    g["snap_h"] = np.array(snap.entropy)
    g["snap_per_view"] = np.array(snap.per_view, dtype=np.float64)
    g["snap_img"] = snap.image
    ent_imgs = [np.full((64, 64), 7, np.uint8), np.tile(np.arange(256, dtype=np.uint8), 256).reshape(256, 256),
                rng.integers(0, 256, size=(32, 32), dtype=np.uint8), snap.image]
    for i, im in enumerate(ent_imgs):
        g[f"ent{i}_in"] = im
        g[f"ent{i}_h"] = np.array(image_entropy(im).entropy)
    g["ent_n"] = np.array(len(ent_imgs))

    np.savez_compressed(OUT, **g)
    print(f"wrote {OUT} ({OUT.stat().st_size / 1e6:.2f} MB, {len(g)} arrays)")





def data_preview_golden() -> None:
    """Reference build_data_preview (pipeline.py:240-257) on two mounted phantoms."""
    from ctprev.pipeline import build_data_preview
    out = Path(__file__).resolve().parent / "ref_golden_datapreview.npz"
    g = {}
    specs = [
        PhantomSpec(dims=(160, 160, 96),
                    container=CylinderSpec(cx=81.0, cy=78.0, r=65.0, wall=2.0, value=(140, 145)),
                    objects=(SphereSpec(cx=75.0, cy=85.0, cz=40.0, r=22.0, value=(200, 210)),), seed=5),
        PhantomSpec(dims=(272, 264, 260),
                    container=CylinderSpec(cx=135.0, cy=131.0, r=120.0, wall=4.0, value=(40, 60)),
                    objects=(SphereSpec(cx=120.0, cy=140.0, cz=150.0, r=50.0, value=(120, 200)),
                             BoxSpec((60, 60, 20), (200, 90, 80), value=(90, 95))), seed=9),
    ]
    for i, spec in enumerate(specs):
        vol = generate_phantom(spec).volume
        dp = build_data_preview(vol)
        g[f"dp{i}_in"] = vol.voxels.copy()
        g[f"dp{i}_bins"] = np.array(dp.filtered_bins, dtype=np.int64)
        g[f"dp{i}_atlases"] = np.stack(dp.slicemaps.atlases)
    g["dp_n"] = np.array(len(specs))
    # acceptance criterion 8 (test_acceptance.py:217-244): 36 views, 256^2, 256 steps, surface T=60
    l_ph = generate_phantom(PhantomSpec(
        dims=(96, 96, 96),
        objects=(BoxSpec((8, 40, 8), (88, 56, 24), value=(150, 150)),
                 BoxSpec((8, 40, 24), (24, 56, 88), value=(220, 220)),
                 SphereSpec(70.0, 48.0, 60.0, r=10.0, value=(90, 90))),
        seed=4)).volume
    snap = optimal_snapshot(l_ph, n_views=36, params=ViewParams(image_dim=256, steps=256, mode=SURFACE, threshold=60))
    g["acc_snap_az"] = np.array(snap.azimuth_deg)
    g["acc_snap_h"] = np.array(snap.entropy)
    g["acc_snap_per_view"] = np.array(snap.per_view, dtype=np.float64)
    g["acc_snap_img"] = snap.image
    # apply_circle_mask (mask.py:194-212), fractional centres, margins, boundary-touching radii
    from ctprev.mask import Circle, apply_circle_mask
    rng = np.random.default_rng(77)
    mvol = rng.integers(1, 256, size=(3, 57, 63), dtype=np.uint8)
    cases = [(31.0, 28.0, 20.0, 0.02), (30.5, 27.25, 26.0, 0.0), (12.3, 40.7, 33.3, 0.1), (0.0, 0.0, 70.0, 0.5),
             (62.9, 56.9, 5.0, 0.02)]
    for i, (cx, cy, r, m) in enumerate(cases):
        g[f"cm{i}_params"] = np.array([cx, cy, r, m])
        g[f"cm{i}_out"] = apply_circle_mask(Volume(mvol), Circle(cx, cy, r), margin=m).voxels.copy()
    g["cm_in"] = mvol
    g["cm_n"] = np.array(len(cases))
    np.savez_compressed(out, **g)
    print(f"wrote {out} ({out.stat().st_size / 1e6:.2f} MB)")


def interactive_preview_golden() -> None:
    """Reference build_interactive_preview (pipeline.py:267-309) on the two data-preview
    phantoms (inputs: ref_golden_datapreview.npz dp0_in / dp1_in) and a constant
    volume (no circle, degenerate histogram).  Stored: the circle, thresholds,
    warnings, each scheme's masked-level histogram (recomputed with the reference's
    own functions, the Otsu input), SHA-256 of each scheme's atlas bytes, and the
    128-scheme atlas itself."""
    import hashlib
    from ctprev.mask import apply_circle_mask
    from ctprev.pipeline import _rescale_circle, _scheme_volume, build_interactive_preview
    from ctprev.threshold import otsu_threshold
    dp = np.load(Path(__file__).resolve().parent / "ref_golden_datapreview.npz")
    out = Path(__file__).resolve().parent / "ref_golden_interactive.npz"
    const = np.full((32, 48, 40), 7, dtype=np.uint8)
    vols = [dp["dp0_in"], dp["dp1_in"], const]
    g = {"ip_const_in": const, "ip_n": np.array(len(vols))}
    for i, v in enumerate(vols):
        vol = Volume(v)
        ip = build_interactive_preview(vol)
        c = ip.circle
        g[f"ip{i}_circle"] = np.array([np.nan] * 4 if c is None else [c.cx, c.cy, c.r, c.votes])
        g[f"ip{i}_warnings"] = np.array(",".join(ip.warnings))
        for s in (128, 256, 512):
            t = ip.thresholds[s]
            g[f"ip{i}_thr{s}"] = np.array(-1 if t is None else t)
            a = np.stack(ip.slicemaps[s].atlases)
            g[f"ip{i}_sha{s}"] = np.array(hashlib.sha256(a.tobytes()).hexdigest())
            g[f"ip{i}_shape{s}"] = np.array(a.shape)
            down = _scheme_volume(vol, s)
            if c is not None:
                down = apply_circle_mask(down, _rescale_circle(c, _scheme_volume(vol, 512), down))
            h = volume_histogram(down)
            g[f"ip{i}_hist{s}"] = h.bins.copy()
            if t is not None:
                assert otsu_threshold(h).value == t
        g[f"ip{i}_atlas128"] = np.stack(ip.slicemaps[128].atlases)
    np.savez_compressed(out, **g)
    print(f"wrote {out} ({out.stat().st_size / 1e6:.2f} MB)")


def bundle_golden() -> None:
    """The reference's own bundle flow (ingest_stack + build_bundle, pipeline.py:356-500)
    for the two bundles whose checksums are mounted -- fixture-128
    (frontend/scripts/make-fixtures.py:67-81, n_views 4) and demo-scan-01
    (demos/full_pipeline.py:49-68, n_views 6).  Every file's sha256 is checked
    against the mounted meta.json first (27/27 each), then the decoded products are
    frozen: the input volume, data atlases + bins, interactive atlases per scheme +
    circle / thresholds / warnings, and the thumbnail + its sidecar."""
    import hashlib
    import json
    import shutil
    import tempfile
    from PIL import Image
    from ctprev.phantom import CylinderSpec, PhantomSpec, SphereSpec, generate_phantom
    from ctprev.pipeline import build_bundle, ingest_stack
    ref = Path("/root/reference/pkg")
    cases = [
        ("fixture-128", "Viewer Fixture", 4, ref / "frontend/tests/fixtures/bundles/fixture-128/meta.json",
         PhantomSpec(dims=(128, 128, 128), fill=(4, 18),
                     container=CylinderSpec(cx=65.0, cy=63.0, r=52.0, wall=2.5, value=(140, 145)),
                     objects=(SphereSpec(cx=60.0, cy=68.0, cz=52.0, r=20.0, value=(200, 210)),
                              SphereSpec(cx=76.0, cy=54.0, cz=92.0, r=10.0, value=(220, 230))),
                     salt_pepper=0.0005, seed=11)),
        ("demo-scan-01", "Demo Scan 01", 6, ref / "demos/out/full_pipeline/bundles/demo-scan-01/meta.json",
         PhantomSpec(dims=(160, 160, 96),
                     container=CylinderSpec(cx=81.0, cy=78.0, r=65.0, wall=2.0, value=(140, 145)),
                     objects=(SphereSpec(cx=75.0, cy=85.0, cz=40.0, r=22.0, value=(200, 210)),),
                     salt_pepper=0.001, seed=5)),
    ]
    g = {"b_n": np.array(len(cases))}
    work = Path(tempfile.mkdtemp(prefix="ctp_bundles_"))
    try:
        for i, (bid, name, n_views, meta_path, spec) in enumerate(cases):
            vol = generate_phantom(spec).volume
            stack = work / f"stack{i}"
            stack.mkdir()
            names = []
            for z in range(vol.nz):  # the scripts' write_stack: one L-mode PNG per slice + stack.json
                fn = f"slice_{z:04d}.png"
                Image.fromarray(np.asarray(vol.voxels[z]), mode="L").save(stack / fn)
                names.append(fn)
            (stack / "stack.json").write_text(json.dumps({"name": name, "slices": names, "bit_depth": 8}))
            root = work / f"root{i}"
            ingest_stack(stack / "stack.json", root, dataset_id=bid)
            meta = build_bundle(root, bid, n_views=n_views)
            bundle = root / bid
            want = json.loads(meta_path.read_text())["checksums"]
            ok = 0
            for rel, digest in want.items():
                if hashlib.sha256((bundle / rel).read_bytes()).hexdigest() == digest:
                    ok += 1
            print(f"{bid}: {ok}/{len(want)} files match the mounted checksums")
            assert ok == len(want), bid

            def png(rel):
                with Image.open(bundle / rel) as im:
                    return np.asarray(im).copy()

            nz, ny, nx = vol.voxels.shape
            g[f"b{i}_id"] = np.array(bid)
            g[f"b{i}_nviews"] = np.array(n_views)
            g[f"b{i}_checks"] = np.array([ok, len(want)])
            g[f"b{i}_vol"] = np.fromfile(bundle / "volume.raw", dtype=np.uint8).reshape(nz, ny, nx)
            g[f"b{i}_meta"] = np.array(json.dumps(meta, sort_keys=True))
            g[f"b{i}_thumb"] = png("thumbnail.png")
            g[f"b{i}_sidecar"] = np.array((bundle / "thumbnail.json").read_text())
            dman = json.loads((bundle / "data" / "manifest.json").read_text())
            g[f"b{i}_data"] = np.stack([png(f"data/{a}") for a in dman["atlases"]])
            for s in (128, 256, 512):
                man = json.loads((bundle / "interactive" / str(s) / "manifest.json").read_text())
                g[f"b{i}_int{s}"] = np.stack([png(f"interactive/{s}/{a}") for a in man["atlases"]])
            if bid == "fixture-128":
                # the viewer's reference frames (make-fixtures.py:99-130; frames/params.json): renders of
                # the decoded interactive 128 scheme at the scheme's own threshold
                from ctprev.render import ViewParams, render_view
                from ctprev.slicemap import decode_slicemaps, load_slicemaps
                frames_meta = json.loads((ref / "frontend/tests/fixtures/frames/params.json").read_text())
                dec = decode_slicemaps(load_slicemaps(bundle / "interactive" / "128" / "manifest.json"))
                imgs = []
                for fr in frames_meta["frames"]:
                    vp = ViewParams(azimuth_deg=fr["azimuth"], image_dim=frames_meta["image_dim"],
                                    steps=frames_meta["steps"], mode=fr["mode"], threshold=fr["threshold"],
                                    gain=frames_meta["gain"])
                    imgs.append(render_view(dec, vp))
                g["frames_params"] = np.array(json.dumps(frames_meta))
                g["frames_img"] = np.stack(imgs)
    finally:
        shutil.rmtree(work, ignore_errors=True)
    out = Path(__file__).resolve().parent / "ref_golden_bundles.npz"
    np.savez_compressed(out, **g)
    print(f"wrote {out} ({out.stat().st_size / 1e6:.2f} MB)")


def bundle_checksums() -> None:
    """The mounted meta.json checksums of the two recorded bundles (27 files each),
    copied to tests/golden/ref_bundle_checksums.json so the GPU box -- which has no
    /root/reference -- can check a build_bundle run under install() against them."""
    import json
    ref = Path("/root/reference/pkg")
    src = {"fixture-128": ref / "frontend/tests/fixtures/bundles/fixture-128/meta.json",
           "demo-scan-01": ref / "demos/out/full_pipeline/bundles/demo-scan-01/meta.json"}
    out = {bid: {"source": str(p.relative_to(ref)), "checksums": json.loads(p.read_text())["checksums"]}
           for bid, p in src.items()}
    dst = Path(__file__).resolve().parent / "ref_bundle_checksums.json"
    dst.write_text(json.dumps(out, indent=1, sort_keys=True) + "\n")
    print(f"wrote {dst}")


if __name__ == "__main__":
    if "--only-checksums" in sys.argv:
        bundle_checksums()
        sys.exit(0)
    if "--only-bundles" in sys.argv:
        bundle_golden()
        sys.exit(0)
    if "--only-interactive" in sys.argv:
        interactive_preview_golden()
        sys.exit(0)
    if "--only-extra" not in sys.argv:
        main()
    data_preview_golden()
    interactive_preview_golden()
    bundle_golden()
    bundle_checksums()
