"""ctprev's OWN callers with the B200 path installed: the
reference's ``ingest_stack`` + ``build_bundle`` (pipeline.py:356-500) run
unmodified after ``install()`` rebinds every binding site, on the two bundles
whose checksums the reference recorded (fixture-128: frontend/tests/fixtures/
bundles/fixture-128/meta.json; demo-scan-01: demos/out/full_pipeline/bundles/
demo-scan-01/meta.json; copied to tests/golden/ref_bundle_checksums.json).

* with the reference's own PNG writer kept (``exclude=("save_slicemaps",)``):
  all 27/27 files of each bundle must hash to the recorded checksums -- every
  atlas pixel, the filtered bins, thresholds, circle, the thumbnail and its
  sidecar entropy come from the device path;
* with everything installed (the device PNG writer too): the non-atlas files
  hash identically and every atlas PNG decodes to the recorded pixels.

ctprev is imported from ``baseline/_ref`` (the pip install the reference arm
uses; it travels to the GPU box) or the mounted source tree."""
from __future__ import annotations

import hashlib
import importlib
import json
import os
import sys
from pathlib import Path

import numpy as np
import pytest

ROOT = Path(__file__).resolve().parents[1]
GOLDEN = ROOT / "tests" / "golden"


def _import_ctprev():
    os.environ.setdefault("NUMBA_CACHE_DIR", "/tmp/ctp_numba_install_test")
    for d in (ROOT / "baseline" / "_ref", Path("/root/reference/pkg/src")):
        if (d / "ctprev").is_dir():
            if str(d) not in sys.path:
                sys.path.insert(0, str(d))
            break
    else:
        pytest.skip("ctprev is not installed (baseline/_ref) nor mounted")
    return importlib.import_module("ctprev")


def _write_stack(vol: np.ndarray, name: str, d: Path) -> Path:
    """The scripts' write_stack: one L-mode PNG per slice + stack.json (make-fixtures.py)."""
    from PIL import Image
    d.mkdir(parents=True)
    names = []
    for z in range(vol.shape[0]):
        fn = f"slice_{z:04d}.png"
        Image.fromarray(np.ascontiguousarray(vol[z]), mode="L").save(d / fn)
        names.append(fn)
    (d / "stack.json").write_text(json.dumps({"name": name, "slices": names, "bit_depth": 8}))
    return d / "stack.json"


@pytest.mark.gpu
@pytest.mark.parametrize("device_png", [False, True])
def test_build_bundle_under_install_matches_recorded_checksums(cuda, tmp_path, device_png):
    _import_ctprev()
    import ctprev.pipeline as pl
    from PIL import Image
    from paper_2311_15038_b200 import _lib, ops
    from paper_2311_15038_b200.install import install, uninstall
    want_all = json.loads((GOLDEN / "ref_bundle_checksums.json").read_text())
    with np.load(GOLDEN / "ref_golden_bundles.npz") as z:
        g = {k: z[k] for k in z.files}
    patched = install(exclude=() if device_png else ("save_slicemaps",))
    try:
        assert "ctprev.pipeline.build_interactive_preview" in patched
        assert pl.build_data_preview is ops.build_data_preview and pl.load_volume is ops.load_volume
        _lib.launch_count(reset=True)
        for i in range(int(g["b_n"])):
            bid = str(g[f"b{i}_id"])
            meta0 = json.loads(str(g[f"b{i}_meta"]))
            stack = _write_stack(g[f"b{i}_vol"], meta0["name"], tmp_path / f"stack{i}")
            root = tmp_path / f"root{i}"
            pl.ingest_stack(stack, root, dataset_id=bid)                          # pipeline.py:356-398
            pl.build_bundle(root, bid, n_views=int(g[f"b{i}_nviews"]))           # pipeline.py:420-500
            bundle = root / bid
            want = want_all[bid]["checksums"]
            assert len(want) == 27
            ok, decoded = 0, 0
            for rel, digest in want.items():
                got = hashlib.sha256((bundle / rel).read_bytes()).hexdigest()
                is_atlas = rel.endswith(".png") and rel != "thumbnail.png"
                if device_png and is_atlas:
                    # our writer: different deflate bytes, the same pixels
                    parts = rel.split("/")
                    k = int(parts[-1].rsplit("_", 1)[1].split(".")[0])
                    ref = g[f"b{i}_data"][k] if parts[0] == "data" else g[f"b{i}_int{int(parts[1])}"][k]
                    with Image.open(bundle / rel) as im:
                        assert np.array_equal(np.asarray(im), ref), (bid, rel)
                    decoded += 1
                else:
                    assert got == digest, (bid, rel)
                    ok += 1
            assert ok + decoded == 27, (bid, ok, decoded)
        assert _lib.launch_count() > 0  # the device path ran
    finally:
        uninstall()
