"""Ingest: ctprev's raw + JSON header format streamed into the
device path.  Header validation and the chunk reader run on the CPU; the
streamed preview is compared with the in-memory one on the GPU."""
from __future__ import annotations

import json
from pathlib import Path

import numpy as np
import pytest

REF = Path("/root/reference/pkg/src")


def _write(tmp, name, vol, header=None):
    nz, ny, nx = vol.shape
    (tmp / f"{name}.raw").write_bytes(vol.tobytes())
    h = {"dims": [nx, ny, nz], "dtype": "u8", "order": "xyz", "voxel_size_um": 1.5} if header is None else header
    (tmp / f"{name}.json").write_text(h if isinstance(h, str) else json.dumps(h))
    return tmp / f"{name}.json"


def _bad_headers(tmp):
    vol = np.arange(2 * 3 * 4, dtype=np.uint8).reshape(2, 3, 4)
    cases = {
        "json": _write(tmp, "json", vol, "{not json"),
        "dtype": _write(tmp, "dtype", vol, {"dims": [4, 3, 2], "dtype": "u16", "order": "xyz"}),
        "order": _write(tmp, "order", vol, {"dims": [4, 3, 2], "dtype": "u8", "order": "zyx"}),
        "dims": _write(tmp, "dims", vol, {"dims": [4, 3], "dtype": "u8", "order": "xyz"}),
        "size": _write(tmp, "size", vol, {"dims": [4, 3, 3], "dtype": "u8", "order": "xyz"}),
    }
    _write(tmp, "missing", vol)
    (tmp / "missing.raw").unlink()
    cases["missing"] = tmp / "missing.json"
    return cases


def test_read_header_errors(tmp_path):
    from paper_2311_15038_b200 import errors as E
    from paper_2311_15038_b200.ingest import read_header
    want = {"json": E.InvalidManifest, "dtype": E.UnsupportedPixelFormat, "order": E.UnsupportedPixelFormat,
            "dims": E.InvalidManifest, "size": E.DimensionMismatch, "missing": E.MissingSlice}
    for k, p in _bad_headers(tmp_path).items():
        with pytest.raises(want[k]):
            read_header(p)
    vol = np.zeros((5, 6, 7), dtype=np.uint8)
    shape, raw, vs = read_header(_write(tmp_path, "ok", vol))
    assert shape == (5, 6, 7) and raw.name == "ok.raw" and vs == 1.5
    import paper_2311_15038_b200 as P
    rnd = np.random.default_rng(2).integers(0, 256, size=(9, 6, 7), dtype=np.uint8)
    v = P.load_volume(_write(tmp_path, "rnd", rnd), threads=3)   # the host drop-in (volume.py:229-249)
    assert np.array_equal(v.voxels, rnd) and v.voxel_size_um == 1.5
    for k, p in _bad_headers(tmp_path).items():
        with pytest.raises(want[k]):
            P.load_volume(p)


@pytest.mark.skipif(not REF.exists(), reason="reference not mounted")
def test_read_header_errors_match_load_volume(tmp_path):
    """Same error class NAMES and messages as the reference's load_volume (volume.py:229-249)."""
    import subprocess
    import sys
    cases = _bad_headers(tmp_path)
    code = ("import sys, json; sys.path.insert(0, %r)\n"
            "from ctprev.volume import load_volume\n"
            "out = {}\n"
            "for k, p in json.loads(sys.argv[1]).items():\n"
            "    try:\n        load_volume(p); out[k] = None\n"
            "    except Exception as e:\n        out[k] = [type(e).__name__, str(e)]\n"
            "print(json.dumps(out))\n") % str(REF)
    r = subprocess.run([sys.executable, "-c", code, json.dumps({k: str(p) for k, p in cases.items()})],
                       capture_output=True, text=True, env={"NUMBA_CACHE_DIR": "/tmp/numba_cache_ingest",
                                                            "PYTHONDONTWRITEBYTECODE": "1", "PATH": "/usr/bin"})
    ref = json.loads(r.stdout.strip().splitlines()[-1])
    from paper_2311_15038_b200.ingest import read_header
    for k, p in cases.items():
        try:
            read_header(p)
            got = None
        except Exception as e:
            got = [type(e).__name__, str(e)]
        if k == "json":  # the JSON decoder's own message text
            assert got[0] == ref[k][0]
        else:
            assert got == ref[k], k


def test_raw_reader_slabs(tmp_path):
    from paper_2311_15038_b200.ingest import RawReader, read_header
    rng = np.random.default_rng(3)
    vol = rng.integers(0, 256, size=(37, 19, 23), dtype=np.uint8)
    shape, raw, _ = read_header(_write(tmp_path, "v", vol))
    with RawReader(raw, shape) as rd:
        for z0, z1 in ((0, 37), (34, 37), (5, 17), (36, 37)):
            out = np.empty((z1 - z0,) + shape[1:], dtype=np.uint8)
            rd(z0, z1, out)
            assert np.array_equal(out, vol[z0:z1])


@pytest.mark.gpu
@pytest.mark.parametrize("shape,schemes,chunk", [((256, 256, 256), (256, 128), 32), ((200, 200, 200), (128,), 64)])
def test_preview_from_raw_equals_in_memory(tmp_path, cuda, shape, schemes, chunk):
    """Streamed from disk through pinned chunks == preview_pipeline on the loaded volume
    (power-of-two levels stream in z-chunks; a general ratio runs whole-volume)."""
    import paper_2311_15038_b200 as P
    from paper_2311_15038_b200.ingest import preview_from_raw
    rng = np.random.default_rng(11)
    vol = np.clip(np.rint(rng.normal(20, 6, shape)), 0, 255).astype(np.uint8)
    vol[shape[0] // 3: shape[0] // 2, 40:120, 30:150] = rng.integers(120, 220, size=(shape[0] // 2 - shape[0] // 3, 80, 120),
                                                                     dtype=np.uint8)
    vol[-3:] = rng.integers(0, 60, size=(3,) + shape[1:], dtype=np.uint8)
    hp = _write(tmp_path, "scan", vol)
    got = preview_from_raw(hp, schemes=schemes, chunk_slices=chunk)
    ref = P.preview_pipeline(P.Volume(vol), schemes=schemes)
    assert np.array_equal(got.histogram, ref.histogram)
    assert got.bins == ref.bins
    for s in schemes:
        assert np.array_equal(np.stack(got.slicemaps[s].atlases), np.stack(ref.slicemaps[s].atlases)), s


@pytest.mark.gpu
@pytest.mark.parametrize("u16", [False, True])
def test_preview_session_host_buffers_equal_in_memory(cuda, u16):
    """PreviewSession.run (pinned host volume -> z-chunk H2D / fused pass / atlas D2H on
    three streams, the bench's e2e path) == the one-launch device step, twice in a row
    (buffers reused)."""
    import torch
    import paper_2311_15038_b200 as P
    from paper_2311_15038_b200.device import AtlasSpec
    from paper_2311_15038_b200.pipeline import PreviewSession
    rng = np.random.default_rng(5)
    shape = (512, 256, 256)
    schemes = {256: AtlasSpec.of(P.plan_scheme(256)), 128: AtlasSpec.of(P.plan_scheme(128))}
    sess = PreviewSession(shape, torch.uint16 if u16 else torch.uint8, schemes, chunk_slices=64)
    for it in range(2):
        if u16:  # 12-bit data (the config-3/5 extension), incl. values that saturate
            vol = np.clip(np.rint(rng.normal(400 + 100 * it, 120, shape)), 0, 4200).astype(np.uint16)
            vol[-3:, :64] = 2800
        else:
            vol = np.clip(np.rint(rng.normal(30 + 10 * it, 8, shape)), 0, 255).astype(np.uint8)
            vol[-3:, :64] = 200
        host = torch.from_numpy(vol).pin_memory()
        out = sess.run(host)
        ref = P.preview_pipeline(vol, schemes=(256, 128))  # the array form takes uint16 too
        assert np.array_equal(out["hist"].numpy(), ref.histogram)
        assert frozenset(np.nonzero(out["flags"].numpy())[0].tolist()) == ref.bins
        for s in (256, 128):
            assert np.array_equal(out["atlases"][s].numpy(), np.stack(ref.slicemaps[s].atlases)), (it, s)


# ---------------------------------------------------------------- slice stacks (volume.py:167-202)

def _write_stack(tmp, vol, name="stack", manifest=None, mode="L"):
    from PIL import Image
    files = []
    for z in range(vol.shape[0]):
        f = f"{name}_{z:04d}.png"
        im = Image.fromarray(vol[z])
        (im if mode == "L" else im.convert(mode)).save(tmp / f)
        files.append(f)
    m = {"name": name, "slices": files, "bit_depth": 8} if manifest is None else manifest
    (tmp / f"{name}.json").write_text(m if isinstance(m, str) else json.dumps(m))
    return tmp / f"{name}.json"


def test_ingest_checks_artifact_arguments_before_reading(tmp_path):
    """n_top outside [1, nz] and a negative frac raise RangeOutOfBounds (mask.py:223-226)
    before any read or device allocation, in both ingest entry points and PreviewSession."""
    from paper_2311_15038_b200 import errors as E
    from paper_2311_15038_b200.ingest import preview_from_raw, preview_from_slice_stack
    from paper_2311_15038_b200.pipeline import PreviewSession
    vol = np.random.default_rng(5).integers(0, 256, size=(2, 16, 16), dtype=np.uint8)
    raw = _write(tmp_path, "two", vol)
    stack = _write_stack(tmp_path, vol, name="two_stack")
    for kw in ({"n_top": 3}, {"n_top": 0}, {"frac": -1e-3}):
        with pytest.raises(E.RangeOutOfBounds):
            preview_from_raw(raw, schemes=(16,), **kw)
        with pytest.raises(E.RangeOutOfBounds):
            preview_from_slice_stack(stack, schemes=(16,), **kw)
        with pytest.raises(E.RangeOutOfBounds):
            PreviewSession(vol.shape, None, {}, **kw)


def test_slice_stack_manifest_errors_and_reader(tmp_path):
    """read_manifest / SliceStackReader raise load_slice_stack's error classes under
    its conditions and decode the slices in z order."""
    from paper_2311_15038_b200 import errors as E
    from paper_2311_15038_b200.ingest import SliceStackReader, read_manifest
    rng = np.random.default_rng(3)
    vol = rng.integers(0, 256, size=(5, 7, 9), dtype=np.uint8)
    ok = _write_stack(tmp_path, vol)
    paths, shape = read_manifest(ok)
    assert shape == (5, 7, 9) and len(paths) == 5
    out = np.zeros((3, 7, 9), dtype=np.uint8)
    with SliceStackReader(paths, shape, threads=4) as rd:
        rd(1, 4, out)
    assert np.array_equal(out, vol[1:4])
    (tmp_path / "bad.json").write_text("{not json")
    with pytest.raises(E.InvalidManifest):
        read_manifest(tmp_path / "bad.json")
    (tmp_path / "noslices.json").write_text(json.dumps({"name": "x"}))
    with pytest.raises(E.InvalidManifest):
        read_manifest(tmp_path / "noslices.json")
    (tmp_path / "empty.json").write_text(json.dumps({"slices": []}))
    with pytest.raises(E.InvalidManifest):
        read_manifest(tmp_path / "empty.json")
    (tmp_path / "deep.json").write_text(json.dumps({"slices": ["stack_0000.png"], "bit_depth": 16}))
    with pytest.raises(E.UnsupportedPixelFormat):
        read_manifest(tmp_path / "deep.json")
    (tmp_path / "gone.json").write_text(json.dumps({"slices": ["nope.png"]}))
    with pytest.raises(E.MissingSlice):
        read_manifest(tmp_path / "gone.json")
    import paper_2311_15038_b200 as P
    v = P.load_slice_stack(ok, threads=3)            # the host drop-in (volume.py:167-202)
    assert np.array_equal(v.voxels, vol) and v.voxels.flags["C_CONTIGUOUS"]
    rgb = _write_stack(tmp_path, vol[:2], name="rgb", mode="RGB")
    with pytest.raises(E.UnsupportedPixelFormat):
        read_manifest(rgb)
    from PIL import Image
    Image.fromarray(np.zeros((8, 9), np.uint8)).save(tmp_path / "odd.png")
    (tmp_path / "mixed.json").write_text(json.dumps({"slices": ["stack_0000.png", "odd.png"]}))
    paths, shape = read_manifest(tmp_path / "mixed.json")
    with pytest.raises(E.DimensionMismatch):
        with SliceStackReader(paths, shape, threads=2) as rd:
            rd(0, 2, np.zeros((2, 7, 9), np.uint8))


@pytest.mark.gpu
def test_preview_from_slice_stack_equals_in_memory(cuda, tmp_path):
    """A PNG slice stack decoded in parallel straight into the streaming pass (chunks
    of 32 slices) == preview_pipeline on the assembled volume."""
    import paper_2311_15038_b200 as P
    from paper_2311_15038_b200.ingest import preview_from_slice_stack
    rng = np.random.default_rng(9)
    vol = np.clip(np.rint(rng.normal(25, 7, (96, 128, 128))), 0, 255).astype(np.uint8)
    vol[20:70, 30:90, 40:100] = rng.integers(120, 220, size=(50, 60, 60), dtype=np.uint8)
    vol[-3:, :40] = 150
    man = _write_stack(tmp_path, vol)
    got = preview_from_slice_stack(man, schemes=(128, P.SlicemapScheme(64, 512, 8, 1)), chunk_slices=32)
    ref = P.preview_pipeline(vol, schemes=(128, P.SlicemapScheme(64, 512, 8, 1)))
    assert np.array_equal(got.histogram, ref.histogram)
    assert got.bins == ref.bins
    for s in (128, 64):
        assert np.array_equal(np.stack(got.slicemaps[s].atlases), np.stack(ref.slicemaps[s].atlases)), s


@pytest.mark.skipif(not REF.exists(), reason="reference not mounted")
def test_slice_stack_errors_match_load_slice_stack(tmp_path):
    """Same error class names as the reference's load_slice_stack (volume.py:167-202)
    for every bad-manifest / bad-slice case, and the same volume for a good stack."""
    import subprocess
    import sys
    from PIL import Image
    rng = np.random.default_rng(4)
    vol = rng.integers(0, 256, size=(4, 6, 10), dtype=np.uint8)
    cases = {"ok": _write_stack(tmp_path, vol)}
    (tmp_path / "bad.json").write_text("{not json")
    cases["json"] = tmp_path / "bad.json"
    (tmp_path / "noslices.json").write_text(json.dumps({"name": "x"}))
    cases["noslices"] = tmp_path / "noslices.json"
    (tmp_path / "empty.json").write_text(json.dumps({"slices": []}))
    cases["empty"] = tmp_path / "empty.json"
    (tmp_path / "deep.json").write_text(json.dumps({"slices": ["stack_0000.png"], "bit_depth": 16}))
    cases["deep"] = tmp_path / "deep.json"
    (tmp_path / "gone.json").write_text(json.dumps({"slices": ["stack_0000.png", "nope.png"]}))
    cases["gone"] = tmp_path / "gone.json"
    cases["rgb"] = _write_stack(tmp_path, vol[:2], name="rgb", mode="RGB")
    Image.fromarray(np.zeros((8, 9), np.uint8)).save(tmp_path / "odd.png")
    (tmp_path / "mixed.json").write_text(json.dumps({"slices": ["stack_0000.png", "odd.png"]}))
    cases["mixed"] = tmp_path / "mixed.json"
    (tmp_path / "sub").mkdir()
    Image.fromarray(np.zeros((8, 9), np.uint8)).save(tmp_path / "sub" / "odd.png")
    (tmp_path / "mixed_sub.json").write_text(json.dumps({"slices": ["stack_0000.png", "sub/odd.png"]}))
    cases["mixed_sub"] = tmp_path / "mixed_sub.json"
    code = ("import sys, json; sys.path.insert(0, %r)\n"
            "from ctprev.volume import load_slice_stack\n"
            "out = {}\n"
            "for k, p in json.loads(sys.argv[1]).items():\n"
            "    try:\n        v = load_slice_stack(p); out[k] = int(v.voxels.astype('int64').sum())\n"
            "    except Exception as e:\n        out[k] = type(e).__name__ + ': ' + str(e)\n"
            "print(json.dumps(out))\n") % str(REF)
    r = subprocess.run([sys.executable, "-c", code, json.dumps({k: str(p) for k, p in cases.items()})],
                       capture_output=True, text=True, env={"NUMBA_CACHE_DIR": "/tmp/numba_cache_ingest",
                                                            "PYTHONDONTWRITEBYTECODE": "1", "PATH": "/usr/bin"})
    ref = json.loads(r.stdout.strip().splitlines()[-1])
    from paper_2311_15038_b200.ingest import SliceStackReader, read_manifest
    for k, p in cases.items():
        try:
            paths, shape = read_manifest(p)
            out = np.zeros(shape, np.uint8)
            with SliceStackReader(paths, shape, threads=2) as rd:
                rd(0, shape[0], out)
            got = int(out.astype(np.int64).sum())
        except Exception as e:
            got = type(e).__name__ + ": " + str(e)
        assert got == ref[k], (k, got, ref[k])   # class AND message (volume.py:199 names the manifest entry)
