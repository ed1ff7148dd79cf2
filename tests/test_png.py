"""Atlas PNG writing: the device scanline filter against the
oracle restatement, the parallel-deflate PNG container against Pillow (lossless
round trip), and save_slicemaps' files + manifest against the reference's."""
from __future__ import annotations

import io
import json

import numpy as np
import pytest

from oracle import ctp_oracle as O


def _images():
    rng = np.random.default_rng(8)
    smooth = np.clip(np.cumsum(rng.integers(-3, 4, size=(3, 70, 93)), axis=2) + 128, 0, 255).astype(np.uint8)
    noise = rng.integers(0, 256, size=(3, 70, 93), dtype=np.uint8)
    flat = np.zeros((3, 70, 93), dtype=np.uint8)
    flat[:, 20:40, 10:50] = 77
    return np.concatenate([smooth, noise, flat])


def _png_filter_unfilter_roundtrip(filt):
    """Undo PNG filters (spec semantics) -- independent of the encoder under test."""
    h, w1 = filt.shape
    w = w1 - 1
    out = np.zeros((h, w), dtype=np.int64)
    for y in range(h):
        f = int(filt[y, 0])
        r = filt[y, 1:].astype(np.int64)
        b = out[y - 1] if y > 0 else np.zeros(w, dtype=np.int64)
        row = np.zeros(w, dtype=np.int64)
        for x in range(w):
            a = row[x - 1] if x > 0 else 0
            c = b[x - 1] if x > 0 else 0
            if f == 0:
                pr = 0
            elif f == 1:
                pr = a
            elif f == 2:
                pr = b[x]
            elif f == 3:
                pr = (a + b[x]) >> 1
            else:
                p = a + b[x] - c
                pa, pb, pc = abs(p - a), abs(p - b[x]), abs(p - c)
                pr = a if (pa <= pb and pa <= pc) else (b[x] if pb <= pc else c)
            row[x] = (r[x] + pr) & 0xFF
        out[y] = row
    return out.astype(np.uint8)


def test_oracle_png_filter_inverts():
    for img in _images()[::3]:
        for flt in (-1, 0, 1, 2, 3, 4):
            f = O.png_filter(img, flt)
            assert f.shape == (img.shape[0], img.shape[1] + 1) and set(np.unique(f[:, 0])) <= set(range(5))
            assert flt < 0 or set(np.unique(f[:, 0])) == {flt}
            assert np.array_equal(_png_filter_unfilter_roundtrip(f), img)


def test_png_container_decodes_with_pillow():
    from PIL import Image
    from paper_2311_15038_b200.png import png_from_filtered
    for img in _images():
        for rows in (1, 7, 256):
            data = png_from_filtered(O.png_filter(img), level=6, block_rows=rows)
            with Image.open(io.BytesIO(data)) as im:
                assert im.mode == "L" and im.size == (img.shape[1], img.shape[0])
                assert np.array_equal(np.asarray(im), img)


@pytest.mark.gpu
def test_device_png_filter_equals_oracle(cuda):
    """Every fixed filter bit for bit; the adaptive (entropy) choice decodes exactly and
    agrees with the oracle's choice on the rows that are not near-ties."""
    import torch
    from paper_2311_15038_b200 import device as dev
    imgs = _images()
    t = torch.from_numpy(imgs).to(cuda)
    for flt in range(5):
        got = dev.png_filter(t, filter=flt).cpu().numpy()
        for i in range(imgs.shape[0]):
            assert np.array_equal(got[i], O.png_filter(imgs[i], flt)), (flt, i)
    got = dev.png_filter(t).cpu().numpy()
    agree = 0
    for i in range(imgs.shape[0]):
        assert np.array_equal(_png_filter_unfilter_roundtrip(got[i]), imgs[i]), i
        agree += int((got[i][:, 0] == O.png_filter(imgs[i])[:, 0]).sum())
    assert agree >= 0.95 * imgs.shape[0] * imgs.shape[1]


@pytest.mark.gpu
def test_save_slicemaps_roundtrip(cuda, tmp_path):
    """save_slicemaps: the reference's file names and manifest; every atlas decodes
    (Pillow, as load_slicemaps does) to the same bytes -- c1-sized 4096^2 atlas."""
    from PIL import Image
    import paper_2311_15038_b200 as P
    from paper_2311_15038_b200.png import save_slicemaps
    rng = np.random.default_rng(2)
    vol = np.clip(np.rint(rng.normal(20, 6, (256, 256, 256))), 0, 255).astype(np.uint8)
    vol[100:160, 60:200, 80:180] = 170
    sset = P.encode_slicemaps(P.Volume(vol), P.SlicemapScheme(256, 4096, 16, 1))
    mp = save_slicemaps(sset, tmp_path / "sm")
    man = json.loads(mp.read_text())
    assert man == {"scheme": {"s": 256, "atlas": 4096, "grid": 16, "maps": 1}, "atlases": ["sm_256_0.png"]}
    with Image.open(tmp_path / "sm" / "sm_256_0.png") as im:
        assert im.mode == "L" and np.array_equal(np.asarray(im), sset.atlases[0])


@pytest.mark.gpu
def test_device_deflate_streams(cuda):
    """ctp_deflate_u8 + host assembly: valid zlib streams (zlib.decompress gives back the
    filtered bytes exactly) and PNGs Pillow decodes to the images, for zeros (matches
    only), noise (stored blocks), smooth data (dynamic Huffman + matches), several chunks
    per image with a partial last chunk, and a one-row image."""
    import zlib
    import torch
    from PIL import Image
    from paper_2311_15038_b200 import device as dev
    from paper_2311_15038_b200.png import deflate_device, encode_pngs_device
    rng = np.random.default_rng(4)
    cases = [np.zeros((3, 40, 57), np.uint8), rng.integers(0, 256, (2, 150, 301), dtype=np.uint8),
             np.clip(np.cumsum(rng.integers(-3, 4, (2, 300, 517)), axis=2) + 128, 0, 255).astype(np.uint8),
             np.full((1, 1, 70000), 9, np.uint8)]
    imgs = _images()
    cases.append(imgs)
    for c in cases:
        t = torch.from_numpy(np.ascontiguousarray(c)).to(cuda)
        filt = dev.png_filter(t)
        for i, z in enumerate(deflate_device(filt)):
            assert zlib.decompress(z) == filt[i].cpu().numpy().tobytes(), (c.shape, i)
        for i, p in enumerate(encode_pngs_device(c)):
            with Image.open(io.BytesIO(p)) as im:
                assert np.array_equal(np.asarray(im), c[i]), (c.shape, i)


@pytest.mark.gpu
def test_save_slicemaps_device_compressor(cuda, tmp_path):
    from PIL import Image
    import paper_2311_15038_b200 as P
    from paper_2311_15038_b200.png import save_slicemaps
    rng = np.random.default_rng(6)
    vol = np.clip(np.rint(rng.normal(20, 6, (128, 128, 128))), 0, 255).astype(np.uint8)
    sset = P.encode_slicemaps(P.Volume(vol), P.plan_scheme(128))
    mp = save_slicemaps(sset, tmp_path / "sm", compressor="device")
    assert json.loads(mp.read_text()) == sset.manifest()
    for m, name in enumerate(sset.scheme.atlas_names()):
        with Image.open(tmp_path / "sm" / name) as im:
            assert np.array_equal(np.asarray(im), sset.atlases[m])
