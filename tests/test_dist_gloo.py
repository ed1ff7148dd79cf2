"""z-slab sharding host logic at world_size 2 on the CPU (gloo).

The collective code path of paper_2311_15038_b200.dist.ShardedPreview (LUT
broadcast from the rank holding the top slices, int64 histogram all-reduce,
atlas byte-range gather to rank 0) runs unchanged; only the per-slab compute is
swapped for an oracle-backed stand-in, because there is no GPU here.  Rank 0
checks the gathered result against the oracle run on the whole volume.
"""
from __future__ import annotations

import os
import socket
import sys
from pathlib import Path

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

ROOT = Path(__file__).resolve().parents[1]


def _free_port() -> int:
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


class OracleSlabCompute:
    """Test-only SlabCompute: the CPU oracle on this rank's slab."""

    nbins = 256

    def __init__(self, schemes, level_of):
        self.schemes = schemes
        self.level_of = level_of

    def artifact_lut(self, top_slab, n_top, frac):
        from oracle import ctp_oracle as O
        bins = O.artifact_bins(top_slab.numpy(), n_top, frac)
        return torch.from_numpy(O.filter_lut(bins).copy())

    def fused(self, slab, lut, z_base, full_nz, hist, atlases):
        from oracle import ctp_oracle as O
        v = slab.numpy()
        hist += torch.from_numpy(O.histogram(v))
        f = O.apply_lut(v, lut.numpy())
        nz, ny, nx = v.shape
        for s, l in self.level_of.items():
            sp = self.schemes[s]
            lv = O.downscale(f, (nx >> l, ny >> l, nz >> l))
            a = atlases[l].numpy()
            per = sp.grid * sp.grid
            for kz in range(lv.shape[0]):
                k = (z_base >> l) + kz
                m, w = divmod(k, per)
                cy, cx = divmod(w, sp.grid)
                a[m, cy * sp.s:cy * sp.s + lv.shape[1], cx * sp.s:cx * sp.s + lv.shape[2]] = lv[kz]


def _worker(rank, world, port, q):
    try:
        sys.path.insert(0, str(ROOT))
        os.environ["MASTER_ADDR"] = "127.0.0.1"
        os.environ["MASTER_PORT"] = str(port)
        dist.init_process_group("gloo", rank=rank, world_size=world)
        from paper_2311_15038_b200.device import AtlasSpec
        from paper_2311_15038_b200.dist import ShardedPreview
        from oracle import ctp_oracle as O

        rng = np.random.default_rng(42)
        nz, ny, nx = 128, 128, 128
        vol = np.clip(np.rint(rng.normal(20, 6, (nz, ny, nx))), 0, 255).astype(np.uint8)
        vol[40:90, 10:50, 20:70] = rng.integers(120, 200, size=(50, 40, 50), dtype=np.uint8)
        vol[60:70] = rng.integers(0, 256, size=(10, ny, nx), dtype=np.uint8)
        schemes = {64: AtlasSpec(64, 512, 8, 1), 32: AtlasSpec(32, 256, 8, 1)}
        level_of = {64: 1, 32: 2}
        sh = ShardedPreview((nz, ny, nx), schemes, level_of, OracleSlabCompute(schemes, level_of), rank, world,
                            torch.device("cpu"))
        res = sh.step(torch.from_numpy(vol[sh.z0:sh.z1].copy()))
        if rank == 0:
            hist, bins, f, levels, atl = O.preview_pipeline(vol, [64, 32],
                                                            schemes=[(64, 512, 8, 1), (32, 256, 8, 1)])
            ok = np.array_equal(res["hist"].numpy(), hist)
            ok &= np.array_equal(res["lut"].numpy(), O.filter_lut(bins))
            ok &= np.array_equal(res["atlases"][1].numpy(), np.stack(atl[0]))
            ok &= np.array_equal(res["atlases"][2].numpy(), np.stack(atl[1]))
            q.put(("ok" if ok else "mismatch", (sh.z0, sh.z1)))
        dist.barrier()
        dist.destroy_process_group()
    except Exception as e:  # pragma: no cover - reported to the parent
        q.put(("error", repr(e)))


@pytest.mark.timeout(180)
@pytest.mark.parametrize("world", [2, 4])
def test_sharded_preview_gloo(world):
    """z-slab sharding (LUT broadcast from the top-slab owner, histogram all-reduce,
    atlas cell-row gather to rank 0) equals the whole-volume oracle bit for bit."""
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, world, port, q)) for r in range(world)]
    for p in procs:
        p.start()
    for p in procs:
        p.join(timeout=170)
    status, info = q.get(timeout=5)
    assert status == "ok", info
    assert all(p.exitcode == 0 for p in procs)


def test_slab_bounds_and_alignment():
    from paper_2311_15038_b200.device import AtlasSpec
    from paper_2311_15038_b200.dist import atlas_byte_range, slab_alignment, slab_bounds

    schemes = {512: AtlasSpec(512, 4096, 8, 8), 256: AtlasSpec(256, 2048, 8, 4), 128: AtlasSpec(128, 1024, 8, 2)}
    level_of = {512: 1, 256: 2, 128: 3}
    a = slab_alignment(schemes, level_of)
    assert a == 64  # whole level-3 cell rows of an 8-grid: 8 << 3
    for world in (1, 2, 4, 8):
        bounds = [slab_bounds(1024, world, r, a) for r in range(world)]
        assert bounds[0][0] == 0 and bounds[-1][1] == 1024
        assert all(b[1] == c[0] for b, c in zip(bounds, bounds[1:]))
        assert all((b[1] - b[0]) % a == 0 for b in bounds)
    # rank r's level-1 slices at 8 ranks are exactly atlas map r
    for r in range(8):
        z0, z1 = slab_bounds(1024, 8, r, a)
        assert atlas_byte_range(schemes[512], z0 >> 1, z1 >> 1) == (r * 4096 * 4096, (r + 1) * 4096 * 4096)
    with pytest.raises(ValueError):
        atlas_byte_range(schemes[512], 3, 64)


class OracleRenderCompute:
    """Test-only RenderCompute: the CPU oracle on a volume that holds ONLY this
    rank's slab -- every other slice is poisoned, so a row that read outside its
    rank's held slices would differ from the whole-volume render."""

    def render(self, slab, z_base, full_nz, views, rows, channels, fp32):
        from oracle import ctp_oracle as O
        v = slab.numpy()
        full = np.full((full_nz,) + v.shape[1:], 251, dtype=np.uint8)
        full[z_base:z_base + v.shape[0]] = v
        imgs = [_oracle_image(O, full, p) for p in views]
        return torch.from_numpy(np.stack(imgs)[:, rows[0]:rows[1]].copy())


def _oracle_image(O, vol, p):
    if p.mode == "mip":
        return O.render_mip(vol, p.azimuth_deg, p.image_dim, p.steps)
    return O.render_view(vol, p.azimuth_deg, p.image_dim, p.steps, p.mode, p.threshold)


def _render_worker(rank, world, port, q, replicated):
    try:
        sys.path.insert(0, str(ROOT))
        os.environ["MASTER_ADDR"] = "127.0.0.1"
        os.environ["MASTER_PORT"] = str(port)
        dist.init_process_group("gloo", rank=rank, world_size=world)
        from paper_2311_15038_b200.dist import ShardedRender
        from paper_2311_15038_b200.types import ViewParams
        from oracle import ctp_oracle as O

        rng = np.random.default_rng(7)
        nz, ny, nx = 40, 36, 44  # non-cubic: the rows of the image cover more than the volume
        vol = np.clip(np.rint(rng.normal(20, 6, (nz, ny, nx))), 0, 255).astype(np.uint8)
        zz, yy, xx = np.mgrid[:nz, :ny, :nx]
        shell = np.abs(np.sqrt(((zz - 19.5) / 15) ** 2 + ((yy - 17) / 13) ** 2 + ((xx - 22) / 17) ** 2) - 1.0) < 0.12
        vol[shell] = 180
        dim = 80  # rows finer than slices: the bands' edge rows need the halo (core-only slabs fail)
        views = [ViewParams(azimuth_deg=a, image_dim=dim, steps=64, mode=m, threshold=90)
                 for m in ("surface", "mip") for a in (0.0, 130.0)]
        sr = ShardedRender((nz, ny, nx), dim, OracleRenderCompute(), rank, world, torch.device("cpu"),
                           replicated=replicated)
        local = torch.from_numpy(vol[sr.h0:sr.h1].copy())
        out = sr.render(local, views, channels=1)
        if rank == 0:
            ref = np.stack([_oracle_image(O, vol, p) for p in views])
            ok = np.array_equal(out.numpy(), ref)
            q.put(("ok" if ok else "mismatch", (sr.bands, sr.held)))
        dist.barrier()
        dist.destroy_process_group()
    except Exception as e:  # pragma: no cover - reported to the parent
        q.put(("error", repr(e)))


@pytest.mark.timeout(240)
@pytest.mark.parametrize("replicated", [False, True])
def test_sharded_render_gloo_world2(replicated):
    """Sort-last z-slab rendering (row-band gather) and the replicated image-row split
    equal the whole-volume oracle images bit for bit."""
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_render_worker, args=(r, 2, port, q, replicated)) for r in range(2)]
    for p in procs:
        p.start()
    for p in procs:
        p.join(timeout=230)
    status, info = q.get(timeout=5)
    assert status == "ok", info
    assert all(p.exitcode == 0 for p in procs)


def test_row_bands_partition_and_halo():
    from paper_2311_15038_b200.dist import held_slices, row_band, row_slices, slab_bounds

    for shape, dim in (((1024, 1024, 1024), 1024), ((96, 80, 112), 64), ((2048, 1536, 1536), 512)):
        lo, hi = row_slices(shape, dim)
        for world in (1, 2, 4, 8):
            bands = [row_band(shape, dim, *slab_bounds(shape[0], world, r, 1)) for r in range(world)]
            rows = sorted(j for a, b in bands for j in range(a, b))
            assert rows == list(range(dim))
            for r, (a, b) in enumerate(bands):
                h0, h1 = held_slices(shape, dim, *slab_bounds(shape[0], world, r, 1))
                for j in range(a, b):
                    assert lo[j] > hi[j] or (h0 <= lo[j] and hi[j] < h1)
