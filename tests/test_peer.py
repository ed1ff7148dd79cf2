"""The atlas gather fused into the pass: in peer mode every
rank > 0 maps rank 0's atlases through CUDA IPC and its fused kernel stores its
slab's cell rows there directly.  Two processes on ONE GPU (gloo for the host
collectives): the kernels never wait on one another -- each runs to completion
on its own, the gloo all-reduce orders them -- so this is a functional test of
the IPC path, not a timing one.  Rank 0's atlases must equal the single-process
step bit for bit after EVERY step of a multi-step run on different volumes (the
peer stores of step k+1 must not overwrite what rank 0 still reads of step k)."""
from __future__ import annotations

import os
import socket
import sys
from pathlib import Path

import pytest

ROOT = Path(__file__).resolve().parents[1]


def _free_port() -> int:
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


def _worker(rank, world, port, q):
    try:
        sys.path.insert(0, str(ROOT))
        os.environ["MASTER_ADDR"] = "127.0.0.1"
        os.environ["MASTER_PORT"] = str(port)
        import torch
        import torch.distributed as dist
        dist.init_process_group("gloo", rank=rank, world_size=world)
        torch.cuda.set_device(0)
        device = torch.device("cuda", 0)
        from paper_2311_15038_b200 import _lib, device as dev, synth
        from paper_2311_15038_b200.device import AtlasSpec
        from paper_2311_15038_b200.dist import DeviceSlabCompute, ShardedPreview
        from paper_2311_15038_b200.types import plan_scheme
        _lib.load()
        spec = synth.small((256, 256, 256), seed=3)
        schemes = {128: AtlasSpec.of(plan_scheme(128)), 64: AtlasSpec(64, 512, 8, 1)}
        level_of = {128: 1, 64: 2}
        fused = {1: schemes[128], 2: schemes[64]}
        sh = ShardedPreview(spec.shape, schemes, level_of, DeviceSlabCompute(torch.uint8, fused), rank, world,
                            device, peer_atlases=True)
        # several steps on DIFFERENT volumes, no barrier between them: rank 1 may run ahead
        # into step k+1 while rank 0 still checks step k's atlases -- the LUT all-reduce must
        # hold rank 1's stores into rank 0's atlases back until rank 0 has entered step k+1
        bad = []
        for k in range(3):
            spec_k = synth.small((256, 256, 256), seed=3 + k)
            slab = synth.generate(spec_k, z_range=(sh.z0, sh.z1), device=device)
            res = sh.step(slab)
            if rank == 0:
                torch.cuda.synchronize()
                got = {l: res["atlases"][l].clone() for l in (1, 2)}
                got_hist = res["hist"].clone()
                full = synth.generate(spec_k, device=device)
                outs, hist, _, _ = dev.preview_step(full, fused, 3, 0.0005)
                torch.cuda.synchronize()
                if not (torch.equal(got_hist, hist) and torch.equal(got[1], outs[1]) and torch.equal(got[2], outs[2])):
                    bad.append(k)
                del full
        if rank == 0:
            q.put(("ok" if not bad else f"mismatch at steps {bad}", (sh.z0, sh.z1)))
        dist.barrier()
        sh.close()
        dist.destroy_process_group()
    except Exception as e:  # pragma: no cover - reported to the parent
        q.put(("error", f"rank {rank}: {e!r}"))


def _render_worker(rank, world, port, q):
    try:
        sys.path.insert(0, str(ROOT))
        os.environ["MASTER_ADDR"] = "127.0.0.1"
        os.environ["MASTER_PORT"] = str(port)
        import math
        import torch
        import torch.distributed as dist
        dist.init_process_group("gloo", rank=rank, world_size=world)
        torch.cuda.set_device(0)
        device = torch.device("cuda", 0)
        from paper_2311_15038_b200 import _lib, device as dev, synth
        from paper_2311_15038_b200.dist import DeviceRenderCompute, ShardedRender
        from paper_2311_15038_b200.types import ViewParams
        _lib.load()
        spec = synth.small((192, 160, 176), seed=4)
        dim = 200
        views = [ViewParams(azimuth_deg=a, image_dim=dim, steps=math.ceil(4 * math.sqrt(3) / 2 * 192), mode=m)
                 for m in ("mip",) for a in (0.0, 70.0, 200.0)]
        sr = ShardedRender(spec.shape, dim, DeviceRenderCompute(), rank, world, device, peer_images=True)
        local = synth.generate(spec, z_range=(sr.h0, sr.h1), device=device)
        full = synth.generate(spec, device=device) if rank == 0 else None
        bad = []
        for k, az in enumerate((0.0, 35.0, 110.0)):  # batches of different views, no barrier between
            vk = [ViewParams(azimuth_deg=v.azimuth_deg + az, image_dim=dim, steps=v.steps, mode=v.mode) for v in views]
            out = sr.render(local, vk, channels=4, fp32=True)
            if rank == 0:
                torch.cuda.synchronize()
                got = out.clone()
                ref = dev.render(full, vk, channels=4, fp32=True)
                torch.cuda.synchronize()
                if not torch.equal(got, ref):
                    bad.append(k)
        if rank == 0:
            q.put(("ok" if not bad else f"mismatch at batches {bad}", (sr.bands, sr.held)))
        dist.barrier()
        sr.close()
        dist.destroy_process_group()
    except Exception as e:  # pragma: no cover - reported to the parent
        q.put(("error", f"rank {rank}: {e!r}"))


def _run_two(target):
    import torch.multiprocessing as mp
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=target, args=(r, 2, port, q)) for r in range(2)]
    for p in procs:
        p.start()
    for p in procs:
        p.join(timeout=280)
    status, info = q.get(timeout=5)
    assert status == "ok", info
    assert all(p.exitcode == 0 for p in procs)


@pytest.mark.gpu
@pytest.mark.timeout(300)
def test_peer_images_sort_last_two_processes_one_gpu(cuda):
    """Sort-last rendering with the composite fused into the render: each rank's kernel
    writes its row band of every view into rank 0's images through an IPC mapping."""
    _run_two(_render_worker)


@pytest.mark.gpu
@pytest.mark.timeout(300)
def test_peer_atlases_two_processes_one_gpu(cuda):
    import torch.multiprocessing as mp
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, 2, port, q)) for r in range(2)]
    for p in procs:
        p.start()
    for p in procs:
        p.join(timeout=280)
    status, info = q.get(timeout=5)
    assert status == "ok", info
    assert all(p.exitcode == 0 for p in procs)
