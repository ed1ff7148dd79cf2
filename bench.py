"""Benchmark: the preview data-reduction hot path on B200 (BASELINE.json metric).

Headline workload = BASELINE config 2: a 1024^3 uint8 volume (seeded synthetic
stand-in for a NOVA scan), one step = volume_histogram + artifact_bins +
filter_histogram_bins + the 512^3/256^3/128^3 levels (each direct from the
filtered volume) + their slicemap atlases (8x4096^2, 4x2048^2, 2x1024^2).
value = GVoxel/s with the volume resident in HBM; e2e = the same through the
host-buffer session (pinned host volume in, pinned host atlases out, PCIe
copies inside the timed region).  A secondary ``mip`` object reports config-4
MIP frames/s (36 azimuths, 1024^2, 0.5-voxel steps over a 1024^3 volume).

Multi-GPU (torchrun): every rank owns a 1024-slice z-slab of one (N*1024)-deep
volume (weak scaling, slab height a multiple of 2^levels => no halo); the
artifact LUT is broadcast from the rank holding the top slices and the
histograms are summed with an NCCL all-reduce.

``--impl reference``: the reference's CPU algorithm (the oracle port of
ctprev's numpy code) fanned out over z-slabs on all host cores.
"""
from __future__ import annotations

import argparse
import json
import os
import statistics
import subprocess
import sys
import threading
import time
from pathlib import Path

ROOT = Path(__file__).resolve().parent
sys.path.insert(0, str(ROOT))

METRIC = "pipeline GVoxel/s (hist+filter+slicemaps) & MIP frames/s, % of HBM roofline"
SCHEMES = (512, 256, 128)


def _peaks():
    try:
        return json.loads((ROOT / "MEASURED_PEAKS.json").read_text()), "measured"
    except Exception:
        return {"hbm_gbs": 6650.0, "sm_max_mhz": 1965.0}, "fallback"


class ClockSampler:
    """nvidia-smi clocks + throttle reasons sampled during the timed region."""

    FIELDS = ("index,clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.active,"
              "clocks_event_reasons.hw_slowdown,clocks_event_reasons.hw_thermal_slowdown,"
              "clocks_event_reasons.sw_thermal_slowdown,clocks_event_reasons.sw_power_cap")

    def __init__(self, gpu_index: int):
        self.gpu = gpu_index
        self.rows = []
        self._stop = threading.Event()
        self._t = None

    def _run(self):
        while not self._stop.is_set():
            try:
                out = subprocess.run(["nvidia-smi", "-i", str(self.gpu), f"--query-gpu={self.FIELDS}",
                                      "--format=csv,noheader,nounits"], capture_output=True, text=True, timeout=5)
                if out.returncode == 0 and out.stdout.strip():
                    self.rows.append([x.strip() for x in out.stdout.strip().split(",")])
            except Exception:
                pass
            self._stop.wait(0.1)

    def __enter__(self):
        self._t = threading.Thread(target=self._run, daemon=True)
        self._t.start()
        return self

    def __exit__(self, *a):
        self._stop.set()
        if self._t:
            self._t.join(timeout=10)

    def summary(self):
        if not self.rows:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["nvidia-smi unavailable"], "samples": 0}
        sm = [float(r[1]) for r in self.rows if r[1].replace(".", "").isdigit()]
        mx = [float(r[2]) for r in self.rows if r[2].replace(".", "").isdigit()]
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        reasons = sorted({n for r in self.rows for n, v in zip(names, r[5:9]) if v.lower() == "active"})
        return {"sm_mhz": statistics.median(sm) if sm else None, "sm_max_mhz": max(mx) if mx else None,
                "reasons": reasons, "samples": len(self.rows)}


# ---------------------------------------------------------------------------
# CPU reference (oracle port of ctprev's numpy algorithm), process pool over z-slabs

_CPU_VOL = None


def _cpu_slab(args):
    z0, z1, lut = args
    import numpy as np
    from oracle import ctp_oracle as O
    v = _CPU_VOL[z0:z1]
    h = O.histogram(v)                                   # volume.py:252-262 per slab (exact sum)
    f = O.apply_lut(v, lut)                              # mask.py:246
    nz, ny, nx = v.shape
    out = []
    for s in SCHEMES:                                    # pipeline.py:275 direct from f, slab-separable
        r = _CPU_VOL.shape[2] // s
        out.append(O.downscale(f, (nx // r, ny // r, nz // r)))
    return z0, h, out


def cpu_reference_pass(vol, z_lo: int, z_hi: int, workers: int, pool=None):
    """hist + bins (top slab of the FULL volume) + filter + 3 levels + atlas packing of
    slices [z_lo, z_hi).  Returns voxels processed."""
    import numpy as np
    from oracle import ctp_oracle as O
    bins = O.artifact_bins(vol)                          # mask.py:215-231 (top 3 slices)
    lut = O.filter_lut(bins)
    slab = 64
    tasks = [(z, min(z + slab, z_hi), lut) for z in range(z_lo, z_hi, slab)]
    results = pool.map(_cpu_slab, tasks) if pool else list(map(_cpu_slab, tasks))
    hist = np.zeros(256, dtype=np.int64)
    levels = {s: np.zeros((vol.shape[0] * s // vol.shape[2], s, s), dtype=np.uint8) for s in SCHEMES}
    for z0, h, out in results:
        hist += h
        for s, lv in zip(SCHEMES, out):
            r = vol.shape[2] // s
            levels[s][z0 // r: z0 // r + lv.shape[0]] = lv
    for s in SCHEMES:                                    # slicemap.py:132-141 packing
        sc = O.plan_scheme(s)
        g = sc[2]
        for m in range(sc[3]):
            blk = levels[s][m * g * g:(m + 1) * g * g]
            _ = blk.reshape(g, g, s, s).transpose(0, 2, 1, 3).reshape(g * s, g * s).copy()
    return (z_hi - z_lo) * vol.shape[1] * vol.shape[2]


def run_reference(args):
    rank = int(os.environ.get("RANK", "0"))
    if rank != 0:
        return 0
    import multiprocessing as mp
    import numpy as np
    global _CPU_VOL
    workers = os.cpu_count() or 1
    # the same synthetic volume as the GPU arm (generated on the GPU if present, else on the host)
    try:
        import torch
        from paper_2311_15038_b200 import synth
        if torch.cuda.is_available():
            _CPU_VOL = synth.generate(synth.config("c2")).cpu().numpy()
            torch.cuda.empty_cache()
    except Exception:
        _CPU_VOL = None
    if _CPU_VOL is None:
        rng = np.random.default_rng(0)
        _CPU_VOL = np.clip(np.rint(rng.normal(20, 6, (1024, 1024, 1024)).astype(np.float32)), 0, 255).astype(np.uint8)
    sample = 256  # slices per step (a quarter of the volume) keeps a step at a few seconds
    ctx = mp.get_context("fork")
    with ctx.Pool(workers) as pool:
        for _ in range(args.warmup):
            cpu_reference_pass(_CPU_VOL, 0, sample, workers, pool)
        t0 = time.perf_counter()
        vox = 0
        for i in range(args.steps):
            z0 = (i * sample) % 1024
            vox += cpu_reference_pass(_CPU_VOL, z0, z0 + sample, workers, pool)
        dt = time.perf_counter() - t0
    v = vox / dt / 1e9
    line = {"metric": METRIC, "value": v, "unit": "GVoxel/s", "n_gpus": args.gpus, "steps": args.steps,
            "warmup": args.warmup, "ms_per_step": dt / args.steps * 1e3, "higher_is_better": True,
            "scaling": "weak", "vs_baseline": None, "dtype": "u8", "data": "synthetic (config-2 generator)",
            "impl": "reference",
            "config": {"workload": "c2: 1024^3 u8 hist+filter+3-level pyramid+atlases", "sample_slices": sample},
            "cpu_baseline": {"value": v, "unit": "GVoxel/s", "cores": workers, "kind": "port",
                             "sample": f"{sample} of 1024 z-slices per step (hist/bins/filter/levels/atlases), "
                                       f"numpy oracle port of ctprev, process pool over 64-slice slabs"},
            "e2e": {"value": v, "unit": "GVoxel/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0}}
    print(json.dumps(line))
    return 0


# ---------------------------------------------------------------------------
# GPU arm

def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=200)
    ap.add_argument("--warmup", type=int, default=10)
    ap.add_argument("--impl", default="b200", choices=["b200", "reference"])
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--no-mip", action="store_true")
    ap.add_argument("--mip-batches", type=int, default=1)
    args = ap.parse_args()
    if args.impl == "reference":
        return run_reference(args)

    import numpy as np
    import torch
    import torch.distributed as dist

    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    torch.cuda.set_device(local)
    device = torch.device("cuda", local)
    if world > 1:
        dist.init_process_group("nccl", device_id=device)

    from paper_2311_15038_b200 import _lib, device as dev, synth
    from paper_2311_15038_b200.pipeline import PreviewSession, plan_preview, run_preview
    from paper_2311_15038_b200.device import AtlasSpec
    from paper_2311_15038_b200.types import plan_scheme

    _lib.load()
    spec = synth.config("c2")
    nz, ny, nx = spec.shape
    full_nz = nz * world
    z_base = rank * nz
    # this rank's z-slab of the (world*1024)-deep volume
    vol = synth.generate(synth.SynthSpec((full_nz, ny, nx), spec.dtype, spec.seed, spec.n_shells, spec.bg_mean,
                                         spec.bg_sd, spec.shell_mean, spec.shell_sd, spec.axes, spec.thickness,
                                         spec.speckle_p), z_range=(z_base, z_base + nz), device=device)
    schemes = {s: AtlasSpec.of(plan_scheme(s)) for s in SCHEMES}
    plan = plan_preview((nz, ny, nx), schemes)
    assert not plan.general and plan.nlev == 3
    hist = torch.zeros(256, dtype=torch.int64, device=device)
    top_owner = world - 1
    stream = torch.cuda.current_stream()
    ev_k0 = [torch.cuda.Event(enable_timing=True) for _ in range(args.steps)]
    ev_k1 = [torch.cuda.Event(enable_timing=True) for _ in range(args.steps)]
    outs_cache = {}

    def step(i=None):
        # LUT from the top slices of the WHOLE volume (mask.py:227): owned by the last rank
        if rank == top_owner:
            lut, flags = dev.artifact_lut(vol, 3, 0.0005)
        else:
            lut = torch.empty(256, dtype=torch.uint8, device=device)
        if world > 1:
            dist.broadcast(lut, src=top_owner)
        hist.zero_()
        if i is not None:
            ev_k0[i].record(stream)
        outs = dev.preview(vol, lut, plan.fused, hist=hist, z_base=z_base, full_nz=full_nz,
                           out_tensors=outs_cache)
        if i is not None:
            ev_k1[i].record(stream)
        outs_cache.update(outs)
        if world > 1:
            dist.all_reduce(hist)
        return outs

    # warmup
    for _ in range(args.warmup):
        step()
    torch.cuda.synchronize()
    if world > 1:
        dist.barrier()
    _lib.launch_count(reset=True)
    sampler = ClockSampler(local)
    with sampler:
        torch.cuda.synchronize()
        if world > 1:
            dist.barrier()
        t0 = torch.cuda.Event(enable_timing=True)
        t1 = torch.cuda.Event(enable_timing=True)
        t0.record(stream)
        for i in range(args.steps):
            step(i)
        t1.record(stream)
        torch.cuda.synchronize()
        if world > 1:
            dist.barrier()
    launches = _lib.launch_count()
    ms = t0.elapsed_time(t1)
    kern_ms = [a.elapsed_time(b) for a, b in zip(ev_k0, ev_k1)]
    ms_t = torch.tensor([ms], dtype=torch.float64, device=device)
    if world > 1:
        dist.all_reduce(ms_t, op=dist.ReduceOp.MAX)
    ms = float(ms_t.item())
    voxels_total = nx * ny * nz * world * args.steps
    value = voxels_total / (ms * 1e-3) / 1e9

    # roofline of the dominant kernel (the fused pass): algorithmic bytes per launch
    atlas_bytes = sum(t.numel() for t in outs_cache.values())
    alg_bytes = nx * ny * nz + atlas_bytes
    kmean = statistics.mean(kern_ms)
    peaks, peak_src = _peaks()
    achieved = alg_bytes / (kmean * 1e-3) / 1e9
    traffic = None
    tfile = ROOT / "profiles" / "traffic_fused_c2.json"
    if tfile.exists():
        try:
            traffic = json.loads(tfile.read_text()).get("dram_bytes_per_launch")
        except Exception:
            traffic = None

    # correctness spot check of this very run (hist total)
    assert int(hist.sum().item()) == nx * ny * nz * world

    # ---- e2e through the host-buffer session (rank-local slab, pinned host memory)
    e2e = None
    if True:
        sess = PreviewSession((nz, ny, nx), torch.uint8, schemes, chunk_slices=64, device=device)
        host = torch.empty((nz, ny, nx), dtype=torch.uint8, pin_memory=True)
        host.copy_(vol)
        for _ in range(2):
            sess.run(host)
        e_steps = max(3, min(10, args.steps))
        torch.cuda.synchronize()
        if world > 1:
            dist.barrier()
        w0 = time.perf_counter()
        for _ in range(e_steps):
            r = sess.run(host)
        torch.cuda.synchronize()
        e_s = time.perf_counter() - w0
        et = torch.tensor([e_s], dtype=torch.float64, device=device)
        if world > 1:
            dist.all_reduce(et, op=dist.ReduceOp.MAX)
        e_s = float(et.item())
        e2e = {"value": nx * ny * nz * world * e_steps / e_s / 1e9, "unit": "GVoxel/s",
               "h2d_bytes_per_step": sess.h2d_bytes, "d2h_bytes_per_step": sess.d2h_bytes,
               "steps": e_steps, "path": "PreviewSession: pinned host volume -> z-chunk streamed H2D / fused "
                                         "pass / atlas D2H on 3 streams"}
        del sess, host
        torch.cuda.empty_cache()

    # ---- CPU baseline (rank 0, N=1 only): oracle port on all host cores, bounded sample
    cpu = None
    if rank == 0 and world == 1 and not args.no_cpu_baseline:
        import multiprocessing as mp
        global _CPU_VOL
        _CPU_VOL = vol.cpu().numpy()
        workers = os.cpu_count() or 1
        with mp.get_context("fork").Pool(workers) as pool:
            cpu_reference_pass(_CPU_VOL, 0, 64, workers, pool)
            c0 = time.perf_counter()
            n = cpu_reference_pass(_CPU_VOL, 0, 256, workers, pool)
            c_s = time.perf_counter() - c0
        cpu = {"value": n / c_s / 1e9, "unit": "GVoxel/s", "cores": workers, "kind": "port",
               "sample": "256 of 1024 z-slices of the same c2 volume: hist + artifact bins + filter + 512/256/128 "
                         "levels + atlas packing (numpy oracle port of ctprev, process pool over 64-slice slabs)",
               "seconds": c_s}
        _CPU_VOL = None

    # ---- MIP frames/s (config 4), rank 0 image-tile split across ranks
    mip = None
    if not args.no_mip:
        mip = bench_mip(args, device, rank, world, dist)

    if rank == 0:
        line = {
            "metric": METRIC, "value": value, "unit": "GVoxel/s", "n_gpus": world, "steps": args.steps,
            "warmup": args.warmup, "ms_per_step": ms / args.steps, "higher_is_better": True, "scaling": "weak",
            "vs_baseline": None, "dtype": "u8", "data": "synthetic (seeded config-2 generator, on device)",
            "config": {"workload": "c2: 1024^3 u8/GPU, hist + artifact-bin filter + 512/256/128 levels + "
                                   "slicemap atlases (8x4096^2, 4x2048^2, 2x1024^2)",
                       "voxels_per_gpu": nx * ny * nz, "parallelism": f"z-slab x{world}",
                       "l2": "input 1 GiB per step > 126 MB L2 (no flush needed)"},
            "roofline": {"bound": "hbm", "achieved": achieved, "peak": peaks["hbm_gbs"], "unit": "GB/s",
                         "frac": achieved / peaks["hbm_gbs"], "traffic": traffic,
                         "kernel": "preview_kernel<uint8_t,3>", "kernel_ms": kmean,
                         "alg_bytes_per_launch": alg_bytes, "peak_source": peak_src},
            "cpu_baseline": cpu,
            "e2e": e2e,
            "gpu_launches": launches,
            "clocks": sampler.summary(),
            "mip": mip,
        }
        print(json.dumps(line))
    if world > 1:
        dist.destroy_process_group()
    return 0


def bench_mip(args, device, rank, world, dist):
    import torch
    from paper_2311_15038_b200 import device as dev, synth
    from paper_2311_15038_b200.types import ViewParams
    spec = synth.config("c4")
    vol = synth.generate(spec, device=device)
    n = spec.shape[0]
    dim = 1024
    import math
    steps = math.ceil(4 * math.sqrt(3.0) / 2.0 * n)  # 0.5-voxel step over the 2R window: 3548 for 1024^3
    views = [ViewParams(azimuth_deg=10.0 * k, image_dim=dim, steps=steps, mode="mip") for k in range(36)]
    rows = (rank * dim // world, (rank + 1) * dim // world)   # image-tile split, volume replicated
    out = torch.empty((36, rows[1] - rows[0], dim, 4), dtype=torch.uint8, device=device)
    dev.render(vol, views, channels=4, fp32=True, rows=rows, out=out)   # warmup
    torch.cuda.synchronize()
    if world > 1:
        dist.barrier()
    a = torch.cuda.Event(enable_timing=True)
    b = torch.cuda.Event(enable_timing=True)
    a.record()
    for _ in range(args.mip_batches):
        dev.render(vol, views, channels=4, fp32=True, rows=rows, out=out)
    b.record()
    torch.cuda.synchronize()
    ms = a.elapsed_time(b)
    t = torch.tensor([ms], dtype=torch.float64, device=device)
    if world > 1:
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
    ms = float(t.item())
    frames = 36 * args.mip_batches
    samples = frames * dim * dim * steps
    del vol
    torch.cuda.empty_cache()
    return {"value": frames / (ms * 1e-3), "unit": "frames/s", "ms_per_frame": ms / frames,
            "gsamples_per_s": samples / (ms * 1e-3) / 1e9, "steps_per_ray": steps, "image": "1024^2 RGBA8",
            "volume": "1024^3 u8 (config-4 generator)", "views": 36, "batches": args.mip_batches,
            "precision": "fp32 trilinear", "hbm_frac": (spec.nbytes * frames / (ms * 1e-3) / 1e9) / _peaks()[0]["hbm_gbs"]}


if __name__ == "__main__":
    sys.exit(main())
