"""Why is the c4 MIP batch sometimes 1.08 and sometimes 1.84 ms/frame in bench.py?  Per-batch times with the SM
clock (NVML) sampled during each batch, under: a fresh process; after large torch allocations were freed
(empty_cache) before the row planes are allocated; after the GPU idled; after the host ran a CPU-heavy leg."""
import math, os, sys, threading, time
from pathlib import Path
sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
import numpy as np
import torch
import pynvml
from paper_2311_15038_b200 import _lib, device as dev, synth
from paper_2311_15038_b200.types import ViewParams

_lib.load()
pynvml.nvmlInit()
h = pynvml.nvmlDeviceGetHandleByIndex(0)
rows, stop = [], threading.Event()
def loop():
    while not stop.is_set():
        rows.append((time.time(), pynvml.nvmlDeviceGetClockInfo(h, pynvml.NVML_CLOCK_SM),
                     pynvml.nvmlDeviceGetClockInfo(h, pynvml.NVML_CLOCK_MEM),
                     pynvml.nvmlDeviceGetPowerUsage(h) / 1e3, pynvml.nvmlDeviceGetCurrentClocksEventReasons(h)))
        time.sleep(0.002)
threading.Thread(target=loop, daemon=True).start()

spec = synth.config("c4")
vol = synth.generate(spec)
steps = math.ceil(4 * math.sqrt(3.0) / 2.0 * 1024)
views = [ViewParams(azimuth_deg=10.0 * k, image_dim=1024, steps=steps, mode="mip") for k in range(36)]

def batches(tag, n=4):
    out = []
    for _ in range(n):
        w0 = time.time()
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record(); dev.render(vol, views, channels=4, fp32=True); b.record(); torch.cuda.synchronize()
        w1 = time.time()
        r = [x for x in rows if w0 <= x[0] <= w1]
        sm = int(np.median([x[1] for x in r])) if r else -1
        mem = int(np.median([x[2] for x in r])) if r else -1
        pw = int(max([x[3] for x in r])) if r else -1
        rs = 0
        for x in r: rs |= x[4]
        out.append(f"{a.elapsed_time(b) / 36:.3f}ms@{sm}/{mem}MHz/{pw}W/r{rs:x}")
    print(f"{tag:34s}", "  ".join(out), flush=True)

batches("fresh (first = plane alloc)", 6)
dev.render_release(); torch.cuda.empty_cache()
batches("after render_release", 12)
# big torch allocations freed before the planes are allocated again
dev.render_release()
junk = [torch.empty(1 << 30, dtype=torch.uint8, device="cuda") for _ in range(60)]
del junk[::2]; torch.cuda.empty_cache()
batches("planes among fragmented memory", 12)
del junk; dev.render_release(); torch.cuda.empty_cache()
batches("after freeing everything", 4)
time.sleep(10)
batches("after 10 s GPU idle", 6)
# CPU-heavy leg on all cores in a subprocess (like bench.py's cpu_baseline), GPU idle meanwhile
import subprocess
subprocess.run([sys.executable, "-c", "import numpy as np, concurrent.futures as cf\n"
                "def f(i):\n a=np.random.default_rng(i).integers(0,255,size=(64,1024,1024),dtype=np.uint8); return int(np.bincount(a.ravel()).sum())\n"
                "with cf.ProcessPoolExecutor(16) as ex: print(sum(ex.map(f, range(64))))"], capture_output=True)
batches("after a 16-process CPU leg", 6)
# pinned host memory held (like the e2e legs leave behind in torch's host cache)
pin = [torch.empty(1 << 30, dtype=torch.uint8, pin_memory=True) for _ in range(3)]
batches("with 3 GiB pinned host memory held", 4)
del pin
dev.render_release(); torch.cuda.empty_cache()
batches("planes re-allocated afterwards", 4)
stop.set()
