import os, sys, time
sys.path.insert(0, '/root/repo')
import numpy as np, torch
from paper_2311_15038_b200 import hostio
a = np.random.default_rng(0).integers(0, 256, size=(1024, 1024, 1024), dtype=np.uint8)
dev = torch.device('cuda', 0)
for _ in range(3): hostio.h2d(a, dev); torch.cuda.synchronize()
ts = []
for _ in range(5):
    t0 = time.perf_counter(); t = hostio.h2d(a, dev); torch.cuda.synchronize(); ts.append(time.perf_counter() - t0)
print(f"bufs={hostio.NBUF} chunk={hostio.CHUNK>>20}MB h2d 1 GiB: {min(ts)*1e3:.1f} ms {a.nbytes/min(ts)/1e9:.1f} GB/s")
if os.environ.get("CTP_PROF_REGISTER") != "1": sys.exit(0)
# cudaHostRegister in place
cudart = torch.cuda.cudart()
ts=[]
for _ in range(3):
    t0 = time.perf_counter()
    r = cudart.cudaHostRegister(a.ctypes.data, a.nbytes, 0)
    t1 = time.perf_counter()
    g = torch.empty(a.shape, dtype=torch.uint8, device=dev)
    g.copy_(torch.from_numpy(a), non_blocking=True); torch.cuda.synchronize()
    t2 = time.perf_counter()
    cudart.cudaHostUnregister(a.ctypes.data)
    t3 = time.perf_counter()
    ts.append((t1-t0, t2-t1, t3-t2))
print("register/copy/unregister ms:", [tuple(round(x*1e3,1) for x in t) for t in ts])
