"""Host <-> device movement for the host-array drop-ins (``ops``).

The reference's entry points take and return host numpy arrays (volume.py:38-62:
``Volume.voxels`` is a frozen C-contiguous array; slicemap.py:95-110), so every
drop-in call crosses PCIe.  Two things keep that cost at the PCIe floor:

* ``DeviceCache`` -- a device-resident copy of every large FROZEN host array
  the drop-ins have uploaded or produced, keyed on the array object itself
  (weak reference: the entry dies with the array).  The reference freezes a
  Volume's voxels in place (volume.py:44-47: "pass a copy if the caller still
  needs to mutate it") and its callers chain results --
  ``f = filter_histogram_bins(v, bins)``, ``downscale_volume(f, ...)``,
  ``encode_slicemaps(level, ...)``, the three builders of one ``build_bundle``
  on one loaded volume -- so a chain uploads its volume ONCE and every later
  call starts from HBM.  Outputs are still fresh host arrays (the reference's
  contract); the cache only avoids re-uploading them.
* staged uploads of pageable arrays: chunks are copied into pinned staging
  buffers by a thread pool (numpy releases the GIL) while earlier chunks are
  already in flight on a copy stream; large outputs are read back straight
  into pinned memory (torch's caching host allocator), which the returned
  numpy array keeps alive.
"""
from __future__ import annotations

import os
import sys
import threading
import warnings
import weakref
from collections import OrderedDict
from concurrent.futures import ThreadPoolExecutor

import numpy as np
import torch

from . import trace

_NP2T = {np.dtype(np.uint8): torch.uint8, np.dtype(np.uint16): torch.uint16, np.dtype(np.int64): torch.int64,
         np.dtype(np.float32): torch.float32, np.dtype(np.float64): torch.float64, np.dtype(np.int32): torch.int32}

CACHE_MIN_BYTES = 1 << 20       # smaller arrays are cheaper to re-upload than to track
STAGE_MIN_BYTES = 8 << 20       # smaller uploads go straight through torch
PINNED_OUT_MIN_BYTES = 1 << 20  # smaller outputs are read back into pageable memory
# staging: NBUF pinned buffers of CHUNK bytes = NBUF concurrent memcpy threads; measured on the
# B200 box (16 host cores, tools/prof_h2d.py, 1 GiB pageable): 8 x 16 MB 35.9 GB/s, 8 x 32 MB
# 43-45 GB/s (PCIe pinned copy: 55 GB/s), 12 x 32 MB the same, 128 MB chunks 32 GB/s
# (round 2, tools/r2_h2d_parts.sh: filling each chunk with 2-8 pool tasks so the first DMA starts
# sooner changes nothing, 24.1-24.6 ms either way -- the host's memcpy rate beside the DMA reads
# is the bound, not the start-up of the pipeline)
CHUNK = int(os.environ.get("CTP_STAGE_CHUNK_MB", "32")) << 20
NBUF = int(os.environ.get("CTP_STAGE_BUFS", str(min(8, os.cpu_count() or 8))))


class DeviceCache:
    """Frozen host array -> its device copy, LRU within a byte budget."""

    def __init__(self, budget: int | None = None):
        env = os.environ.get("CTP_DEVICE_CACHE_BYTES")
        self.budget = int(env) if env is not None else (budget if budget is not None else 24 << 30)
        self.enabled = os.environ.get("CTP_DEVICE_CACHE", "1") != "0"
        self._lock = threading.Lock()
        self._entries: OrderedDict = OrderedDict()   # id(arr) -> (weakref(arr), tensor)
        self.bytes = 0
        self.hits = self.misses = 0

    @staticmethod
    def cacheable(arr: np.ndarray) -> bool:
        if not (isinstance(arr, np.ndarray) and arr.flags.c_contiguous and arr.nbytes >= CACHE_MIN_BYTES
                and arr.dtype in _NP2T):
            return False
        # frozen all the way down: a read-only VIEW of a writeable array (Volume(big[a:b])
        # freezes only the view, volume.py:60-62) can still change through its base -- unless
        # nothing but the view refers to that base any more (Volume(data.reshape(nz, ny, nx)),
        # volume.py:249: numpy collapses .base to the owner, so any other view or name of
        # the owner shows up in its reference count)
        b = arr.base
        while isinstance(b, np.ndarray):
            if b.flags.writeable and sys.getrefcount(b) > 3:  # arr.base + `b` + the argument
                return False
            b = b.base
        return not arr.flags.writeable

    def get(self, arr: np.ndarray, device) -> torch.Tensor | None:
        if not self.enabled or not self.cacheable(arr):
            return None
        with self._lock:
            e = self._entries.get(id(arr))
            if e is None or e[0]() is not arr or e[1].device != device or arr.flags.writeable:
                self.misses += 1
                return None
            self._entries.move_to_end(id(arr))
            self.hits += 1
            return e[1]

    def put(self, arr: np.ndarray, t: torch.Tensor) -> None:
        if not self.enabled or not self.cacheable(arr) or t.numel() * t.element_size() > self.budget:
            return
        key = id(arr)

        def _gone(_ref, key=key, cache=self):
            cache._drop(key)

        with self._lock:
            old = self._entries.pop(key, None)
            if old is not None:
                self.bytes -= old[1].numel() * old[1].element_size()
            self._entries[key] = (weakref.ref(arr, _gone), t)
            self.bytes += t.numel() * t.element_size()
            while self.bytes > self.budget and len(self._entries) > 1:
                _, (_, ev) = self._entries.popitem(last=False)
                self.bytes -= ev.numel() * ev.element_size()

    def _drop(self, key) -> None:
        with self._lock:
            e = self._entries.get(key)
            if e is not None and e[0]() is None:
                del self._entries[key]
                self.bytes -= e[1].numel() * e[1].element_size()

    def clear(self) -> None:
        with self._lock:
            self._entries.clear()
            self.bytes = 0


CACHE = DeviceCache()


class _Stager:
    """Pinned staging buffers + a copy stream per device, reused across uploads."""

    def __init__(self, device):
        self.device = device
        self.bufs = [torch.empty(CHUNK, dtype=torch.uint8, pin_memory=True) for _ in range(NBUF)]
        self.views = [b.numpy() for b in self.bufs]
        self.events = [None] * NBUF
        self.stream = torch.cuda.Stream(device)
        self.pool = ThreadPoolExecutor(max_workers=NBUF)
        self.lock = threading.Lock()


_STAGERS: dict = {}
_STAGERS_LOCK = threading.Lock()


def _stager(device) -> _Stager:
    with _STAGERS_LOCK:
        s = _STAGERS.get(device.index)
        if s is None:
            s = _STAGERS[device.index] = _Stager(device)
        return s


def h2d(arr: np.ndarray, device) -> torch.Tensor:
    """A device copy of a host array, ordered before later work on the current stream."""
    with trace.range("hostio.h2d"):
        return _h2d(arr, device)


def _h2d(arr: np.ndarray, device) -> torch.Tensor:
    a = np.ascontiguousarray(arr)
    dt = _NP2T.get(a.dtype)
    if dt is None:
        raise TypeError(f"no device dtype for {a.dtype}")
    if a.nbytes < STAGE_MIN_BYTES:
        with warnings.catch_warnings():
            warnings.simplefilter("ignore", UserWarning)  # non-writable numpy -> torch view (the copy never writes)
            return torch.from_numpy(a).to(device, non_blocking=False)
    out = torch.empty(a.shape, dtype=dt, device=device)
    src = a.reshape(-1).view(np.uint8)
    dst = out.view(-1).view(torch.uint8)
    st = _stager(device)
    cur = torch.cuda.current_stream(device)
    with st.lock:
        st.stream.wait_stream(cur)          # `out` was allocated on the current stream
        n = src.nbytes
        offs = list(range(0, n, CHUNK))
        futs = {}

        def fill(i):
            b = i % NBUF
            o = offs[i]
            m = min(CHUNK, n - o)
            np.copyto(st.views[b][:m], src[o:o + m])
            return m

        def submit(i):
            b = i % NBUF
            if st.events[b] is not None:
                st.events[b].synchronize()  # the DMA out of this staging buffer has finished
            futs[i] = st.pool.submit(fill, i)

        for i in range(min(NBUF, len(offs))):
            submit(i)
        for i, o in enumerate(offs):
            m = futs.pop(i).result()
            b = i % NBUF
            with torch.cuda.stream(st.stream):
                dst[o:o + m].copy_(st.bufs[b][:m], non_blocking=True)
                ev = torch.cuda.Event()
                ev.record(st.stream)
                st.events[b] = ev
            if i + NBUF < len(offs):
                submit(i + NBUF)
        cur.wait_stream(st.stream)
        out.record_stream(st.stream)
    return out


def d2h(t: torch.Tensor) -> np.ndarray:
    """A fresh host array of a device tensor (synchronous).  Large ones land in pinned
    memory, which the returned array keeps alive."""
    if t.numel() * t.element_size() < PINNED_OUT_MIN_BYTES:
        return t.cpu().numpy()
    with trace.range("hostio.d2h"):
        return _d2h_pinned(t)


def _d2h_pinned(t: torch.Tensor) -> np.ndarray:
    h = torch.empty(t.shape, dtype=t.dtype, pin_memory=True)
    h.copy_(t, non_blocking=True)
    torch.cuda.current_stream(t.device).synchronize()
    return h.numpy()


def d2h_frozen(t: torch.Tensor) -> np.ndarray:
    """``d2h`` for a result the reference wraps in a frozen Volume: the array is frozen
    here (Volume would freeze it in place anyway, volume.py:60-62) and its device copy
    stays cached, so a drop-in called on it next starts from HBM."""
    a = d2h(t)
    a.setflags(write=False)
    CACHE.put(a, t)
    return a
