"""Build the in-tree CUDA library ``_lib/libctprev_b200.so`` for sm_100a.

Plain nvcc, one object per translation unit, linked into one shared library
with the C ABI of ``include/ctprev_b200.h``.  Run ``python -m
paper_2311_15038_b200._build`` (or ``__graft_entry__.build()``).
"""
from __future__ import annotations

import concurrent.futures as cf
import os
import shutil
import subprocess
import sys
from pathlib import Path

PKG = Path(__file__).resolve().parent
CSRC = PKG / "csrc"
OUT_DIR = PKG / "_lib"
LIB = OUT_DIR / "libctprev_b200.so"
ARCH = ["-gencode", "arch=compute_100a,code=sm_100a"]
COMMON = ["-O3", "-lineinfo", "-std=c++17", "-Xcompiler", "-fPIC", "-Xptxas", "-v"]
COMMON += os.environ.get("CTP_NVCC_EXTRA", "").split()  # variant experiments (tools/), e.g. -DCTP_U16_COLS=8
# render.cu: the fp64 path must not contract a*b+c into FMA, so that its
# arithmetic matches numba's fastmath-free reference bit for bit.
PER_FILE = {"render.cu": ["--fmad=false"]}
SOURCES = ["ctp_common.cu", "hist.cu", "preview.cu", "resample.cu", "render.cu", "synth.cu", "png.cu", "deflate.cu", "ipc.cu"]


def _nvcc() -> str:
    for cand in (shutil.which("nvcc"), "/usr/local/cuda/bin/nvcc"):
        if cand and os.path.exists(cand):
            return cand
    raise RuntimeError("nvcc not found")


def _compile(src: str, build_dir: Path, verbose: bool) -> Path:
    obj = build_dir / (src.replace(".cu", ".o"))
    cmd = [_nvcc(), *ARCH, *COMMON, *PER_FILE.get(src, []), "-c", str(CSRC / src), "-o", str(obj)]
    res = subprocess.run(cmd, capture_output=True, text=True)
    if res.returncode != 0:
        raise RuntimeError(f"nvcc failed for {src}:\n{res.stdout}\n{res.stderr}")
    (build_dir / (src + ".ptxas.txt")).write_text(res.stderr)
    if verbose:
        print(f"[build] {src}")
    return obj


def build(verbose: bool = True, force: bool = False) -> Path:
    build_dir = PKG / "csrc" / "build"
    build_dir.mkdir(parents=True, exist_ok=True)
    OUT_DIR.mkdir(parents=True, exist_ok=True)
    srcs = [CSRC / s for s in SOURCES] + list(CSRC.glob("*.cuh")) + [PKG.parent / "include" / "ctprev_b200.h"]
    if LIB.exists() and not force:
        newest = max(p.stat().st_mtime for p in srcs)
        if LIB.stat().st_mtime > newest:
            if verbose:
                print(f"[build] up to date: {LIB}")
            return LIB
    with cf.ThreadPoolExecutor(max_workers=min(8, os.cpu_count() or 1)) as ex:
        objs = list(ex.map(lambda s: _compile(s, build_dir, verbose), SOURCES))
    tmp = LIB.with_suffix(".so.tmp")
    cmd = [_nvcc(), *ARCH, "-shared", "-o", str(tmp), *map(str, objs), "-cudart=static"]
    res = subprocess.run(cmd, capture_output=True, text=True)
    if res.returncode != 0:
        raise RuntimeError(f"link failed:\n{res.stdout}\n{res.stderr}")
    os.replace(tmp, LIB)
    if verbose:
        print(f"[build] wrote {LIB}")
    return LIB


if __name__ == "__main__":
    build(verbose=True, force="--force" in sys.argv)
