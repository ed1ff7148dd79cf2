"""Summarise tools/profile_round2.sh (gpurun_out/prof2/) into profiles/.

usage: python tools/summarise_r02.py [--tag r02]

Writes <tag>_bench.jsonl, <tag>_bench_reference.jsonl, <tag>_bench_launches.txt (per-kernel
share of the ncu launch list), <tag>_kernels_ncu.txt (every captured kernel: duration, DRAM
bytes, achieved GB/s against the measured HBM peak, issue / shared-pipe utilisation, shared
wavefronts per instruction) and traffic_fused_c2.json (DRAM bytes per launch of the c2 step
kernel, read by bench.py's roofline).  Needs ncu on PATH for the .ncu-rep files.
"""
from __future__ import annotations

import argparse
import collections
import csv
import io
import json
import subprocess
from pathlib import Path

ROOT = Path(__file__).resolve().parents[1]
SRC = ROOT / "gpurun_out" / "prof2"
DST = ROOT / "profiles"


def peak() -> float:
    try:
        return float(json.loads((ROOT / "MEASURED_PEAKS.json").read_text())["hbm_gbs"])
    except Exception:
        return 6551.0


def last_json(path: Path) -> dict:
    return json.loads([ln for ln in path.read_text().splitlines() if ln.strip().startswith("{")][-1])


def ncu_rows(rep: Path) -> list[dict]:
    out = subprocess.run(["ncu", "-i", str(rep), "--page", "raw", "--csv", "--print-units", "base"],
                         capture_output=True, text=True).stdout
    rows = list(csv.reader(io.StringIO(out)))
    h = rows[0]
    return [{h[i]: r[i] for i in range(len(h))} for r in rows[2:]]


def num(d: dict, k: str) -> float:
    try:
        return float(d.get(k, "nan").replace(",", ""))
    except ValueError:
        return float("nan")


def kernel_line(d: dict) -> str:
    t_us = num(d, "gpu__time_duration.sum") / 1e3   # base units: ns, bytes
    rd = num(d, "dram__bytes_read.sum")
    wr = num(d, "dram__bytes_write.sum")
    gbs = (rd + wr) / (t_us * 1e-6) / 1e9 if t_us > 0 else float("nan")
    inst = num(d, "smsp__inst_executed.sum")
    shw = num(d, "l1tex__data_pipe_lsu_wavefronts_mem_shared.sum")
    return (f"{t_us:10.1f} {rd / 1e6:10.1f} {wr / 1e6:9.1f} {gbs:8.0f} {gbs / peak():6.1%} "
            f"{num(d, 'smsp__issue_active.avg.pct_of_peak_sustained_active'):6.1f} "
            f"{num(d, 'l1tex__data_pipe_lsu_wavefronts_mem_shared.sum.pct_of_peak_sustained_elapsed'):6.1f} "
            f"{inst / 1e6:9.1f} {shw / 1e6:9.1f}  {d.get('Grid Size', ''):>12s}  {d.get('Kernel Name', '')[:100]}")


def kernels(tag: str) -> None:
    lines = [f"# ncu --set full --clock-control none captures (tools/profile_round2.sh), B200; peak = "
             f"{peak():.0f} GB/s (MEASURED_PEAKS.json hbm_gbs)",
             "# GB/s = (dram__bytes_read + dram__bytes_write) / gpu__time_duration -- one cold-cache, serialised launch",
             "# issue% = smsp__issue_active (of active); shm% = shared-memory LSU wavefronts (of peak, elapsed);",
             "# inst M = warp instructions; shwf M = shared wavefronts",
             "    dur_us    read_MB  write_MB     GB/s  %peak issue%   shm%    inst_M    shwf_M          grid  kernel"]
    for name in ("fused_c2_step", "fused_c3_u16", "secondary"):
        rep = SRC / f"{name}.ncu-rep"
        if not rep.exists():
            lines.append(f"# {name}: missing")
            continue
        lines.append(f"# --- {name}")
        if name == "secondary":
            lines.append("# launch order (tools/prof_secondary.py; torch's own fill/scan kernels in between): downscale 1024^3->512^3, "
                         "c5's 768^2x1024->512^3, encode 512, decode 512, PNG filter, deflate (+ compact), circle span + apply, "
                         "hist u8 (volume), hist u8 (top slab) + lut_build, lut_apply u8, hist u16, hist u16 (top slab) + lut_build, "
                         "lut_apply u16, render fp64 SURFACE (2 views), image_hist, render fp64 ADDITIVE (2 views), "
                         "blend_rows + render_rows<MIP> (8 views), blend_rows + render_rows<ALPHA> (8 views)")
        for d in ncu_rows(rep):
            lines.append(kernel_line(d))
        if name == "fused_c2_step":
            d = ncu_rows(rep)[0]
            per = num(d, "dram__bytes_read.sum") + num(d, "dram__bytes_write.sum")
            (DST / "traffic_fused_c2.json").write_text(json.dumps(
                {"dram_bytes_per_launch": per, "source": f"profiles/{tag}_kernels_ncu.txt (fused_c2_step)"}) + "\n")
    (DST / f"{tag}_kernels_ncu.txt").write_text("\n".join(lines) + "\n")


def launches(tag: str) -> None:
    rows = list(csv.reader(io.StringIO("\n".join(ln for ln in (SRC / "launches.csv").read_text().splitlines()
                                                  if ln.startswith('"')))))
    h = rows[0]
    ik, iv, im = h.index("Kernel Name"), h.index("Metric Value"), h.index("Metric Name")
    tot = collections.defaultdict(float)
    cnt = collections.Counter()
    for r in rows[1:]:
        if r[im] != "gpu__time_duration.sum":
            continue
        key = (r[ik], r[h.index("Grid Size")])
        tot[key] += float(r[iv].replace(",", ""))
        cnt[key] += 1
    allt = sum(tot.values())
    lines = ["# ncu --metrics gpu__time_duration.sum --clock-control none -c 400 python bench.py --steps 20 --warmup 3 "
             "--no-mip --no-cpu-baseline --no-configs --no-e2e --no-sustained",
             "# (cold-cache, serialised per-launch times; the SHARE of the step is what compares with the bench).",
             "# The timed c2 step is ONE preview_kernel launch on grid (148,1,1) (artifact-LUT phase + fused pass);",
             "# synth_kernel generates the volume once.",
             "launches   total_us   mean_us  share  grid          kernel"]
    for key, t in sorted(tot.items(), key=lambda kv: -kv[1]):
        lines.append(f"{cnt[key]:8d} {t * 1e-3:10.1f} {t * 1e-3 / cnt[key]:9.2f}  {t / allt:.3f}  "
                     f"{key[1]:12s}  {key[0][:110]}")
    (DST / f"{tag}_bench_launches.txt").write_text("\n".join(lines) + "\n")


def main() -> None:
    ap = argparse.ArgumentParser()
    ap.add_argument("--tag", default="r02")
    a = ap.parse_args()
    DST.mkdir(exist_ok=True)
    for src, dst in (("bench.jsonl", "bench.jsonl"), ("bench_reference.jsonl", "bench_reference.jsonl")):
        p = SRC / src
        if p.exists():
            (DST / f"{a.tag}_{dst}").write_text(json.dumps(last_json(p)) + "\n")
    if (SRC / "launches.csv").exists():
        launches(a.tag)
    kernels(a.tag)
    print("wrote", sorted(str(p.name) for p in DST.glob(f"{a.tag}_*")))


if __name__ == "__main__":
    main()
