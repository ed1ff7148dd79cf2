"""Summarise a tools/profile_round.sh pass (gpurun_out/prof/) into profiles/.

usage: python tools/summarise_profiles.py [--tag r01]

Writes profiles/<tag>_bench.jsonl (the bench line), <tag>_bench_reference.jsonl,
<tag>_bench_launches.txt (per-kernel share of the ncu launch list),
<tag>_fused_c2_step_ncu.txt (key metrics + warp-state shares of the step kernel)
and traffic_fused_c2.json (DRAM bytes per launch, read by bench.py's roofline).
Needs ncu on PATH for the .ncu-rep.
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
SRC = ROOT / "gpurun_out" / "prof"
DST = ROOT / "profiles"


def last_json(path: Path) -> dict:
    return json.loads([ln for ln in path.read_text().splitlines() if ln.strip().startswith("{")][-1])


def launches(tag: str) -> None:
    rows = list(csv.reader(io.StringIO("\n".join(ln for ln in (SRC / "launches.csv").read_text().splitlines()
                                                  if ln.startswith('"')))))
    h = rows[0]
    ik, iv, im = h.index("Kernel Name"), h.index("Metric Value"), h.index("Metric Name")
    tot = collections.defaultdict(float)
    cnt = collections.Counter()
    grid = {}
    for r in rows[1:]:
        if r[im] != "gpu__time_duration.sum":
            continue
        v = float(r[iv].replace(",", ""))
        name = r[ik]
        if "preview_kernel" in name:  # the whole-volume step vs the e2e session's 64-slice chunks
            name = ("[c2 step, whole volume] " if v > 150e3 else "[e2e 64-slice chunk] ") + name
        key = (name, r[h.index("Grid Size")])
        tot[key] += v
        cnt[key] += 1
    unit = "ns"
    allt = sum(tot.values())
    lines = ["# ncu --metrics gpu__time_duration.sum --clock-control none -c 400 python bench.py --steps 20 --warmup 3 "
             "--no-mip --no-cpu-baseline --no-configs",
             "# (cold-cache, serialised per-launch times; the SHARE of the step is what compares with the bench).",
             "# The timed c2 step is ONE preview_kernel launch on grid (148,1,1) (artifact-LUT phase + fused pass); the",
             "# smaller-grid / 64-slice launches are the e2e PreviewSession chunks; synth_kernel generates the volume once.",
             "launches   total_us   mean_us  share  grid          kernel"]
    for key, t in sorted(tot.items(), key=lambda kv: -kv[1]):
        scale = 1e-3 if unit == "ns" else 1.0
        lines.append(f"{cnt[key]:8d} {t * scale:10.1f} {t * scale / cnt[key]:9.2f}  {t / allt:.3f}  "
                     f"{key[1]:12s}  {key[0][:110]}")
    (DST / f"{tag}_bench_launches.txt").write_text("\n".join(lines) + "\n")


def ncu_raw(rep: Path) -> dict:
    out = subprocess.run(["ncu", "-i", str(rep), "--page", "raw", "--csv"], capture_output=True, text=True).stdout
    rows = list(csv.reader(io.StringIO(out)))
    h, u, v = rows[0], rows[1], rows[2]
    return {h[i]: (v[i], u[i]) for i in range(len(h))}


def step_ncu(tag: str) -> None:
    d = ncu_raw(SRC / "fused_c2_step.ncu-rep")

    def f(k):
        return float(d[k][0].replace(",", ""))

    keys = ["gpu__time_duration.sum", "dram__bytes_read.sum", "dram__bytes_write.sum",
            "dram__throughput.avg.pct_of_peak_sustained_elapsed", "smsp__inst_executed.sum",
            "smsp__issue_active.avg.pct_of_peak_sustained_active", "smsp__inst_executed_op_shared_atom.sum",
            "l1tex__data_pipe_lsu_wavefronts_mem_shared.sum",
            "l1tex__data_pipe_lsu_wavefronts_mem_shared.sum.pct_of_peak_sustained_elapsed",
            "l1tex__data_pipe_lsu_wavefronts_mem_shared_op_atom.sum", "sm__cycles_elapsed.avg"]
    lines = ["# ncu --set full --clock-control none -k regex:preview_kernel -s 5 -c 1 python bench.py --steps 3 "
             "--warmup 3 --no-mip --no-e2e --no-cpu-baseline --no-configs",
             "# the c2 step kernel (one cooperative launch: artifact-LUT phase + fused hist/filter/pyramid/atlas pass)"]
    for k in keys:
        if k in d:
            lines.append(f"  {k:75s} {d[k][0]:>16s} {d[k][1]}")
    st = {k.replace("smsp__pcsamp_warps_issue_stalled_", ""): int(d[k][0].replace(",", "")) for k in d
          if k.startswith("smsp__pcsamp_warps_issue_stalled") and not k.endswith("not_issued")
          and d[k][0] not in ("", "0")}
    tot = sum(st.values())
    lines.append("# warp-state samples: " + ", ".join(f"{k} {100 * v / tot:.1f}%"
                                                     for k, v in sorted(st.items(), key=lambda kv: -kv[1])[:10]))
    vox = 1024 ** 3
    lines.append(f"# instructions per voxel {32 * f('smsp__inst_executed.sum') / vox:.2f}; shared atomics per 32 voxels "
                 f"{32 * f('smsp__inst_executed_op_shared_atom.sum') / vox:.3f}; atom wavefronts per ATOMS "
                 f"{f('l1tex__data_pipe_lsu_wavefronts_mem_shared_op_atom.sum') / f('smsp__inst_executed_op_shared_atom.sum'):.3f}")
    (DST / f"{tag}_fused_c2_step_ncu.txt").write_text("\n".join(lines) + "\n")
    rd, wr = f("dram__bytes_read.sum"), f("dram__bytes_write.sum")
    scale = {"Gbyte": 1e9, "Mbyte": 1e6, "Kbyte": 1e3, "byte": 1.0}
    rd *= scale[d["dram__bytes_read.sum"][1]]
    wr *= scale[d["dram__bytes_write.sum"][1]]
    t = f("gpu__time_duration.sum") * (1e-3 if d["gpu__time_duration.sum"][1] == "ns" else 1.0)
    traffic = {
        "kernel": "preview_kernel<uint8_t,3,1024,2,1024,WANT0=false,POW2=true> cooperative step (artifact-LUT phase + "
                  "fused hist+LUT+3-level pyramid+atlases), c2 1024^3 u8",
        "source": "tools/profile_round.sh: ncu --set full --clock-control none -k regex:preview_kernel -s 5 -c 1 "
                  "python bench.py --steps 3 --warmup 3 --no-mip --no-e2e --no-cpu-baseline --no-configs",
        "gpu_time_us": t,
        "dram_bytes_read": rd,
        "dram_bytes_write": wr,
        "dram_bytes_per_launch": rd + wr,
        "alg_bytes_per_launch": 1073741824 + 153092096,
        "shared_atomics_warp_instr": f("smsp__inst_executed_op_shared_atom.sum"),
        "issue_active_pct": f("smsp__issue_active.avg.pct_of_peak_sustained_active"),
        "note": "read = the volume + the 3 top slices of the LUT phase (3 MiB); DRAM write < atlas bytes because part "
                "of the 153 MB of atlas writes is still dirty in L2 when the kernel ends",
    }
    (DST / "traffic_fused_c2.json").write_text(json.dumps(traffic, indent=1) + "\n")


def main() -> None:
    ap = argparse.ArgumentParser()
    ap.add_argument("--tag", default="r01")
    a = ap.parse_args()
    (DST / f"{a.tag}_bench.jsonl").write_text(json.dumps(last_json(SRC / "bench.jsonl")) + "\n")
    (DST / f"{a.tag}_bench_reference.jsonl").write_text(json.dumps(last_json(SRC / "bench_reference.jsonl")) + "\n")
    launches(a.tag)
    step_ncu(a.tag)


if __name__ == "__main__":
    main()
