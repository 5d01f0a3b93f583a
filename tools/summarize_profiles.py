"""Summarise a round's ncu captures into profiles/ (run in the build container).

  python tools/summarize_profiles.py r01
reads gpurun_out/{launches_<r>.csv, prof_k2_<r>.ncu-rep, prof_k1_<r>.ncu-rep, bench_<r>.json}
writes profiles/<r>_launches.csv, profiles/<r>_summary.md, profiles/k2_traffic.json
"""
import collections
import csv
import io
import json
import shutil
import subprocess
import sys
from pathlib import Path

ROOT = Path(__file__).resolve().parents[1]
R = sys.argv[1]
G = ROOT / "gpurun_out"
P = ROOT / "profiles"
P.mkdir(exist_ok=True)

METRICS = ["gpu__time_duration.sum", "dram__bytes_read.sum", "dram__bytes_write.sum",
           "gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed", "sm__throughput.avg.pct_of_peak_sustained_elapsed",
           "sm__pipe_tensor_cycles_active.avg.pct_of_peak_sustained_active", "launch__registers_per_thread",
           "sm__warps_active.avg.pct_of_peak_sustained_active", "launch__grid_size", "launch__block_size",
           "smsp__inst_executed.sum"]


def raw(rep):
    out = subprocess.run(["ncu", "-i", str(rep), "--page", "raw", "--csv"], capture_output=True, text=True).stdout
    rows = list(csv.reader(io.StringIO(out)))
    hdr, units, vals = rows[0], rows[1], rows[2]
    return {h: (v, u) for h, u, v in zip(hdr, units, vals)}


lines = [f"# Round {R[1:]} profile summary", ""]
bench = G / f"bench_{R}.json"
if bench.exists():
    shutil.copy(bench, P / f"{R}_bench.json")
    b = json.loads(bench.read_text().strip().splitlines()[-1])
    lines += ["## bench.py (1x B200)", "", "```", json.dumps({k: b.get(k) for k in
              ("value", "unit", "ms_per_step", "step_gbs", "roofline", "e2e", "cpu_baseline", "clocks",
               "gpu_launches")}, indent=1), "```", ""]
lc = G / f"launches_{R}.csv"
if lc.exists():
    shutil.copy(lc, P / f"{R}_launches.csv")
    rows = list(csv.reader(open(lc)))
    hdr = None
    agg = collections.defaultdict(list)
    for r in rows:
        if r and r[0] == "ID":
            hdr = r
            continue
        if hdr and len(r) == len(hdr):
            d = dict(zip(hdr, r))
            agg[d["Kernel Name"].split("(")[0]].append(float(d["Metric Value"]))
    tot = sum(sum(v) for v in agg.values())
    lines += ["## Launch list (ncu gpu__time_duration, --clock-control none; serialised, cold)", "",
              "| kernel | launches | mean us | share |", "|---|---|---|---|"]
    for k, v in sorted(agg.items(), key=lambda kv: -sum(kv[1])):
        lines.append(f"| `{k}` | {len(v)} | {sum(v) / len(v) / 1000:.1f} | {sum(v) / tot:.1%} |")
    lines.append("")
for name in ("k2", "k1", "k6"):
    rep = G / f"prof_{name}_{R}.ncu-rep"
    if not rep.exists():
        continue
    m = raw(rep)
    lines += [f"## {name.upper()} `ncu --set full` (one launch)", "", "| metric | value |", "|---|---|"]
    for key in METRICS:
        if key in m:
            lines.append(f"| {key} | {m[key][0]} {m[key][1]} |")
    if name == "k2":
        rd = float(m["dram__bytes_read.sum"][0].replace(",", ""))
        wr = float(m["dram__bytes_write.sum"][0].replace(",", ""))
        scale = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9}
        rd *= scale.get(m["dram__bytes_read.sum"][1], 1)
        wr *= scale.get(m["dram__bytes_write.sum"][1], 1)
        (P / "k2_traffic.json").write_text(json.dumps({"bytes_per_launch": rd + wr, "read": rd, "write": wr,
                                                       "source": f"profiles/{R}_summary.md (ncu --set full)"}))
    lines.append("")
(P / f"{R}_summary.md").write_text("\n".join(lines) + "\n")
print("\n".join(lines))
