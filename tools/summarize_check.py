"""Summarise one round check (tools/gpu/round_check.sh <tag>) from gpurun_out/
into profiles/<tag>_summary.md and copy the small artefacts beside it.

Reads the bench JSON lines, the ncu launch list (CSV) and the three
`ncu --set full` captures (with the local ncu, `--page raw --csv`).
Usage: python tools/summarize_check.py <tag>"""
import csv
import io
import json
import shutil
import subprocess
import sys
from collections import defaultdict
from pathlib import Path

ROOT = Path(__file__).resolve().parents[1]
OUT, PROF = ROOT / "gpurun_out", ROOT / "profiles"
METRICS = ["gpu__time_duration.sum", "dram__bytes_read.sum", "dram__bytes_write.sum",
           "gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed",
           "sm__throughput.avg.pct_of_peak_sustained_elapsed",
           "sm__pipe_tensor_cycles_active.avg.pct_of_peak_sustained_active", "launch__registers_per_thread",
           "sm__warps_active.avg.pct_of_peak_sustained_active", "launch__grid_size", "launch__block_size",
           "smsp__inst_executed.sum"]


def last_json(p):
    for line in reversed(p.read_text().strip().splitlines()):
        if line.startswith("{"):
            return json.loads(line)
    return None


def ncu_raw(rep):
    r = subprocess.run(["ncu", "-i", str(rep), "--page", "raw", "--csv"], capture_output=True, text=True)
    rows = list(csv.reader(io.StringIO(r.stdout)))
    if len(rows) < 3:
        return {}
    head, units, vals = rows[0], rows[1], rows[2]
    return {h: (v, u) for h, u, v in zip(head, units, vals)}


def launch_table(p):
    rows = [r for r in csv.reader(io.StringIO("\n".join(
        line for line in p.read_text().splitlines() if line.startswith('"'))))]
    if not rows:
        return []
    h = rows[0]
    ki, mi, vi = h.index("Kernel Name"), h.index("Metric Name"), h.index("Metric Value")
    agg = defaultdict(list)
    for r in rows[1:]:
        if r[mi] == "gpu__time_duration.sum":
            agg[r[ki]].append(float(r[vi].replace(",", "")))
    unit = rows[1][h.index("Metric Unit")] if len(rows) > 1 else "ns"
    scale = {"ns": 1e-3, "us": 1.0, "usecond": 1.0, "nsecond": 1e-3, "msecond": 1e3, "ms": 1e3}.get(unit, 1e-3)
    tot = sum(sum(v) for v in agg.values())
    return sorted(((k, len(v), sum(v) / len(v) * scale, sum(v) / tot) for k, v in agg.items()), key=lambda x: -x[3])


def main():
    tag = sys.argv[1]
    lines = [f"# Round check {tag}: summary", ""]
    b = last_json(OUT / f"bench_{tag}.json")
    ref = last_json(OUT / f"bench_ref_{tag}.json")
    lines += ["## bench.py (1x B200)", "", "```", json.dumps({k: b[k] for k in (
        "value", "unit", "ms_per_step", "roofline", "e2e", "cpu_baseline", "clocks", "gpu_launches") if k in b},
        indent=1), "```", ""]
    ext = {k: {kk: b[k].get(kk) for kk in ("value", "ms_per_step")} for k in (
        "value_layerwise", "value_layerwise_qpred", "victim_cache_off", "e2e_with_cpu_worker") if k in b}
    lines += ["Other lines of the same run: `" + json.dumps(ext) + "`", ""]
    if ref:
        lines += [f"Reference arm (`--impl reference`): {ref.get('value'):.3f} {ref.get('unit')}, "
                  f"{ref.get('ms_per_step'):.1f} ms per step (sampled, 16 cores)", ""]
    lines += ["## Config sweep", "", "| run | tokens/s | ms/step | e2e ms | roofline frac | SM MHz |",
              "|---|---|---|---|---|---|"]
    for p in sorted(OUT.glob(f"sweep_*_{tag}.json")):
        d = last_json(p)
        if not d:
            lines.append(f"| {p.stem} | (no line) | | | | |")
            continue
        e2e = (d.get("e2e") or {}).get("ms_per_step")
        lines.append(f"| {p.stem.replace('_' + tag, '')} ({d.get('config', {}).get('workload')}) | "
                     f"{d.get('value', 0):.0f} | {d.get('ms_per_step', 0):.3f} | "
                     f"{'' if e2e is None else f'{e2e:.3f}'} | {(d.get('roofline') or {}).get('frac', 0):.3f} | "
                     f"{(d.get('clocks') or {}).get('sm_mhz')} |")
    lines += ["", "## Launch list (ncu gpu__time_duration, --clock-control none; serialised, cold)", "",
              "| kernel | launches | mean us | share |", "|---|---|---|---|"]
    for k, n, mean, share in launch_table(OUT / f"launches_{tag}.csv"):
        lines.append(f"| `{k[:80]}` | {n} | {mean:.1f} | {100 * share:.1f}% |")
    k1_traffic = None
    for name, rep in (("K1", "k1"), ("K2", "k2"), ("K6", "k6")):
        m = ncu_raw(OUT / f"prof_{rep}_{tag}.ncu-rep")
        lines += ["", f"## {name} `ncu --set full` (one launch)", "", "| metric | value |", "|---|---|"]
        for key in METRICS:
            if key in m:
                lines.append(f"| {key} | {m[key][0]} {m[key][1]} |")
        if name in ("K1", "K2") and "dram__bytes_read.sum" in m:
            scale = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9}
            rd = float(m["dram__bytes_read.sum"][0]) * scale.get(m["dram__bytes_read.sum"][1], 1)
            wr = float(m["dram__bytes_write.sum"][0]) * scale.get(m["dram__bytes_write.sum"][1], 1)
            if name == "K1":
                k1_traffic = rd + wr
                continue
            (PROF / "k2_traffic.json").write_text(json.dumps({
                "bytes_per_launch": rd + wr, "read": rd, "write": wr, "k1_bytes_per_launch": k1_traffic,
                "source": f"profiles/{tag}_summary.md (ncu --set full)"}) + "\n")
    (PROF / f"{tag}_summary.md").write_text("\n".join(lines) + "\n")
    for src, dst in ((f"bench_{tag}.json", f"{tag}_bench.json"), (f"bench_ref_{tag}.json", f"{tag}_bench_ref.json"),
                     (f"launches_{tag}.csv", f"{tag}_launches.csv"), (f"pytest_gpu_{tag}.log", f"{tag}_pytest_gpu.log"),
                     (f"phases_{tag}.err", f"{tag}_phases.txt"), (f"smoke_{tag}.log", f"{tag}_smoke.log")):
        if (OUT / src).exists():
            shutil.copy(OUT / src, PROF / dst)
    for p in OUT.glob(f"sweep_*_{tag}.json"):
        shutil.copy(p, PROF / f"{tag}_{p.stem.replace('_' + tag, '')}.json")
    print((PROF / f"{tag}_summary.md").read_text())


if __name__ == "__main__":
    main()
