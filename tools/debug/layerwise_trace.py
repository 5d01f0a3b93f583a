"""Layer-by-layer mode under torch.profiler (CUPTI): every kernel's device
start / end, to see what overlaps with what inside a layer."""
import json, os, sys
sys.path[:0] = ["."]
import numpy as np
import torch
import bench
from torch.profiler import profile, ProfilerActivity

cfg = dict(bench.CONFIGS["qwen3-32b-32k"])
cfg.update(q_dtype=torch.bfloat16, cpu_dtype=torch.bfloat16, drift=0.15, recall_policy="stagger")
dev = torch.device("cuda")
wl = bench.TierWorkload(cfg, dev, 1234, 400, range(32))
eng = wl.make_engine()
L = wl.L
qt_live = torch.empty_like(wl.q_path_t[0]); qp_live = torch.empty_like(wl.q_path_p[0])
step = [0]

def one():
    step[0] += 1
    s = step[0]
    j = s % len(wl.q_path_t)
    for i in range(L):
        qt_live[i].copy_(wl.q_path_t[j][i])
        if i + 1 < L:
            qp_live[i + 1].copy_(wl.q_path_p[j][i + 1])
        eng.decode_layer(s, i, qt_live[i], qp_live[i + 1] if i + 1 < L else None, wl.cpu_o[i], wl.cpu_ml[i],
                         wl.k_new[i], wl.v_new[i], wl.out_o[i], wl.out_ml[i])

for _ in range(6): one()
eng.sync(); torch.cuda.synchronize()
with profile(activities=[ProfilerActivity.CUDA]) as prof:
    for _ in range(2): one()
    eng.sync(); torch.cuda.synchronize()
out = sys.argv[1] if len(sys.argv) > 1 else "gpurun_out/lw_trace.json"
prof.export_chrome_trace(out)
ev = json.load(open(out))["traceEvents"]
k = [e for e in ev if e.get("cat") == "kernel"]
k.sort(key=lambda e: e["ts"])
print(len(k), "kernels")
t0 = k[0]["ts"]
for e in k[:160]:
    print(f'{e["ts"]-t0:10.1f} {e["dur"]:8.1f} s{e["args"].get("stream")} {e["name"][:70]}')
# per-name totals
from collections import defaultdict
agg = defaultdict(lambda: [0, 0.0])
for e in k:
    n = e["name"][:60]; agg[n][0] += 1; agg[n][1] += e["dur"]
for n, (c, d) in sorted(agg.items(), key=lambda x: -x[1][1]):
    print(f"{c:6d} {d/c:9.1f} us avg  {d/1e3:8.2f} ms  {n}")
span = (k[-1]["ts"] + k[-1]["dur"] - t0) / 2
print(f"span per step {span/1e3:.3f} ms")
