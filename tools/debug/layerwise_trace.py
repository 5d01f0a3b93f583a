"""Layer-by-layer mode under torch.profiler (CUPTI): every kernel's device
start / end, to see what overlaps with what inside a layer."""
import json, os, sys
sys.path[:0] = ["."]
import numpy as np
import torch
import bench
from torch.profiler import profile, ProfilerActivity

cfg = dict(bench.CONFIGS["qwen3-32b-32k"])
# the bench's defaults: bf16 queries and CPU partials, the reference cadence, SM recall gather,
# the victim cache sized automatically
cfg.update(q_dtype=torch.bfloat16, cpu_dtype=torch.bfloat16, drift=0.15, recall_policy="reference", recall_mode=1)
dev = torch.device("cuda")
warm = bench.TierWorkload.auto_warm_slots(cfg, 32, 400, dev)
wl = bench.TierWorkload(cfg, dev, 1234, 400, range(32), warm_slots=warm, host_units=32 * cfg["hkv"])
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
import time
for _ in range(3):  # host enqueue time of one step (no sync inside) vs its device span
    torch.cuda.synchronize()
    t0h = time.perf_counter(); one(); t1h = time.perf_counter()
    torch.cuda.synchronize(); t2h = time.perf_counter()
    print(f"host enqueue {1e3 * (t1h - t0h):.3f} ms, enqueue+drain {1e3 * (t2h - t0h):.3f} ms")
with profile(activities=[ProfilerActivity.CUDA]) as prof:
    for _ in range(2): one()
    eng.sync(); torch.cuda.synchronize()
out = sys.argv[1] if len(sys.argv) > 1 else "gpurun_out/lw_trace.json"
prof.export_chrome_trace(out)
ev = json.load(open(out))["traceEvents"]
allk = [e for e in ev if e.get("cat") in ("kernel", "gpu_memcpy", "gpu_memset")]
allk.sort(key=lambda e: e["ts"])
k = [e for e in allk if e.get("cat") == "kernel"]
k.sort(key=lambda e: e["ts"])
ta = allk[0]["ts"]
print("--- one layer window with copies")
for e in allk[200:240]:
    print(f'{e["ts"]-ta:10.1f} {e["dur"]:8.1f} s{e["args"].get("stream")} {e.get("cat")[:6]} {e["name"][:60]}')
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
# per layer: K2 start-to-start, K2 duration, the K1 beside it, the gap K2(i) end -> K2(i+1) start
k2 = [e for e in k if "sparse_decode" in e["name"]]
k1 = [e for e in k if "score_topk" in e["name"]]
if len(k2) > 2:
    per, dur, gap = [], [], []
    for a, b in zip(k2, k2[1:]):
        per.append(b["ts"] - a["ts"]); dur.append(a["dur"]); gap.append(b["ts"] - a["ts"] - a["dur"])
    print(f"K2 per layer: start-to-start {np.median(per):.1f} us, duration {np.median(dur):.1f} us, "
          f"idle gap {np.median(gap):.1f} us (medians over {len(per)})")
    print(f"K1 per layer: duration {np.median([e['dur'] for e in k1]):.1f} us (median over {len(k1)})")
