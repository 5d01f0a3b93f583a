"""The fused step around a recall (bench defaults, reference cadence: every
layer recalls at steps 16, 32, ...) under torch.profiler: every kernel and
stream operation of the recall step and the step after it, to see what the
recall costs beyond the extra resident blocks K2 then streams."""
import json, sys
from collections import defaultdict
sys.path[:0] = ["."]
import torch
import bench
from torch.profiler import profile, ProfilerActivity

cfg = dict(bench.CONFIGS["qwen3-32b-32k"])
cfg.update(q_dtype=torch.bfloat16, cpu_dtype=torch.bfloat16, drift=0.15, recall_policy="reference", recall_mode=1)
dev = torch.device("cuda")
W = bench.TierWorkload.auto_warm_slots(cfg, 32, 400, dev)
wl = bench.TierWorkload(cfg, dev, 1234, 400, range(32), warm_slots=W, host_units=32 * cfg["hkv"])
eng = wl.make_engine()
n = len(wl.q_path_t)


def one(s):
    j = s % n
    eng.decode_step_kv(s, wl.q_path_t[j], wl.q_path_p[j], wl.cpu_o, wl.cpu_ml, wl.k_new, wl.v_new, wl.out_o,
                       wl.out_ml)


for s in range(1, 31):
    one(s)
eng.sync(); torch.cuda.synchronize()
with profile(activities=[ProfilerActivity.CUDA]) as prof:
    for s in range(31, 35):  # 32 recalls, 33 runs after it
        one(s)
    eng.sync(); torch.cuda.synchronize()
out = sys.argv[1] if len(sys.argv) > 1 else "gpurun_out/recall_step_trace.json"
prof.export_chrome_trace(out)
ev = [e for e in json.load(open(out))["traceEvents"] if e.get("cat") in ("kernel", "gpu_memcpy", "gpu_memset")]
ev.sort(key=lambda e: e["ts"])
t0 = ev[0]["ts"]
k1 = [e for e in ev if "score_topk" in e["name"]]
starts = [e["ts"] for e in k1]
print(f"{len(ev)} device events; K1 starts (step boundaries):", [f"{(t - t0) / 1e3:.3f}" for t in starts])
for a, b in zip(starts, starts[1:] + [ev[-1]["ts"] + ev[-1]["dur"]]):
    agg = defaultdict(lambda: [0, 0.0])
    for e in ev:
        if a <= e["ts"] < b:
            agg[e["name"][:70]][0] += 1
            agg[e["name"][:70]][1] += e["dur"]
    print(f"--- step window {(b - a) / 1e3:.3f} ms")
    for name, (c, d) in sorted(agg.items(), key=lambda x: -x[1][1]):
        print(f"   {c:5d} x {d / max(c, 1):9.1f} us = {d / 1e3:7.3f} ms  {name}")
big = [e for e in ev if "sparse_decode" not in e["name"] and "score_topk" not in e["name"]]
print("--- non-K1/K2 events in order (first 120)")
for e in big[:120]:
    print(f'{(e["ts"] - t0):10.1f} {e["dur"]:8.1f} s{e["args"].get("stream")} {e["name"][:60]}')
