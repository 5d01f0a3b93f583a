"""The host-buffer path (scout_engine_decode_step_kv_host) under torch.profiler
(CUPTI): every kernel and copy's device start / end over 3 steps, to see what
separates e2e from the device-resident step."""
import json, sys
sys.path[:0] = ["."]
import torch
import bench
from torch.profiler import profile, ProfilerActivity

cfg = dict(bench.CONFIGS["qwen3-32b-32k"])
cfg.update(q_dtype=torch.bfloat16, cpu_dtype=torch.bfloat16, drift=0.15, recall_policy="reference")
dev = torch.device("cuda")
W = bench.TierWorkload.auto_warm_slots(cfg, 32, 400, dev)
wl = bench.TierWorkload(cfg, dev, 1234, 400, range(32), warm_slots=W, host_units=32 * cfg["hkv"])
eng = wl.make_engine()
n, h_qt, h_qp, h_kv = bench._pinned_inputs(wl, True)
h_co = wl.cpu_o.cpu().pin_memory(); h_cm = wl.cpu_ml.cpu().pin_memory()
h_out = torch.empty(wl.out_o.shape, dtype=torch.float32).pin_memory()
h_oml = torch.empty(wl.out_ml.shape, dtype=torch.float32).pin_memory()
h_ids = torch.empty(wl.L, wl.U, wl.k, dtype=torch.int32).pin_memory()
h_n = torch.empty(wl.L, wl.U, dtype=torch.int32).pin_memory()
s = [0]
def one():
    s[0] += 1
    j = s[0] % n
    eng.decode_step_kv_host(s[0], h_qt[j], h_qp[j], h_co, h_cm, *h_kv, h_out, h_oml, h_ids, h_n)
for _ in range(8): one()
eng.sync(); torch.cuda.synchronize()
with profile(activities=[ProfilerActivity.CUDA]) as prof:
    for _ in range(3): one()
    eng.sync(); torch.cuda.synchronize()
out = sys.argv[1] if len(sys.argv) > 1 else "gpurun_out/e2e_trace.json"
prof.export_chrome_trace(out)
ev = [e for e in json.load(open(out))["traceEvents"] if e.get("cat") in ("kernel", "gpu_memcpy", "gpu_memset")]
ev.sort(key=lambda e: e["ts"])
t0 = ev[0]["ts"]
big = [e for e in ev if e["dur"] > 20 or e.get("cat") == "kernel"]
for e in big[:400]:
    print(f'{e["ts"]-t0:10.1f} {e["dur"]:8.1f} s{e["args"].get("stream")} {e.get("cat")[:6]} {e["name"][:60]}')
k2 = [e for e in ev if "sparse_decode" in e["name"]]
for a, b in zip(k2, k2[1:]):
    print(f"K2 start to next K2 start: {b['ts'] - a['ts']:.1f} us (K2 {a['dur']:.1f})")
