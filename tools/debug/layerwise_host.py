"""Layer-by-layer mode: where the host time of a step goes (per-call host
durations of the query copies and of scout_engine_decode_layer, by layer)."""
import sys, time
sys.path[:0] = ["."]
import numpy as np
import torch
import bench

cfg = dict(bench.CONFIGS["qwen3-32b-32k"])
cfg.update(q_dtype=torch.bfloat16, cpu_dtype=torch.bfloat16, drift=0.15, recall_policy="stagger")
dev = torch.device("cuda")
wl = bench.TierWorkload(cfg, dev, 1234, 400, range(32))
eng = wl.make_engine()
L = wl.L
qt_live = torch.empty_like(wl.q_path_t[0]); qp_live = torch.empty_like(wl.q_path_p[0])
step = [0]
tc = np.zeros(L); tl = np.zeros(L)

def one(rec):
    step[0] += 1
    s = step[0]
    j = s % len(wl.q_path_t)
    for i in range(L):
        t0 = time.perf_counter()
        qt_live[i].copy_(wl.q_path_t[j][i])
        if i + 1 < L:
            qp_live[i + 1].copy_(wl.q_path_p[j][i + 1])
        t1 = time.perf_counter()
        eng.decode_layer(s, i, qt_live[i], qp_live[i + 1] if i + 1 < L else None, wl.cpu_o[i], wl.cpu_ml[i],
                         wl.k_new[i], wl.v_new[i], wl.out_o[i], wl.out_ml[i])
        t2 = time.perf_counter()
        if rec:
            tc[i] += t1 - t0; tl[i] += t2 - t1

for _ in range(5): one(False)
eng.sync(); torch.cuda.synchronize()
n = 32
for _ in range(n): one(True)
torch.cuda.synchronize()
tc *= 1e6 / n; tl *= 1e6 / n
print(f"per step: copies {tc.sum()/1e3:.3f} ms, decode_layer {tl.sum()/1e3:.3f} ms")
print("decode_layer us by layer:", " ".join(f"{x:.0f}" for x in tl))
print("copies us by layer:", " ".join(f"{x:.0f}" for x in tc))
# the wrapper's own cost: _check + pointer extraction, no C call
t0 = time.perf_counter()
for _ in range(1000):
    eng._check(qt_live[1], qp_live[2], wl.cpu_o[1], wl.cpu_ml[1])
print(f"_check: {(time.perf_counter()-t0)*1e3:.1f} us per call")
eng.close()
