"""Layer-by-layer mode: device time vs host issue time per step, with and
without the producer copies, stagger cadence (no recall bursts)."""
import sys, time
sys.path[:0] = ["."]
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

def one(copies):
    step[0] += 1
    s = step[0]
    j = s % len(wl.q_path_t)
    for i in range(L):
        if copies:
            qt_live[i].copy_(wl.q_path_t[j][i])
            if i + 1 < L:
                qp_live[i + 1].copy_(wl.q_path_p[j][i + 1])
            qt, qp = qt_live, qp_live
        else:
            qt, qp = wl.q_path_t[j], wl.q_path_p[j]
        eng.decode_layer(s, i, qt[i], qp[i + 1] if i + 1 < L else None, wl.cpu_o[i], wl.cpu_ml[i],
                         wl.k_new[i], wl.v_new[i], wl.out_o[i], wl.out_ml[i])

for copies in (True, False):
    for _ in range(5): one(copies)
    eng.sync(); torch.cuda.synchronize()
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    n = 32
    t0 = time.perf_counter(); a.record()
    for _ in range(n): one(copies)
    t1 = time.perf_counter(); b.record(); torch.cuda.synchronize()
    print(f"copies={copies}: device {a.elapsed_time(b)/n:.3f} ms/step, host issue {1000*(t1-t0)/n:.3f} ms/step")
# fused for comparison
for _ in range(5):
    step[0] += 1; wl.step(step[0])
eng.sync(); torch.cuda.synchronize()
a.record(); t0 = time.perf_counter()
for _ in range(32):
    step[0] += 1; wl.step(step[0])
t1 = time.perf_counter(); b.record(); torch.cuda.synchronize()
print(f"fused: device {a.elapsed_time(b)/32:.3f} ms/step, host issue {1000*(t1-t0)/32:.3f} ms/step")
