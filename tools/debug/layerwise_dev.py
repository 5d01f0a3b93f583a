"""Layer-by-layer mode, device side: per layer, the query copies, the wait for
K1 + the K2 launch (caller stream), and K2's own kernel time (engine timing
events), stagger cadence."""
import sys
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
n = 16
ev = [[torch.cuda.Event(enable_timing=True) for _ in range(3)] for _ in range(L * n)]

def one(rec, t):
    step[0] += 1
    s = step[0]
    j = s % len(wl.q_path_t)
    for i in range(L):
        e = ev[t * L + i] if rec else None
        if e: e[0].record()
        qt_live[i].copy_(wl.q_path_t[j][i])
        if i + 1 < L:
            qp_live[i + 1].copy_(wl.q_path_p[j][i + 1])
        if e: e[1].record()
        eng.decode_layer(s, i, qt_live[i], qp_live[i + 1] if i + 1 < L else None, wl.cpu_o[i], wl.cpu_ml[i],
                         wl.k_new[i], wl.v_new[i], wl.out_o[i], wl.out_ml[i])
        if e: e[2].record()

for _ in range(5): one(False, 0)
eng.sync(); torch.cuda.synchronize()
eng.stats()
eng.set_timing(True)
for t in range(n): one(True, t)
eng.sync(); torch.cuda.synchronize()
ms, cnt, launches = eng.stats()
cp = np.array([[ev[t*L+i][0].elapsed_time(ev[t*L+i][1]) for i in range(L)] for t in range(n)]) * 1e3
k2 = np.array([[ev[t*L+i][1].elapsed_time(ev[t*L+i][2]) for i in range(L)] for t in range(n)]) * 1e3
gap = np.array([[ev[t*L+i][2].elapsed_time(ev[t*L+i+1][0]) for i in range(L - 1)] for t in range(n)]) * 1e3
tot = [ev[t*L][0].elapsed_time(ev[t*L+L-1][2]) for t in range(n)]
print(f"step {np.mean(tot):.3f} ms; K2 kernel avg {1e3*ms/max(cnt,1):.1f} us over {cnt} launches; launches {launches}")
print(f"per layer: copies {cp.mean():.1f} us, K1-wait+K2 {k2.mean():.1f} us, gap to next layer {gap.mean():.1f} us")
print("K1-wait+K2 by layer:", " ".join(f"{x:.0f}" for x in k2.mean(0)))
print("copies by layer:", " ".join(f"{x:.0f}" for x in cp.mean(0)))
eng.close()
