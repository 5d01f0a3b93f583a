"""The CPU co-attention worker on the bench workload's real CPU share: after
40 steps of the config-3 tier workload, every layer's CPU-side ids (K1's
split) become one worker call per 4-layer chunk, as the engine makes them.
Times the chunks at several thread counts, against the same number of blocks
spread uniformly (5 per unit), to separate per-unit overhead from contention."""
import sys, time, os
sys.path[:0] = [".", "tests", "oracle"]
import numpy as np
import torch
import bench
from paper_2603_27138_b200 import ops

cfg = dict(bench.CONFIGS["qwen3-32b-32k"])
cfg.update(q_dtype=torch.bfloat16, cpu_dtype=torch.bfloat16, drift=0.15, recall_policy="reference")
dev = torch.device("cuda")
wl = bench.TierWorkload(cfg, dev, 1234, 200, range(32), warm_slots=0)
wl.make_engine()
for s in range(1, 41):
    wl.step(s)
wl.engine.sync(); torch.cuda.synchronize()
k1 = {n: t.cpu() for n, t in wl.engine.k1_outputs().items()}
L, U, G, k, nbs = wl.L, wl.U, wl.G, wl.k, int(wl.layer_states[0].digests.shape[-1])
n_cpu = k1["n_cpu"]  # [L][U]
ids = k1["cpu_ids"]  # [L][U][k]
print("CPU blocks per step", int(n_cpu.sum()), "units with any", int((n_cpu > 0).sum()), "of", L * U,
      "max per unit", int(n_cpu.max()))
hist = torch.bincount(n_cpu.flatten().long())
print("blocks-per-unit histogram", hist.tolist()[:20])
l_ = torch.arange(L).view(L, 1, 1).long(); u_ = torch.arange(U).view(1, U, 1).long()
hidx = ((l_ * U + u_) * nbs + ids.long()) % wl.host_blocks  # [L][U][k]
q = wl.q_path_p[40 % len(wl.q_path_p)].float().cpu()  # [L][U*G][D]
CH = 4
for T in (16, 15, 14, 12, 8):
    if T > os.cpu_count():
        continue
    tot = 0.0
    for rep in range(2):
        t0 = time.perf_counter()
        for lo in range(0, L, CH):
            n = min(CH, L - lo)
            ops.cpu_partial_attention(wl.host_tier, torch.bfloat16, hidx[lo:lo + n].reshape(n * U, k),
                                      n_cpu[lo:lo + n].reshape(n * U), q[lo:lo + n].reshape(n * U * G, 128), G,
                                      threads=T)
        tot = time.perf_counter() - t0
    nb = int(n_cpu.sum())
    print(f"threads {T:2d}: real share {tot * 1e3:7.2f} ms per step ({nb / tot / 1e6:.2f} M blocks/s)")
    # the same blocks, 5 per unit on fewer units
    nu = nb // 5
    idx5 = torch.randint(0, wl.host_blocks, (nu, k), dtype=torch.int64)
    n5 = torch.full((nu,), 5, dtype=torch.int32)
    q5 = torch.randn(nu * G, 128)
    ops.cpu_partial_attention(wl.host_tier, torch.bfloat16, idx5, n5, q5, G, threads=T)
    t0 = time.perf_counter()
    for lo in range(0, nu, 1024):
        m = min(1024, nu - lo)
        ops.cpu_partial_attention(wl.host_tier, torch.bfloat16, idx5[lo:lo + m], n5[lo:lo + m], q5[lo * G:(lo + m) * G], G,
                                  threads=T)
    t5 = time.perf_counter() - t0
    print(f"threads {T:2d}: uniform 5/unit {t5 * 1e3:7.2f} ms ({nb / t5 / 1e6:.2f} M blocks/s)")
