"""One layer of config 3 in isolation: K2 (256 units, G=8, 59 resident blocks
each, bf16 queries) and K1 (256 units, nb_stride 520, top-64, block table):
median CUDA-event time per launch, and the HBM rate."""
import sys
sys.path[:0] = [".", "tests", "oracle"]
import numpy as np
import torch
from paper_2603_27138_b200 import ops
from test_gpu_decode_scale import build

rng = np.random.default_rng(0)
U, G, D, NR = 256, 8, 128, 59
c = build(rng, [NR] * U)
q = c["q"].to(torch.bfloat16)
d = c["dev"]


def med(fn, n=50):
    ts = []
    for _ in range(5):
        fn()
    for _ in range(n):
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record(); fn(); b.record()
        b.synchronize()
        ts.append(a.elapsed_time(b) * 1e3)
    return float(np.median(ts)), float(np.min(ts))


k2_bytes = U * NR * 32768 + U * G * D * 2
for ctas in (0, 128):
    ws = ops.DecodeWorkspace(U, G, q.device, ctas)
    o = torch.empty(U * G, D, device="cuda"); ml = torch.empty(U * G, 2, device="cuda")
    m, lo = med(lambda: ops.sparse_decode(q, c["pool"], torch.bfloat16, d["res_slots"], d["res_ids"], d["n_res"],
                                          d["n_tokens"], G, o=o, ml=ml, workspace=ws, max_ctas=ctas))
    print(f"K2 one layer, ctas={ctas or 148}: median {m:.1f} us (min {lo:.1f}), {k2_bytes / m / 1e3:.0f} GB/s")

nbs = 520
dig = torch.randn(U, 2, D, nbs, device="cuda").to(torch.bfloat16)
dig[:, 1] = torch.maximum(dig[:, 0], dig[:, 1])
nt = torch.full((U,), 512 * 64 - 30, dtype=torch.int32, device="cuda")
table = torch.as_tensor(np.where(rng.random((U, nbs)) < 0.9, np.arange(U * nbs).reshape(U, nbs) % 15000, -1)
                        .astype(np.int32), device="cuda")
qb = torch.randn(U * G, D, device="cuda").to(torch.bfloat16)
out = {}
m, lo = med(lambda: ops.score_topk_split(qb, dig, nt, 64, G, block_table=table, out=out))
k1_bytes = U * 2 * D * 512 * 2
print(f"K1 one layer: median {m:.1f} us (min {lo:.1f}), {k1_bytes / m / 1e3:.0f} GB/s of live digests")
