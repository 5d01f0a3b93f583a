# time K2 alone at config-3 scale (256 units x 59 resident blocks), many launches
import sys, time
sys.path[:0] = ["."]
import numpy as np, torch
from paper_2603_27138_b200 import ops
import os
U, G, nb = 256, 8, 512
per = int(os.environ.get('PER', '59'))
L = 8  # distinct "layers" to defeat L2
pool = ops.alloc_pool(L * U * per, torch.bfloat16)
pool.view(torch.bfloat16).normal_()
rng = np.random.default_rng(0)
args = []
for l in range(L):
    slots = torch.from_numpy((l * U * per + rng.permutation(U * per)).reshape(U, per).astype(np.int32)).cuda()
    ids = torch.from_numpy(np.sort(np.stack([rng.choice(nb, per, replace=False) for _ in range(U)]), 1).astype(np.int32)).cuda()
    args.append((slots, ids))
n_res = torch.full((U,), per, dtype=torch.int32, device="cuda")
n_tok = torch.full((U,), nb * 64, dtype=torch.int32, device="cuda")
q = torch.randn(U * G, 128, device="cuda")
ws = ops.DecodeWorkspace(U, G)
o = torch.empty(U * G, 128, device="cuda"); ml = torch.empty(U * G, 2, device="cuda")
for i in range(5):
    s, d = args[i % L]
    ops.sparse_decode(q, pool, torch.bfloat16, s, d, n_res, n_tok, G, o=o, ml=ml, workspace=ws)
torch.cuda.synchronize()
e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
N = 64
e0.record()
for i in range(N):
    s, d = args[i % L]
    ops.sparse_decode(q, pool, torch.bfloat16, s, d, n_res, n_tok, G, o=o, ml=ml, workspace=ws)
e1.record(); torch.cuda.synchronize()
us = e0.elapsed_time(e1) / N * 1000
byts = U * per * 64 * 2 * 128 * 2
print(f"K2 {us:.1f} us/launch, {byts / us / 1e3:.0f} GB/s")
