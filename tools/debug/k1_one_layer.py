"""K1 (and K2) of ONE config-3 layer, as the layer-by-layer mode launches them
(256 units, nb_stride 520, G=8, top-64, bf16 queries and digests; K2: 256 units,
59 resident blocks): a few launches for ncu (-k regex:score_topk -s 3 -c 1)."""
import sys
sys.path[:0] = [".", "tests", "oracle"]
import numpy as np
import torch
from paper_2603_27138_b200 import ops

rng = np.random.default_rng(0)
U, G, D = 256, 8, 128
nbs = 520
dig = torch.randn(U, 2, D, nbs, device="cuda").to(torch.bfloat16)
dig[:, 1] = torch.maximum(dig[:, 0], dig[:, 1])
nt = torch.full((U,), 512 * 64 - 30, dtype=torch.int32, device="cuda")
table = torch.as_tensor(np.where(rng.random((U, nbs)) < 0.9, np.arange(U * nbs).reshape(U, nbs) % 15000, -1)
                        .astype(np.int32), device="cuda")
qb = torch.randn(U * G, D, device="cuda").to(torch.bfloat16)
out = {}
for _ in range(6):
    ops.score_topk_split(qb, dig, nt, 64, G, block_table=table, out=out)
torch.cuda.synchronize()
print("done")
