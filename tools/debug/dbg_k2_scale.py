import sys, math
sys.path[:0] = ["tests", "oracle", "."]
import numpy as np, torch
from paper_2603_27138_b200 import ops
U_list = [int(x) for x in sys.argv[1:]] or [32, 64, 128]
for U in U_list:
    G = 8
    per = 64
    pool = ops.alloc_pool(U * per, torch.bfloat16)
    pool.view(torch.bfloat16).normal_()
    rng = np.random.default_rng(U)
    res_slots = torch.arange(U * per, dtype=torch.int32).view(U, per).cuda()
    res_ids = torch.from_numpy(np.sort(np.stack([rng.choice(512, per, replace=False) for _ in range(U)]), 1).astype(np.int32)).cuda()
    n_res = torch.full((U,), per, dtype=torch.int32, device="cuda")
    n_tok = torch.full((U,), 32768, dtype=torch.int32, device="cuda")
    q = torch.randn(U * G, 128, device="cuda")
    co = torch.randn(U * G, 128, device="cuda")
    cml = torch.stack([torch.randn(U * G), torch.rand(U * G) * 10 + 1], 1).cuda().contiguous()
    try:
        o, ml = ops.sparse_decode(q, pool, torch.bfloat16, res_slots, res_ids, n_res, n_tok, G, cpu_o=co, cpu_ml=cml)
        torch.cuda.synchronize()
        print(U, "ok", float(o.abs().max()))
    except Exception as e:
        print(U, "FAIL", e)
        break
