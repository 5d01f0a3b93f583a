import sys, math
sys.path[:0] = ["tests", "oracle", "."]
import numpy as np, torch
from test_gpu_decode import build_case, oracle_outputs
from paper_2603_27138_b200 import ops

for G, max_ctas, seed in [(2, 0, 2000), (1, 3, 1003), (8, 7, 77), (4, 0, 4000)]:
    rng = np.random.default_rng(seed)
    U = 10
    nb_list = [int(x) for x in rng.integers(1, 40, size=U)]
    n_res = [int(rng.integers(0, nb + 1)) for nb in nb_list]
    n_res[0] = 0; n_res[1] = nb_list[1]
    c = build_case(rng, U, G, nb_list, n_res, torch.bfloat16)
    d = c["dev"]
    wo, wml = oracle_outputs(c, U, G, torch.bfloat16)
    for rep in range(3):
        o, ml = ops.sparse_decode(d["q"], c["pool"], torch.bfloat16, d["res_slots"], d["res_ids"], d["n_res"], d["n_tokens"], G, max_ctas=max_ctas)
        torch.cuda.synchronize()
        o = o.cpu().double().numpy(); ml = ml.cpu().double().numpy()
        bad = []
        for h in range(U * G):
            if wml[h, 1] == 0:
                ok = np.all(o[h] == 0)
            else:
                ok = np.abs(o[h] - wo[h]).max() <= 2e-2 * np.abs(wo[h]).max()
            if not ok:
                bad.append((h // G, h % G, float(np.abs(o[h] - wo[h]).max()), ml[h].tolist(), wml[h].tolist()))
        print(f"G={G} max_ctas={max_ctas} rep={rep} n_res={n_res} nb={nb_list} T={sum(n_res)} bad={len(bad)}")
        for b in bad[:6]:
            print("   ", b)
