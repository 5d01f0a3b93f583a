"""The bench's own workload (bench.TierWorkload: config-3 shape, 64 layers,
32K context, top-64, per-layer slot counts) through the engine, then checked:
  * slot accounting of the device tier state: every (layer, unit)'s table
    entries are distinct slots of its own range, disjoint from its free stack,
    and together they account for every slot it owns;
  * bench.verify_step (float64 re-derivation of one step) passes;
  * K1's sets for sampled (layer, unit) pairs are bit-exact against the
    oracle's stacked select_topk (the reference's sequential sum order) on the
    digests and queries of that step."""
import math

import numpy as np
import pytest
import torch

import py_oracle as P

pytestmark = pytest.mark.gpu


def _workload(batch, policy, steps, warm=0):
    import bench

    cfg = dict(bench.CONFIGS["qwen3-32b-32k"])
    cfg.update(q_dtype=torch.bfloat16, cpu_dtype=torch.bfloat16, drift=0.15, recall_policy=policy, batch=batch)
    wl = bench.TierWorkload(cfg, torch.device("cuda"), 1234, steps + 16, range(batch), warm_slots=warm)
    wl.make_engine()
    return bench, wl


@pytest.mark.parametrize("policy,warm", [("reference", 0), ("reference", 48), ("stagger", 48)])
def test_bench_workload_slots_and_verify(cuda, policy, warm):
    """warm > 0: the bench's victim cache (warm images placed with the fast
    set, then every evicted block's): recalls served warm, same checks."""
    steps = 40
    bench, wl = _workload(2, policy, steps, warm)
    for s in range(1, steps + 1):
        wl.step(s)
    wl.engine.sync()
    torch.cuda.synchronize()
    wl.engine.check_state()
    tr = wl.tier
    for l in range(wl.L):
        spu = tr.spu_l[l]
        for u in range(wl.U):
            base = tr.layer_base[l] + u * spu
            used = tr.table[l, u][tr.table[l, u] >= 0].cpu().numpy()
            free = np.array(tr.free_ring(l, u), dtype=np.int64)
            assert len(set(used.tolist())) == len(used), (l, u)
            allslots = np.concatenate([used, free])
            assert len(set(allslots.tolist())) == len(allslots) == spu, (l, u)
            assert allslots.min() >= base and allslots.max() < base + spu, (l, u)
    if warm:
        w, c = wl.engine.recall_stats()
        assert w > 0
    v = bench.verify_step(wl, steps + 1)
    assert v["pass"], v


def test_bench_workload_topk_bit_exact(cuda):
    """K1 at the bench shape (512+ blocks, G=8, k=64, bf16 queries and digests)
    against the oracle's stacked select_topk for sampled (layer, unit) pairs."""
    bench, wl = _workload(1, "reference", 4)
    for s in range(1, 4):
        wl.step(s)
    wl.engine.sync()
    torch.cuda.synchronize()
    ntok = wl.n_tokens.cpu().numpy()
    j = 4 % len(wl.q_path_t)
    digs = {l: wl.layer_states[l].digests.double().cpu().numpy() for l in (0, 1, 31, 63)}
    wl.step(4)
    wl.engine.sync()
    torch.cuda.synchronize()
    k1 = {n: t.cpu().numpy() for n, t in wl.engine.k1_outputs().items()}
    G, k = wl.G, wl.k
    for l, dig in digs.items():
        q = (wl.q_path_t[j][0] if l == 0 else wl.q_path_p[j][l]).float().cpu().numpy()
        for u in range(wl.U):
            nb = (int(ntok[u]) + 63) // 64
            want, _ = P.unit_topk(q[u * G:(u + 1) * G].astype(np.float64), dig[u], nb, k)
            got = np.sort(np.concatenate([k1["res_ids"][l, u, :k1["n_res"][l, u]],
                                          k1["cpu_ids"][l, u, :k1["n_cpu"][l, u]]]))
            assert np.array_equal(np.sort(want), got), (l, u)
