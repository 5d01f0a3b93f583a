"""The composed decode step: the engine's device tier mode with its in-engine
CPU co-attention worker (cfg.cpu_worker: the reference's PrecomputeWorker,
engine.hpp:88-150) computing every layer's CPU partial during the step from
the CPU-side ids K1 selected in that same step and the step's predicted
queries (engine.hpp:236-251), and K2 merging each layer chunk as it lands
(engine.hpp:262-273).

Every (step, layer, unit) output is checked against the reference's own
hybrid-query oracle, recompute_layer_attention (harness.hpp:318-329, through
oracle/_ref): q_true over the resident share, q_pred over the CPU share, both
truncated to the tokens present at the attention, merged and finalised. The
split itself is checked by the engine on the device (check_split,
engine.hpp:317-329) after every step."""
import math

import numpy as np
import pytest
import torch

import py_oracle as P
from paper_2603_27138_b200.engine import DecodeEngine, LayerState
from test_gpu_engine_tier import Side

pytestmark = pytest.mark.gpu
D, BS = 128, 64
BF16_RTOL = 2e-2


def bf16(x):
    return torch.as_tensor(x).to(torch.bfloat16).double().numpy()


@pytest.mark.parametrize("cpu_dtype", [torch.float32, torch.bfloat16])
@pytest.mark.parametrize("G", [4, 8])
def test_engine_with_cpu_worker_matches_recompute_layer_attention(cuda, cpu_dtype, G):
    if P.ref() is None or not hasattr(P.ref(), "ref_recompute_layer_attention"):
        pytest.skip("oracle/_ref without harness.hpp")
    torch.manual_seed(G)
    L, batch, hkv, k, cap, nbs, steps = 4, 2, 2, 6, 8, 24, 12
    U = batch * hkv
    kv = torch.bfloat16
    T0 = 64 * 12 + 40
    seed_rows = [[(torch.randn(U, D), torch.randn(U, D)) for _ in range(T0)] for _ in range(L)]
    sd = Side(L, U, nbs, cap, kv, seed_rows)
    # the K/V stream each (layer, unit) holds, as the cache stores it (bf16)
    K = [[[bf16(seed_rows[l][t][0][u]) for t in range(T0)] for u in range(U)] for l in range(L)]
    V = [[[bf16(seed_rows[l][t][1][u]) for t in range(T0)] for u in range(U)] for l in range(L)]
    layers = [LayerState(sd.dig[i], torch.full((U, nbs), -1, dtype=torch.int32, device="cuda")) for i in range(L)]
    eng = DecodeEngine(layers=L, batch=batch, hq=hkv * G, hkv=hkv, k=k, n_tokens=sd.n_tokens, pool=sd.pool,
                       kv_dtype=kv, layer_states=layers, scale=1 / math.sqrt(D), recall_interval=3,
                       host_tier=sd.host, tier=sd.tier, host_blocks=0, q_dtype=torch.bfloat16, host_staging=True,
                       chunk_layers=2, cpu_dtype=cpu_dtype, cpu_worker=True, cpu_threads=4)
    h_out = torch.empty(L, U * G, D).pin_memory()
    h_ml = torch.empty(L, U * G, 2).pin_memory()
    h_ids = torch.empty(L, U, k, dtype=torch.int32).pin_memory()
    h_n = torch.empty(L, U, dtype=torch.int32).pin_memory()
    with pytest.raises(ValueError):  # the engine computes the partials itself
        eng.decode_step_kv_host(1, torch.zeros(L, U * G, D).bfloat16(), torch.zeros(L, U * G, D).bfloat16(),
                                torch.zeros(L, U * G, D).to(cpu_dtype), torch.zeros(L, U * G, 2), None, None, h_out,
                                h_ml)
    cpu_blocks = 0
    for step in range(1, steps + 1):
        qt = torch.randn(L, U * G, D).bfloat16()
        qp = (qt.float() + 0.3 * torch.randn(L, U * G, D)).bfloat16()
        kn, vn = torch.randn(L, U, D), torch.randn(L, U, D)
        ins = [t.pin_memory() for t in (qt, qp, kn, vn)]
        eng.decode_step_kv_host(step, ins[0], ins[1], None, None, ins[2], ins[3], h_out, h_ml, h_ids, h_n)
        eng.sync()
        torch.cuda.synchronize()
        eng.check_state()  # check_split held for every (layer, unit); no rejected ticket
        lists = {n: t.cpu().numpy() for n, t in eng.k1_outputs().items()}
        t_att = T0 + step - 1  # tokens present at the attention (the append follows it)
        for l in range(L):
            for u in range(U):
                K[l][u].append(bf16(kn[l, u]))
                V[l][u].append(bf16(vn[l, u]))
        for l in range(L):
            assert np.array_equal(h_n[l].numpy(), lists["n_cpu"][l])
            for u in range(U):
                res = lists["res_ids"][l, u, :lists["n_res"][l, u]]
                cpu = lists["cpu_ids"][l, u, :lists["n_cpu"][l, u]]
                cpu_blocks += len(cpu)
                want = P.recompute_layer_attention(np.vstack(K[l][u]), np.vstack(V[l][u]), t_att,
                                                   qt[l, u * G:(u + 1) * G].double().numpy(),
                                                   qp[l, u * G:(u + 1) * G].double().numpy(), res, cpu, 1 / math.sqrt(D))
                got = h_out[l, u * G:(u + 1) * G].double().numpy()
                for g in range(G):
                    err = np.abs(got[g] - want[g]).max()
                    assert err <= BF16_RTOL * max(np.abs(want[g]).max(), 1e-30), (step, l, u, g, err)
    assert cpu_blocks > 0  # the worker had CPU-side blocks to attend
    ms, n = eng.worker_stats()
    assert n == steps and ms > 0
    with pytest.raises(ValueError):
        eng.decode_step_kv(steps + 1, *(torch.zeros(L, U * G, D, device="cuda").bfloat16() for _ in range(2)), None, None,
                           torch.zeros(L, U, D, device="cuda"), torch.zeros(L, U, D, device="cuda"),
                           torch.empty(L, U * G, D, device="cuda"), torch.empty(L, U * G, 2, device="cuda"))
    eng.close()
