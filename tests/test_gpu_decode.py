"""K2 (+fused K3) parity on the GPU against the oracle / reference golden
vectors: bf16 KV within 2e-2 relative (max-abs error / max-abs reference per
head), f32 KV within 1e-3 max-abs — the north star's tolerances."""
import math

import numpy as np
import pytest
import torch

import py_oracle as P
from helpers import D, from_bf16, load_golden
from paper_2603_27138_b200 import ops

pytestmark = pytest.mark.gpu
BF16_RTOL = 2e-2
F32_ATOL = 1e-3


def build_case(rng, U, G, nb_list, n_res_list, dtype, kscale=1.0):
    """Random units: unit u has nb_list[u] blocks (last one ragged) of which
    n_res_list[u] (ascending ids, incl. possibly the open block) are resident."""
    dev = torch.device("cuda")
    tot_slots = sum(n_res_list) + 1
    pool = ops.alloc_pool(tot_slots, dtype)
    ks = max(max(n_res_list), 1)
    res_slots = np.zeros((U, ks), np.int32)
    res_ids = np.zeros((U, ks), np.int32)
    n_tokens = np.zeros(U, np.int32)
    host = {}
    slot = 1  # slot 0 unused: catches off-by-one reads
    perm = rng.permutation(tot_slots - 1) + 1
    for u in range(U):
        nb = nb_list[u]
        tail = int(rng.integers(1, 65))
        n_tokens[u] = 64 * (nb - 1) + tail
        ids = np.sort(rng.choice(nb, size=n_res_list[u], replace=False)) if n_res_list[u] else np.zeros(0, int)
        for j, bid in enumerate(ids):
            rows = tail if bid == nb - 1 else 64
            k = rng.standard_normal((rows, D)).astype(np.float32) * kscale
            v = rng.standard_normal((rows, D)).astype(np.float32)
            s = int(perm[slot - 1])
            slot += 1
            ops.write_blocks(pool, dtype, [s], torch.from_numpy(k)[None], torch.from_numpy(v)[None])
            host[(u, j)] = (k, v)
            res_slots[u, j], res_ids[u, j] = s, bid
    q = rng.standard_normal((U * G, D)).astype(np.float32)
    to = lambda a: torch.as_tensor(a, device=dev)  # noqa: E731
    n_res = np.array(n_res_list, np.int32)
    return dict(pool=pool, q=q, res_slots=res_slots, res_ids=res_ids, n_res=n_res, n_tokens=n_tokens, host=host,
                dev=dict(q=to(q), res_slots=to(res_slots), res_ids=to(res_ids), n_res=to(n_res),
                         n_tokens=to(n_tokens)))


def oracle_outputs(c, U, G, dtype, cpu=None, scale=1 / math.sqrt(D)):
    rnd = (lambda x: torch.from_numpy(x).bfloat16().double().numpy()) if dtype == torch.bfloat16 else (
        lambda x: x.astype(np.float64))
    out_o = np.zeros((U * G, D))
    out_ml = np.zeros((U * G, 2))
    for u in range(U):
        ks = [rnd(c["host"][(u, j)][0]) for j in range(c["n_res"][u])]
        vs = [rnd(c["host"][(u, j)][1]) for j in range(c["n_res"][u])]
        kk = np.vstack(ks) if ks else np.zeros((0, D))
        vv = np.vstack(vs) if vs else np.zeros((0, D))
        for g in range(G):
            h = u * G + g
            p = P.partial_attention(c["q"][h].astype(np.float64), kk, vv, scale)
            if cpu is not None and cpu[1][h, 1] > 0:
                co, cml = cpu[0][h].astype(np.float64), cpu[1][h]
                pc = P.Partial(co * cml[1], float(cml[0]), float(cml[1]), 1)
                p = P.merge(p, pc)
            if p.count == 0:
                out_o[h], out_ml[h] = 0.0, (-np.inf, 0.0)
            else:
                out_o[h] = P.finalize(p)
                out_ml[h] = (p.max_logit, p.denom)
    return out_o, out_ml


def check(o, ml, want_o, want_ml, dtype):
    o, ml = o.cpu().double().numpy(), ml.cpu().double().numpy()
    for h in range(o.shape[0]):
        if want_ml[h, 1] == 0:
            assert np.all(o[h] == 0) and ml[h, 1] == 0 and ml[h, 0] == -np.inf
            continue
        err = np.abs(o[h] - want_o[h]).max()
        if dtype == torch.bfloat16:
            assert err <= BF16_RTOL * max(np.abs(want_o[h]).max(), 1e-30), (h, err)
        else:
            assert err <= F32_ATOL, (h, err)
        # (m, l) describe the same partial: compare l * exp(m) relative
        lse_got = ml[h, 0] + math.log(ml[h, 1])
        lse_want = want_ml[h, 0] + math.log(want_ml[h, 1])
        assert abs(lse_got - lse_want) <= (5e-3 if dtype == torch.bfloat16 else 1e-4), h


@pytest.mark.parametrize("G", [1, 2, 4, 8])
@pytest.mark.parametrize("dtype", [torch.bfloat16, torch.float32])
@pytest.mark.parametrize("max_ctas", [0, 3, 40])
def test_sparse_decode_vs_oracle(cuda, G, dtype, max_ctas):
    rng = np.random.default_rng(1000 * G + max_ctas + (dtype == torch.float32))
    U = 10
    nb_list = [int(x) for x in rng.integers(1, 40, size=U)]
    n_res = [int(rng.integers(0, nb + 1)) for nb in nb_list]
    n_res[0] = 0
    n_res[1] = nb_list[1]
    c = build_case(rng, U, G, nb_list, n_res, dtype)
    d = c["dev"]
    o, ml = ops.sparse_decode(d["q"], c["pool"], dtype, d["res_slots"], d["res_ids"], d["n_res"], d["n_tokens"], G,
                              max_ctas=max_ctas)
    torch.cuda.synchronize()
    check(o, ml, *oracle_outputs(c, U, G, dtype), dtype)


@pytest.mark.parametrize("dtype", [torch.bfloat16, torch.float32])
def test_sparse_decode_merges_cpu_partial(cuda, dtype):
    rng = np.random.default_rng(77)
    U, G = 12, 8
    nb_list = [int(x) for x in rng.integers(2, 30, size=U)]
    n_res = [int(rng.integers(0, nb + 1)) for nb in nb_list]
    n_res[3] = 0
    c = build_case(rng, U, G, nb_list, n_res, dtype)
    cpu_o = rng.standard_normal((U * G, D)).astype(np.float32)
    cpu_ml = np.stack([rng.standard_normal(U * G) * 2, rng.random(U * G) * 30 + 0.5], axis=1).astype(np.float32)
    cpu_ml[5 * G:6 * G] = (-np.inf, 0.0)  # empty CPU side for unit 5
    cpu_ml[3 * G + 1] = (-np.inf, 0.0)   # unit 3: both empty for head 1
    d = c["dev"]
    o, ml = ops.sparse_decode(d["q"], c["pool"], dtype, d["res_slots"], d["res_ids"], d["n_res"], d["n_tokens"], G,
                              cpu_o=torch.as_tensor(cpu_o, device="cuda"),
                              cpu_ml=torch.as_tensor(cpu_ml, device="cuda"), max_ctas=7)
    torch.cuda.synchronize()
    check(o, ml, *oracle_outputs(c, U, G, dtype, cpu=(cpu_o, cpu_ml)), dtype)


@pytest.mark.parametrize("G", [1, 8])
def test_sparse_decode_bf16_queries(cuda, G):
    """bf16 queries (q_dtype = SCOUT_BF16) against the oracle on the same
    bf16-rounded query values, with a CPU partial merge."""
    rng = np.random.default_rng(500 + G)
    U = 9
    nb_list = [int(x) for x in rng.integers(1, 30, size=U)]
    n_res = [int(rng.integers(0, nb + 1)) for nb in nb_list]
    c = build_case(rng, U, G, nb_list, n_res, torch.bfloat16)
    c["q"] = torch.from_numpy(c["q"]).bfloat16().float().numpy()
    cpu_o = rng.standard_normal((U * G, D)).astype(np.float32)
    cpu_ml = np.stack([rng.standard_normal(U * G), rng.random(U * G) * 10 + 0.5], axis=1).astype(np.float32)
    d = c["dev"]
    o, ml = ops.sparse_decode(d["q"].bfloat16(), c["pool"], torch.bfloat16, d["res_slots"], d["res_ids"], d["n_res"],
                              d["n_tokens"], G, cpu_o=torch.as_tensor(cpu_o, device="cuda"),
                              cpu_ml=torch.as_tensor(cpu_ml, device="cuda"), max_ctas=5)
    torch.cuda.synchronize()
    check(o, ml, *oracle_outputs(c, U, G, torch.bfloat16, cpu=(cpu_o, cpu_ml)), torch.bfloat16)


def test_sparse_decode_large_logits_bf16(cuda):
    """Keys scaled x8: logits of tens, exercises the online-softmax rescaling."""
    rng = np.random.default_rng(9)
    U, G = 6, 8
    nb_list = [64] * U
    c = build_case(rng, U, G, nb_list, [64, 33, 1, 64, 10, 50], torch.bfloat16, kscale=8.0)
    d = c["dev"]
    o, ml = ops.sparse_decode(d["q"], c["pool"], torch.bfloat16, d["res_slots"], d["res_ids"], d["n_res"],
                              d["n_tokens"], G)
    torch.cuda.synchronize()
    check(o, ml, *oracle_outputs(c, U, G, torch.bfloat16), torch.bfloat16)


@pytest.mark.parametrize("case", sorted(load_golden("attention")))
def test_decode_vs_reference_golden(cuda, case):
    """Reference partial_attention + merge + finalize (golden) reproduced by
    K2 with the second partial fed as the CPU partial."""
    g = load_golden("attention")[case]
    rows = [int(r) for r in g["rows"]]
    k, v = from_bf16(g["k"]), from_bf16(g["v"])
    n = sum(rows)
    # pack the rows contiguously into full blocks (+ one ragged open block)
    nb = (n + 63) // 64
    pool = ops.alloc_pool(nb, torch.bfloat16)
    kp = np.zeros((nb * 64, D), np.float32)
    vp = np.zeros((nb * 64, D), np.float32)
    kp[:n], vp[:n] = k, v
    ops.write_blocks(pool, torch.bfloat16, list(range(nb)), torch.from_numpy(kp).view(nb, 64, D),
                     torch.from_numpy(vp).view(nb, 64, D))
    dev = torch.device("cuda")
    t = lambda a, dt=torch.int32: torch.as_tensor(np.asarray(a), dtype=dt, device=dev)  # noqa: E731
    q = t(g["q"][None], torch.float32)
    cpu_o = t((g["o2_acc"] / g["l2"])[None], torch.float32)
    cpu_ml = t(np.array([[g["m2"], g["l2"]]]), torch.float32)
    o, ml = ops.sparse_decode(q, pool, torch.bfloat16, t([list(range(nb))]), t([list(range(nb))]), t([nb]), t([n]),
                              1, float(g["scale"]), cpu_o=cpu_o, cpu_ml=cpu_ml)
    o = o.cpu().double().numpy()[0]
    assert np.abs(o - g["final"]).max() <= BF16_RTOL * np.abs(g["final"]).max()
    ml = ml.cpu().double().numpy()[0]
    lse = ml[0] + math.log(ml[1])
    assert abs(lse - (g["merged_m"] + math.log(g["merged_l"]))) < 5e-3


@pytest.mark.parametrize("case", ["one_cta_many_units", "few_units_many_ctas"])
def test_sparse_decode_segment_edges(cuda, case):
    """K2's combine paths: one CTA holding 40 units (40 segments handed to the
    combiner warp back to back, 22 units without a resident block: more than
    the plan lists, so the combiner scans n_res) and two long units spread
    over 60 CTAs (the cross-CTA finalize of many partial slots), each with a
    CPU partial to merge."""
    rng = np.random.default_rng(4242 + (case == "few_units_many_ctas"))
    G = 8
    if case == "one_cta_many_units":
        U, max_ctas = 40, 1
        nb_list = [int(x) for x in rng.integers(1, 6, size=U)]
        n_res = [0 if u % 2 == 0 or u > 34 else int(rng.integers(1, nb_list[u] + 1)) for u in range(U)]
    else:
        U, max_ctas = 2, 60
        nb_list = [200, 150]
        n_res = [200, 131]
    c = build_case(rng, U, G, nb_list, n_res, torch.bfloat16)
    cpu_o = rng.standard_normal((U * G, D)).astype(np.float32)
    cpu_ml = np.stack([rng.standard_normal(U * G), rng.random(U * G) * 10 + 0.5], axis=1).astype(np.float32)
    cpu_ml[:G] = (-np.inf, 0.0)  # unit 0: no CPU side
    d = c["dev"]
    o, ml = ops.sparse_decode(d["q"], c["pool"], torch.bfloat16, d["res_slots"], d["res_ids"], d["n_res"],
                              d["n_tokens"], G, cpu_o=torch.as_tensor(cpu_o, device="cuda"),
                              cpu_ml=torch.as_tensor(cpu_ml, device="cuda"), max_ctas=max_ctas)
    torch.cuda.synchronize()
    check(o, ml, *oracle_outputs(c, U, G, torch.bfloat16, cpu=(cpu_o, cpu_ml)), torch.bfloat16)
