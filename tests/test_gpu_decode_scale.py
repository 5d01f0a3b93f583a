"""K2 (+fused K3) at the benchmarked shapes, against the oracle on a sample of
units: config 3's layer (256 units, G=8, ~59 of 512 blocks resident per unit,
top-64, default persistent grid), config 4's batch 128 at one GPU (1024
units: a CTA's range holds more blocks than one plan chunk), skewed residency
(ranges touching more units than one plan chunk lists), and long single units
split over many chunks on one CTA. Pools hold only the resident blocks, filled
on the device; the sampled units' rows are read back for the oracle
(partial_attention + merge + finalize, attention.hpp:73-122)."""
import math

import numpy as np
import pytest
import torch

import py_oracle as P
from paper_2603_27138_b200 import ops

pytestmark = pytest.mark.gpu
D, BS = 128, 64
BF16_RTOL = 2e-2


def build(rng, n_res, nb=512, n_tokens=None, k_stride=None, G=8, seed=0):
    """Unit u: n_res[u] resident blocks, ascending random ids among nb (the open
    block nb-1 included for some units), pool slots shuffled."""
    dev = torch.device("cuda")
    U = len(n_res)
    ks = k_stride or max(max(n_res), 1)
    tot = int(sum(n_res))
    pool = ops.alloc_pool(tot + 1, torch.bfloat16)
    g = torch.Generator(device=dev).manual_seed(seed)
    pool.view(torch.bfloat16).normal_(generator=g)
    res_ids = np.zeros((U, ks), np.int32)
    res_slots = np.zeros((U, ks), np.int32)
    perm = rng.permutation(tot) + 1
    if n_tokens is None:
        n_tokens = np.full(U, nb * BS, np.int32)
        n_tokens[::3] -= rng.integers(1, 64, size=len(n_tokens[::3])).astype(np.int32)  # ragged open blocks
    pos = 0
    for u in range(U):
        n = n_res[u]
        nbu = (int(n_tokens[u]) + BS - 1) // BS
        ids = np.sort(rng.choice(nbu, size=n, replace=False)) if n else np.zeros(0, np.int64)
        if n and u % 2 == 0:
            ids[-1] = nbu - 1  # the open block (always resident in the reference)
            ids = np.unique(ids)
            while len(ids) < n:
                ids = np.unique(np.append(ids, rng.integers(0, nbu - 1)))
        res_ids[u, :n] = ids
        res_slots[u, :n] = perm[pos:pos + n]
        pos += n
    q = torch.randn(U * G, D, device=dev, generator=g)
    to = lambda a: torch.as_tensor(a, device=dev)  # noqa: E731
    return dict(pool=pool, q=q, res_ids=res_ids, res_slots=res_slots, n_res=np.asarray(n_res, np.int32),
                n_tokens=np.asarray(n_tokens, np.int32), U=U, G=G,
                dev=dict(res_slots=to(res_slots), res_ids=to(res_ids), n_res=to(np.asarray(n_res, np.int32)),
                         n_tokens=to(np.asarray(n_tokens, np.int32))))


def unit_rows(c, u):
    """K and V rows unit u's resident blocks hold (valid rows only), as f64."""
    n = int(c["n_res"][u])
    if n == 0:
        return np.zeros((0, D)), np.zeros((0, D))
    nt = int(c["n_tokens"][u])
    nb = (nt + BS - 1) // BS
    slots, rows = [], []
    for j in range(n):
        r = nt - (nb - 1) * BS if c["res_ids"][u, j] == nb - 1 else BS
        slots += [int(c["res_slots"][u, j])] * r
        rows += list(range(r))
    k, v = ops.kv_read_tokens(c["pool"], torch.bfloat16, slots, rows)
    return k.double().cpu().numpy(), v.double().cpu().numpy()


def check_units(c, o, ml, units, q=None, cpu=None, scale=1 / math.sqrt(D)):
    G = c["G"]
    q = (c["q"] if q is None else q).float().cpu().numpy()
    o, ml = o.cpu().double().numpy(), ml.cpu().double().numpy()
    for u in units:
        kk, vv = unit_rows(c, u)
        for gh in range(G):
            h = u * G + gh
            p = P.partial_attention(q[h].astype(np.float64), kk, vv, scale)
            if cpu is not None and cpu[1][h, 1] > 0:
                p = P.merge(p, P.Partial(cpu[0][h].astype(np.float64) * cpu[1][h, 1], float(cpu[1][h, 0]),
                                         float(cpu[1][h, 1]), 1))
            if p.count == 0:
                assert np.all(o[h] == 0) and ml[h, 1] == 0, (u, gh)
                continue
            want = P.finalize(p)
            err = np.abs(o[h] - want).max()
            assert err <= BF16_RTOL * np.abs(want).max(), (u, gh, err)
            lse = ml[h, 0] + math.log(ml[h, 1])
            assert abs(lse - (p.max_logit + math.log(p.denom))) <= 5e-3, (u, gh)


def run(c, max_ctas=0, cpu=None, q=None):
    d = c["dev"]
    kw = {}
    if cpu is not None:
        kw = dict(cpu_o=torch.as_tensor(cpu[0], device="cuda"), cpu_ml=torch.as_tensor(cpu[1], device="cuda"))
    o, ml = ops.sparse_decode(c["q"] if q is None else q, c["pool"], torch.bfloat16, d["res_slots"], d["res_ids"],
                              d["n_res"], d["n_tokens"], c["G"], max_ctas=max_ctas, **kw)
    torch.cuda.synchronize()
    return o, ml


def cpu_partials(rng, UG):
    cpu_o = rng.standard_normal((UG, D)).astype(np.float32)
    cpu_ml = np.stack([rng.standard_normal(UG), rng.random(UG) * 20 + 0.5], axis=1).astype(np.float32)
    cpu_ml[::7] = (-np.inf, 0.0)
    return cpu_o, cpu_ml


def sample(rng, U, n=24):
    return sorted(set([0, 1, U - 1] + [int(x) for x in rng.choice(U, size=min(n, U), replace=False)]))


@pytest.mark.parametrize("q_bf16", [False, True])
def test_config3_layer_shape(cuda, q_bf16):
    """256 units (batch 32 x 8 KV heads), G=8, 50-64 of 512 blocks resident,
    k=64, default grid (one CTA per SM), a CPU partial merged."""
    rng = np.random.default_rng(3)
    U = 256
    n_res = [int(x) for x in rng.integers(50, 65, size=U)]
    c = build(rng, n_res, k_stride=64, seed=3)
    q = c["q"].bfloat16() if q_bf16 else c["q"]
    cpu = cpu_partials(rng, U * 8)
    o, ml = run(c, cpu=cpu, q=q)
    check_units(c, o, ml, sample(rng, U), q=q, cpu=cpu)


def test_skewed_residency(cuda):
    """100 consecutive units with 1 resident block next to 156 with 64: the
    first CTAs' ranges touch ~68 units (more than one plan chunk lists)."""
    rng = np.random.default_rng(4)
    n_res = [1] * 100 + [64] * 156
    c = build(rng, n_res, k_stride=64, seed=4)
    cpu = cpu_partials(rng, 256 * 8)
    o, ml = run(c, cpu=cpu)
    check_units(c, o, ml, list(range(0, 100, 7)) + [99, 100, 101, 255] + sample(rng, 256, 8), cpu=cpu)


@pytest.mark.parametrize("max_ctas", [1, 2, 5])
def test_few_ctas_many_units(cuda, max_ctas):
    """One to five CTAs over 300 units of 0-3 blocks: every CTA's range spans
    dozens of plan chunks of 64 segments, with units without a resident block
    in between (CPU partial only, or zeros)."""
    rng = np.random.default_rng(50 + max_ctas)
    U = 300
    n_res = [int(x) for x in rng.integers(0, 4, size=U)]
    c = build(rng, n_res, nb=8, k_stride=4, seed=5)
    cpu = cpu_partials(rng, U * 8)
    o, ml = run(c, max_ctas=max_ctas, cpu=cpu)
    check_units(c, o, ml, list(range(U)), cpu=cpu)


@pytest.mark.parametrize("max_ctas", [1, 3])
def test_long_units_split_over_chunks(cuda, max_ctas):
    """Units of 300-512 resident blocks (k=512) on 1 or 3 CTAs: each CTA's
    segment of a unit is longer than a plan chunk, so it is split and the
    consumers carry the softmax state across chunks."""
    rng = np.random.default_rng(60 + max_ctas)
    n_res = [512, 300, 450, 389, 511]
    c = build(rng, n_res, nb=512, k_stride=512, seed=6)
    cpu = cpu_partials(rng, len(n_res) * 8)
    o, ml = run(c, max_ctas=max_ctas, cpu=cpu)
    check_units(c, o, ml, list(range(len(n_res))), cpu=cpu)


def test_config4_batch128_one_gpu(cuda):
    """1024 units (batch 128 x 8 KV heads), ~59 resident each: ~400 blocks
    per CTA range on 148 CTAs, above one plan chunk (384), so every CTA plans
    its range in two chunks; the grid stays at one CTA per SM."""
    rng = np.random.default_rng(7)
    U = 1024
    n_res = [int(x) for x in rng.integers(54, 65, size=U)]
    c = build(rng, n_res, k_stride=64, seed=7)
    cpu = cpu_partials(rng, U * 8)
    o, ml = run(c, cpu=cpu)
    check_units(c, o, ml, sample(rng, U, 20), cpu=cpu)


def test_grid_never_exceeds_sm_count(cuda):
    import paper_2603_27138_b200 as pkg

    sms = torch.cuda.get_device_properties(0).multi_processor_count
    lib = pkg.lib()
    for U, k in ((256, 64), (1024, 64), (1024, 512), (4096, 128)):
        assert lib.scout_sparse_decode_grid(U, k, 0) == sms
