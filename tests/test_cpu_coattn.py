"""CPU co-attention worker (scout_cpu_partial_attention, host only) against the
oracle's partial_attention (attention.hpp:73-95) on the same bf16 / f32 block
images: the host tier's swizzled bf16 tile layout is decoded correctly, ragged
rows are masked, empty units give (0, -inf, 0). AVX-512 fp32 vs double: 1e-4;
the AMX-BF16 kernel (bf16 hi+lo query, bf16 P as K2): 1e-2 of max |o| and
1e-3 on the log-sum-exp, the bf16 bar of SURVEY.md §8c."""
import math

import numpy as np
import pytest
import torch

import py_oracle as P
from paper_2603_27138_b200 import ops

D, B = 128, 64


def bf16_tile(x: np.ndarray) -> np.ndarray:
    """[64][128] values -> the pool's swizzled bf16 tile (as uint16)."""
    r = np.arange(B)[:, None]
    d = np.arange(D)[None, :]
    h, rr, j, c, e = r >> 5, r & 31, d >> 6, (d >> 3) & 7, d & 7
    off = (((h * 2 + j) * 32 + rr) << 6) + ((c ^ (rr & 7)) << 3) + e
    bits = torch.from_numpy(np.ascontiguousarray(x, dtype=np.float32)).bfloat16().view(torch.int16).numpy()
    out = np.zeros(B * D, np.int16)
    out[off.ravel()] = bits.ravel()
    return out


@pytest.mark.parametrize("kernel", ["auto", "avx512"])
@pytest.mark.parametrize("kv", ["bf16", "f32"])
@pytest.mark.parametrize("G", [1, 2, 4, 8])
def test_cpu_partial_attention_vs_oracle(kv, G, kernel, monkeypatch):
    if kernel == "avx512":
        if kv == "f32":
            pytest.skip("f32 images always take the AVX-512 kernel")
        monkeypatch.setenv("SCOUT_CPU_AMX", "0")
    dt0 = torch.bfloat16 if kv == "bf16" else torch.float32
    amx = ops.cpu_coattn_kernel(dt0) == "amx-bf16"
    tol_o, tol_lse = (1e-2, 1e-3) if amx else (1e-4, 1e-4)
    rng = np.random.default_rng(G + (kv == "f32") * 10)
    U, nblk, k = 7, 12, 6
    keys = rng.standard_normal((nblk, B, D)).astype(np.float32) * 1.5
    vals = rng.standard_normal((nblk, B, D)).astype(np.float32)
    dt = torch.bfloat16 if kv == "bf16" else torch.float32
    sb = ops.slot_bytes(dt)
    host = torch.zeros(nblk * sb, dtype=torch.uint8)
    for b in range(nblk):
        if kv == "bf16":
            img = np.concatenate([bf16_tile(keys[b]), bf16_tile(vals[b])]).view(np.uint8)
        else:
            img = np.concatenate([keys[b].ravel(), vals[b].ravel()]).view(np.uint8)
        host[b * sb:(b + 1) * sb] = torch.from_numpy(img)
    rnd = (lambda x: torch.from_numpy(x).bfloat16().double().numpy()) if kv == "bf16" else (lambda x: x.astype(np.float64))
    idx = np.zeros((U, k), np.int64)
    rows = np.full((U, k), B, np.int32)
    n = np.array([k, 3, 0, 1, k, 2, k], np.int32)
    for u in range(U):
        idx[u, :n[u]] = rng.choice(nblk, size=n[u], replace=False)
        if n[u]:
            rows[u, n[u] - 1] = int(rng.integers(1, B + 1))  # an open (ragged) block
    rows[5, 1] = 1  # one-row open block
    rows[6, 2] = 33  # odd fill: the last V pair is half valid
    q = rng.standard_normal((U * G, D)).astype(np.float32)
    scale = 1 / math.sqrt(D)
    o, ml = ops.cpu_partial_attention(host, dt, torch.from_numpy(idx), torch.from_numpy(n), torch.from_numpy(q), G,
                                      scale, block_rows=torch.from_numpy(rows), threads=3)
    o, ml = o.numpy(), ml.numpy()
    for u in range(U):
        kk = np.vstack([rnd(keys[idx[u, i], :rows[u, i]]) for i in range(n[u])]) if n[u] else np.zeros((0, D))
        vv = np.vstack([rnd(vals[idx[u, i], :rows[u, i]]) for i in range(n[u])]) if n[u] else np.zeros((0, D))
        for g in range(G):
            h = u * G + g
            p = P.partial_attention(q[h].astype(np.float64), kk, vv, scale)
            if p.count == 0:
                assert np.all(o[h] == 0) and ml[h, 0] == -np.inf and ml[h, 1] == 0
                continue
            want = P.finalize(p)
            assert np.abs(o[h] - want).max() <= tol_o * max(1.0, np.abs(want).max()), (u, g)
            lse = ml[h, 0] + math.log(ml[h, 1])
            assert abs(lse - (p.max_logit + math.log(p.denom))) <= tol_lse, (u, g)


def test_cpu_worker_stale_rows_and_pool():
    """Rows past an open block's fill may hold any bytes in the host tier (NaN
    included): they must not reach the result. Repeated calls with changing
    thread counts go through the persistent pool."""
    rng = np.random.default_rng(3)
    sb = ops.slot_bytes(torch.bfloat16)
    keys = rng.standard_normal((2, B, D)).astype(np.float32)
    vals = rng.standard_normal((2, B, D)).astype(np.float32)
    host = torch.zeros(2 * sb, dtype=torch.uint8)
    for b in range(2):
        img = np.concatenate([bf16_tile(keys[b]), bf16_tile(vals[b])]).view(np.uint8)
        host[b * sb:(b + 1) * sb] = torch.from_numpy(img)
    clean = host.clone()
    # poison rows 20..63 of block 1 (K and V) with NaN bit patterns
    r = np.arange(20, B)[:, None]
    d = np.arange(D)[None, :]
    h, rr, j, c, e = r >> 5, r & 31, d >> 6, (d >> 3) & 7, d & 7
    off = ((((h * 2 + j) * 32 + rr) << 6) + ((c ^ (rr & 7)) << 3) + e).ravel()
    u16 = host.view(torch.int16)
    for base in (sb // 2, sb // 2 + B * D):  # block 1's K tile, V tile (in int16 units)
        u16[torch.from_numpy(base + off)] = 0x7FC0
    U = 6
    idx = torch.tensor([[0, 1]] * U, dtype=torch.int64)
    n = torch.full((U,), 2, dtype=torch.int32)
    rows = torch.tensor([[B, 20]] * U, dtype=torch.int32)
    q = torch.from_numpy(rng.standard_normal((U * 8, D)).astype(np.float32))
    want = ops.cpu_partial_attention(clean, torch.bfloat16, idx, n, q, 8, block_rows=rows, threads=1)
    for t in (1, 4, 2, 8, 3):
        o, ml = ops.cpu_partial_attention(host, torch.bfloat16, idx, n, q, 8, block_rows=rows, threads=t)
        assert torch.isfinite(o).all() and torch.isfinite(ml).all()
        assert torch.equal(o, want[0]) and torch.equal(ml, want[1])


@pytest.mark.parametrize("kv", ["bf16", "f32"])
def test_cpu_partial_attention_ex_dtypes_and_claims(kv):
    """scout_cpu_partial_attention_ex (the model's dtypes): a bf16 query gives
    the bits its exact f32 widening gives, a bf16 o is the f32 result rounded
    to nearest even (torch's rounding, bit for bit), the f32/f32 call equals
    scout_cpu_partial_attention. Many units, most with no or one CPU-side
    block, so units are claimed several at a time; any thread count gives the
    same bits."""
    rng = np.random.default_rng(21 + (kv == "f32"))
    dt = torch.bfloat16 if kv == "bf16" else torch.float32
    sb = ops.slot_bytes(dt)
    nblk, U, k, G = 16, 600, 8, 8
    host = torch.zeros(nblk * sb, dtype=torch.uint8)
    for b in range(nblk):
        kb, vb = rng.standard_normal((2, B, D)).astype(np.float32)
        img = (np.concatenate([bf16_tile(kb), bf16_tile(vb)]) if kv == "bf16"
               else np.concatenate([kb.ravel(), vb.ravel()])).view(np.uint8)
        host[b * sb:(b + 1) * sb] = torch.from_numpy(img)
    n = torch.from_numpy(np.minimum(rng.poisson(0.7, U), k).astype(np.int32))
    idx = torch.from_numpy(rng.integers(0, nblk, (U, k)).astype(np.int64))
    q_bf = torch.from_numpy(rng.standard_normal((U * G, D)).astype(np.float32)).bfloat16()
    q32 = q_bf.float()
    o_ref, ml_ref = ops.cpu_partial_attention(host, dt, idx, n, q32, G, threads=1)
    for t in (1, 5):
        o, ml = ops.cpu_partial_attention_ex(host, dt, idx, n, q32, G, o_dtype=torch.float32, threads=t)
        assert torch.equal(o, o_ref) and torch.equal(ml, ml_ref)
        o, ml = ops.cpu_partial_attention_ex(host, dt, idx, n, q_bf, G, o_dtype=torch.float32, threads=t)
        assert torch.equal(o, o_ref) and torch.equal(ml, ml_ref)
        o, ml = ops.cpu_partial_attention_ex(host, dt, idx, n, q_bf, G, o_dtype=torch.bfloat16, threads=t)
        assert o.dtype == torch.bfloat16
        assert torch.equal(o.view(torch.int16), o_ref.bfloat16().view(torch.int16)) and torch.equal(ml, ml_ref)
    empty = (n == 0).repeat_interleave(G)
    assert empty.any() and torch.all(o_ref[empty] == 0) and torch.all(ml_ref[empty, 0] == -math.inf)
