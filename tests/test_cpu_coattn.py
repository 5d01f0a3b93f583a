"""CPU co-attention worker (scout_cpu_partial_attention, host only) against the
oracle's partial_attention (attention.hpp:73-95) on the same bf16 / f32 block
images: the host tier's swizzled bf16 tile layout is decoded correctly, ragged
rows are masked, empty units give (0, -inf, 0). fp32 vs double: 1e-4."""
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


@pytest.mark.parametrize("kv", ["bf16", "f32"])
@pytest.mark.parametrize("G", [1, 4, 8])
def test_cpu_partial_attention_vs_oracle(kv, G):
    rng = np.random.default_rng(G + (kv == "f32") * 10)
    U, nblk, k = 5, 12, 6
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
    n = np.array([k, 3, 0, 1, k], np.int32)
    for u in range(U):
        idx[u, :n[u]] = rng.choice(nblk, size=n[u], replace=False)
        if n[u]:
            rows[u, n[u] - 1] = int(rng.integers(1, B + 1))  # an open (ragged) block
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
            assert np.abs(o[h] - want).max() <= 1e-4 * max(1.0, np.abs(want).max()), (u, g)
            lse = ml[h, 0] + math.log(ml[h, 1])
            assert abs(lse - (p.max_logit + math.log(p.denom))) <= 1e-4, (u, g)
