"""K0 (slot writes, digest build), K3 (standalone merge), K4 (recall gather)."""
import numpy as np
import pytest
import torch

import py_oracle as P
from helpers import D, from_bf16, load_golden
from paper_2603_27138_b200 import ops

pytestmark = pytest.mark.gpu


@pytest.mark.parametrize("dtype", [torch.bfloat16, torch.float32])
def test_kv_write_read_roundtrip(cuda, dtype):
    rng = np.random.default_rng(1)
    pool = ops.alloc_pool(5, dtype)
    n = 300
    slots = rng.integers(0, 5, size=n)
    rows = rng.integers(0, 64, size=n)
    # unique (slot, row) pairs
    key = np.unique(slots * 64 + rows)
    slots, rows = key // 64, key % 64
    k = torch.randn(len(key), D)
    v = torch.randn(len(key), D)
    ops.kv_write_tokens(pool, dtype, slots, rows, k, v)
    k2, v2 = ops.kv_read_tokens(pool, dtype, slots, rows)
    kr = k.to(dtype).float() if dtype == torch.bfloat16 else k
    vr = v.to(dtype).float() if dtype == torch.bfloat16 else v
    assert torch.equal(k2.cpu(), kr) and torch.equal(v2.cpu(), vr)


@pytest.mark.parametrize("case", sorted(load_golden("digest")))
def test_digest_build_vs_reference_golden(cuda, case):
    g = load_golden("digest")[case]
    k = from_bf16(g["k"])
    rows = k.shape[0]
    pool = ops.alloc_pool(2, torch.bfloat16)
    kp = np.zeros((64, D), np.float32)
    kp[:rows] = k
    ops.write_blocks(pool, torch.bfloat16, [1], torch.from_numpy(kp)[None], torch.from_numpy(kp)[None])
    nbs = 8
    dig = torch.zeros(3, 2, D, nbs, dtype=torch.bfloat16, device="cuda")
    ops.digest_build(pool, torch.bfloat16, 0, [1], [rows], [2], [5], dig, nbs)
    mean = torch.zeros(3, D, nbs, dtype=torch.float64, device="cuda")
    ops.digest_build(pool, torch.bfloat16, 1, [1], [rows], [1], [3], mean, nbs)
    dig = dig.float().double().cpu().numpy()
    assert np.array_equal(dig[2, 0, :, 5], g["lo"]) and np.array_equal(dig[2, 1, :, 5], g["hi"])
    assert np.array_equal(mean.cpu().numpy()[1, :, 3], g["mean"])


def test_merge_partials_vs_oracle(cuda):
    rng = np.random.default_rng(4)
    n = 64
    ao, bo = rng.standard_normal((n, D)).astype(np.float32), rng.standard_normal((n, D)).astype(np.float32)
    aml = np.stack([rng.standard_normal(n) * 3, rng.random(n) * 10 + 0.1], 1).astype(np.float32)
    bml = np.stack([rng.standard_normal(n) * 3, rng.random(n) * 10 + 0.1], 1).astype(np.float32)
    aml[0], bml[1], aml[2], bml[2] = (-np.inf, 0), (-np.inf, 0), (-np.inf, 0), (-np.inf, 0)
    t = lambda x: torch.as_tensor(x, device="cuda")  # noqa: E731
    o, ml = ops.merge_partials(t(ao), t(aml), t(bo), t(bml))
    o, ml = o.cpu().numpy(), ml.cpu().numpy()
    for i in range(n):
        pa = P.Partial(ao[i] * aml[i, 1], float(aml[i, 0]), float(aml[i, 1]), int(aml[i, 1] > 0))
        pb = P.Partial(bo[i] * bml[i, 1], float(bml[i, 0]), float(bml[i, 1]), int(bml[i, 1] > 0))
        m = P.merge(pa, pb)
        if m.count == 0:
            assert np.all(o[i] == 0) and ml[i, 1] == 0
            continue
        if pa.count == 0 or pb.count == 0:  # exact identity
            src = bo[i] if pa.count == 0 else ao[i]
            assert np.array_equal(o[i], src)
        np.testing.assert_allclose(o[i], P.finalize(m), rtol=1e-5, atol=1e-5)


@pytest.mark.parametrize("dtype", [torch.bfloat16, torch.float32])
def test_recall_gather_copies_block_images(cuda, dtype):
    sb = ops.slot_bytes(dtype)
    host = torch.randint(0, 256, (9 * sb,), dtype=torch.uint8).pin_memory()
    pool = torch.zeros(6 * sb, dtype=torch.uint8, device="cuda")
    ops.recall_gather(pool, dtype, host, [8, 0, 3], [5, 1, 2])
    torch.cuda.synchronize()
    p = pool.cpu()
    for s, d in ((8, 5), (0, 1), (3, 2)):
        assert torch.equal(p[d * sb:(d + 1) * sb], host[s * sb:(s + 1) * sb])
    assert torch.count_nonzero(p[:sb]) == 0


@pytest.mark.parametrize("dtype", [torch.bfloat16, torch.float32])
def test_recall_copy_engine_path(cuda, dtype):
    sb = ops.slot_bytes(dtype)
    host = torch.randint(0, 256, (9 * sb,), dtype=torch.uint8).pin_memory()
    pool = torch.zeros(6 * sb, dtype=torch.uint8, device="cuda")
    s = torch.cuda.Stream()
    with torch.cuda.stream(s):
        ops.recall_copy(pool, dtype, host, [8, 0, 3], [5, 1, 2])
    s.synchronize()
    p = pool.cpu()
    for src, d in ((8, 5), (0, 1), (3, 2)):
        assert torch.equal(p[d * sb:(d + 1) * sb], host[src * sb:(src + 1) * sb])
    assert torch.count_nonzero(p[:sb]) == 0


@pytest.mark.parametrize("dtype", [torch.bfloat16, torch.float32])
@pytest.mark.parametrize("method", [0, 1])
def test_kv_append_incremental_digest(cuda, dtype, method):
    """append_token (kv_store.hpp:90-117) on the GPU: after every append the
    open block's digest equals build_digest over its rows (digest.hpp:34-60),
    bit for bit, sealed blocks keep theirs, and the rows read back exactly."""
    rng = np.random.default_rng(17 + method)
    dev = torch.device("cuda")
    U, nbs, steps = 5, 8, 140
    start = np.array([0, 63, 64, 130, 7], np.int32)
    n_slots = U * nbs
    pool = ops.alloc_pool(n_slots, dtype)
    ddt = torch.float64 if method == 1 else dtype
    digests = torch.zeros((U, 1 if method == 1 else 2, D, nbs), dtype=ddt, device=dev)
    rows_k = [[] for _ in range(U)]  # per unit, per block: list of K rows (kv-dtype rounded, f64)
    rows_v = [[] for _ in range(U)]
    slot_of = np.full((U, nbs), -1, np.int64)
    free = list(range(n_slots))[::-1]
    rnd = (lambda x: torch.from_numpy(x).to(dtype).double().numpy()) if dtype == torch.bfloat16 else \
        (lambda x: x.astype(np.float64))
    # prefill: the open block state before the first decode append
    n_tok = torch.zeros(U, dtype=torch.int32, device=dev)
    for u in range(U):
        for t in range(start[u]):
            b = t // 64
            if t % 64 == 0:
                slot_of[u, b] = free.pop()
                rows_k[u].append([]), rows_v[u].append([])
            kr, vr = rng.standard_normal(D).astype(np.float32), rng.standard_normal(D).astype(np.float32)
            rows_k[u][b].append(rnd(kr)), rows_v[u][b].append(rnd(vr))
            ops.kv_write_tokens(pool, dtype, [slot_of[u, b]], [t % 64], torch.from_numpy(kr)[None],
                                torch.from_numpy(vr)[None])
        for b in range(len(rows_k[u])):
            ops.digest_build(pool, dtype, method, [slot_of[u, b]], [len(rows_k[u][b])], [u], [b], digests, nbs)
    n_tok.copy_(torch.from_numpy(start))
    for _ in range(steps):
        pos = n_tok.cpu().numpy()
        open_slot = np.zeros(U, np.int32)
        for u in range(U):
            b = pos[u] // 64
            if pos[u] % 64 == 0:
                slot_of[u, b] = free.pop()
                rows_k[u].append([]), rows_v[u].append([])
            open_slot[u] = slot_of[u, b]
        kr = rng.standard_normal((U, D)).astype(np.float32)
        vr = rng.standard_normal((U, D)).astype(np.float32)
        ops.kv_append(pool, dtype, method, open_slot, n_tok, torch.from_numpy(kr), torch.from_numpy(vr), digests, nbs)
        dg = digests.double().cpu().numpy()
        for u in range(U):
            b = pos[u] // 64
            rows_k[u][b].append(rnd(kr[u])), rows_v[u][b].append(rnd(vr[u]))
            want = P.build_digest(np.array(rows_k[u][b]), method)
            if method == 0:
                assert np.array_equal(dg[u, 0, :, b].view(np.uint64), want[0].view(np.uint64))
                assert np.array_equal(dg[u, 1, :, b].view(np.uint64), want[1].view(np.uint64))
            else:
                assert np.array_equal(dg[u, 0, :, b].view(np.uint64), want.view(np.uint64))
    assert np.array_equal(n_tok.cpu().numpy(), start + steps)
    # every block (sealed and open) digest and rows intact at the end
    dg = digests.double().cpu().numpy()
    for u in range(U):
        for b in range(len(rows_k[u])):
            want = P.build_digest(np.array(rows_k[u][b]), method)
            got = dg[u, 0, :, b] if method == 1 else np.stack([dg[u, 0, :, b], dg[u, 1, :, b]])
            assert np.array_equal(np.asarray(got).view(np.uint64), np.asarray(want).view(np.uint64))
            n = len(rows_k[u][b])
            k2, v2 = ops.kv_read_tokens(pool, dtype, [slot_of[u, b]] * n, list(range(n)))
            assert np.array_equal(k2.cpu().double().numpy(), np.array(rows_k[u][b]))
            assert np.array_equal(v2.cpu().double().numpy(), np.array(rows_v[u][b]))
