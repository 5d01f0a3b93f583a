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
