"""The C++ decode-step engine (K1 stream + one persistent multi-layer K2 +
flag-gated recalls) against per-layer calls of the validated ops, and its
host-buffer path against its device path."""
import math

import numpy as np
import pytest
import torch

from helpers import D, make_digests
from paper_2603_27138_b200 import ops
from paper_2603_27138_b200.engine import DecodeEngine, LayerState

pytestmark = pytest.mark.gpu


def build(rng, L=4, batch=3, hkv=2, G=4, nb=40, k=8, cap=12, recall=True, q_dtype=torch.float32,
          cpu_dtype=torch.float32, gpu_side="predicted_topk_intersect_resident"):
    dev = torch.device("cuda")
    U = batch * hkv
    nbs = ((nb + 7) // 8) * 8
    n_slots = L * U * (cap + k)
    pool = ops.alloc_pool(n_slots, torch.bfloat16)
    pool.view(torch.bfloat16).normal_()
    n_tokens = torch.tensor(rng.integers(64 * (nb - 1) + 1, 64 * nb + 1, size=U), dtype=torch.int32, device=dev)
    host_blocks = 64
    sb = ops.slot_bytes(torch.bfloat16)
    host = torch.randint(0, 256, (host_blocks * sb,), dtype=torch.uint8).pin_memory()
    host.view(torch.bfloat16).copy_(torch.randn(host_blocks * sb // 2).bfloat16())
    layers = []
    for li in range(L):
        dig = torch.from_numpy(make_digests(rng, U, nbs)).to(dev).to(torch.bfloat16).contiguous()
        table = np.full((U, nbs), -1, np.int32)
        dst = []
        for u in range(U):
            ids = rng.choice(nb, size=cap, replace=False)
            table[u, ids] = li * U * (cap + k) + u * (cap + k) + np.arange(cap)
            table[u, nb - 1] = li * U * (cap + k) + u * (cap + k) + cap  # open block always resident
            dst += list(li * U * (cap + k) + u * (cap + k) + cap + 1 + np.arange(3))
        src = torch.tensor(rng.integers(0, host_blocks, size=len(dst)), dtype=torch.int64)
        layers.append(LayerState(dig, torch.from_numpy(table).to(dev),
                                 src if recall else None, torch.tensor(dst, dtype=torch.int32) if recall else None))
    eng = DecodeEngine(layers=L, batch=batch, hq=hkv * G, hkv=hkv, k=k, n_tokens=n_tokens, pool=pool,
                       kv_dtype=torch.bfloat16, layer_states=layers, scale=1 / math.sqrt(D),
                       recall_interval=2 if recall else 0, host_tier=host if recall else None, host_staging=True,
                       chunk_layers=2, q_dtype=q_dtype, cpu_dtype=cpu_dtype, gpu_side_policy=gpu_side)
    q_true = torch.randn(L, U * G, D, device=dev).to(q_dtype)
    q_pred = torch.randn(L, U * G, D, device=dev).to(q_dtype)
    cpu_o = torch.randn(L, U * G, D, device=dev).to(cpu_dtype)
    cpu_ml = torch.stack([torch.randn(L, U * G, device=dev), torch.rand(L, U * G, device=dev) * 5 + 0.5], -1).contiguous()
    return dict(eng=eng, pool=pool, layers=layers, n_tokens=n_tokens, q_true=q_true, q_pred=q_pred, cpu_o=cpu_o,
                cpu_ml=cpu_ml, L=L, U=U, G=G, k=k, host=host, sb=sb)


def reference_step(c):
    """Per-layer K1 + single-layer K2 through the (oracle-validated) ops."""
    outs = []
    for li in range(c["L"]):
        q_sel = c["q_true"][0] if li == 0 else c["q_pred"][li]
        st = c["layers"][li]
        r = ops.score_topk_split(q_sel, st.digests, c["n_tokens"], c["k"], c["G"], block_table=st.table,
                                 k_stride=c["k"])
        o, ml = ops.sparse_decode(c["q_true"][li], c["pool"], torch.bfloat16, r["res_slots"], r["res_ids"],
                                  r["n_res"], c["n_tokens"], c["G"], cpu_o=c["cpu_o"][li].float(), cpu_ml=c["cpu_ml"][li])
        outs.append((o, ml))
    return outs


@pytest.mark.parametrize("cpu_dtype", [torch.float32, torch.bfloat16])
@pytest.mark.parametrize("q_dtype", [torch.float32, torch.bfloat16])
def test_engine_device_step_matches_per_layer_ops(cuda, q_dtype, cpu_dtype):
    """cpu_dtype bf16: the CPU partial's o arrives as bf16 (K2 widens it exactly);
    the per-layer reference gets the same values in f32."""
    c = build(np.random.default_rng(11), recall=False, q_dtype=q_dtype, cpu_dtype=cpu_dtype)
    want = reference_step(c)
    out_o = torch.empty(c["q_true"].shape, device="cuda")
    out_ml = torch.empty(c["L"], c["U"] * c["G"], 2, device="cuda")
    for step in (1, 2, 3):  # several launches: tokens / parities advance
        c["eng"].decode_step(step, c["q_true"], c["q_pred"], c["cpu_o"], c["cpu_ml"], out_o, out_ml)
        torch.cuda.synchronize()
        for li in range(c["L"]):
            assert torch.equal(out_o[li], want[li][0]), (step, li)
            assert torch.equal(out_ml[li], want[li][1]), (step, li)


@pytest.mark.parametrize("cpu_dtype", [torch.float32, torch.bfloat16])
@pytest.mark.parametrize("q_dtype", [torch.float32, torch.bfloat16])
def test_engine_host_path_matches_device_path(cuda, q_dtype, cpu_dtype):
    c = build(np.random.default_rng(12), recall=False, q_dtype=q_dtype, cpu_dtype=cpu_dtype)
    want = reference_step(c)
    pin = lambda t: t.cpu().pin_memory()  # noqa: E731
    h = [pin(c[n]) for n in ("q_true", "q_pred", "cpu_o", "cpu_ml")]
    h_out = torch.empty(c["q_true"].shape, dtype=torch.float32).pin_memory()
    h_ml = torch.empty(c["L"], c["U"] * c["G"], 2).pin_memory()
    h_ids = torch.full((c["L"], c["U"], c["k"]), -1, dtype=torch.int32).pin_memory()
    h_ncpu = torch.full((c["L"], c["U"]), -1, dtype=torch.int32).pin_memory()
    for step in (1, 2):
        c["eng"].decode_step_host(step, *h, h_out, h_ml, h_ids, h_ncpu)
        torch.cuda.synchronize()
        for li in range(c["L"]):
            assert torch.equal(h_out[li], want[li][0].cpu()), (step, li)
            assert torch.equal(h_ml[li], want[li][1].cpu())
    # CPU-side ids / counts delivered for the host worker match K1's
    for li in range(1, c["L"]):
        st = c["layers"][li]
        r = ops.score_topk_split(c["q_pred"][li], st.digests, c["n_tokens"], c["k"], c["G"], block_table=st.table,
                                 k_stride=c["k"])
        ncpu = r["n_cpu"].cpu()
        assert torch.equal(h_ncpu[li], ncpu)
        for u in range(c["U"]):
            assert torch.equal(h_ids[li, u, :ncpu[u]], r["cpu_ids"][u, :ncpu[u]].cpu())


def test_engine_recall_moves_blocks_after_attention(cuda):
    c = build(np.random.default_rng(13), recall=True)
    out_o = torch.empty(c["q_true"].shape, device="cuda")
    out_ml = torch.empty(c["L"], c["U"] * c["G"], 2, device="cuda")
    eng, sb = c["eng"], c["sb"]
    for step in (1, 2, 3, 4):
        eng.decode_step(step, c["q_true"], c["q_pred"], c["cpu_o"], c["cpu_ml"], out_o, out_ml)
    eng.sync()
    torch.cuda.synchronize()
    pool = c["pool"].cpu()
    for li, st in enumerate(c["layers"]):
        for s_, d_ in zip(st.recall_src.tolist(), st.recall_dst.tolist()):
            assert torch.equal(pool[d_ * sb:(d_ + 1) * sb], c["host"][s_ * sb:(s_ + 1) * sb]), (li, d_)


def test_engine_static_all_resident_matches_per_layer_ops(cuda):
    """GpuSidePolicy::all_resident (engine.hpp:28-29, 253-256) in the static
    view: each layer's GPU side is its whole block table (every resident
    block, ascending ids), merged with the CPU partial, on the device path and
    the host-buffer path."""
    c = build(np.random.default_rng(12), recall=False, gpu_side="all_resident")
    want = []
    for li in range(c["L"]):
        table = c["layers"][li].table.cpu().numpy()
        nt = c["n_tokens"].cpu().numpy()
        U, nbs = table.shape
        ids = np.zeros((U, nbs), np.int32)
        slots = np.zeros((U, nbs), np.int32)
        n = np.zeros(U, np.int32)
        for u in range(U):
            f = np.nonzero(table[u, :(int(nt[u]) + 63) // 64] >= 0)[0]
            ids[u, :len(f)], slots[u, :len(f)], n[u] = f, table[u, f], len(f)
        to = lambda a: torch.as_tensor(a, device="cuda")  # noqa: E731
        want.append(ops.sparse_decode(c["q_true"][li], c["pool"], torch.bfloat16, to(slots), to(ids), to(n),
                                      c["n_tokens"], c["G"], cpu_o=c["cpu_o"][li], cpu_ml=c["cpu_ml"][li]))
    out_o = torch.empty(c["q_true"].shape, device="cuda")
    out_ml = torch.empty(c["L"], c["U"] * c["G"], 2, device="cuda")
    for step in (1, 2):
        c["eng"].decode_step(step, c["q_true"], c["q_pred"], c["cpu_o"], c["cpu_ml"], out_o, out_ml)
        torch.cuda.synchronize()
        for li in range(c["L"]):
            assert torch.equal(out_o[li], want[li][0]) and torch.equal(out_ml[li], want[li][1]), (step, li)
    h = lambda t: t.cpu().pin_memory()  # noqa: E731
    h_o = torch.empty(out_o.shape).pin_memory()
    h_ml = torch.empty(out_ml.shape).pin_memory()
    c["eng"].decode_step_host(3, h(c["q_true"]), h(c["q_pred"]), h(c["cpu_o"]), h(c["cpu_ml"]), h_o, h_ml)
    c["eng"].sync()
    torch.cuda.synchronize()
    for li in range(c["L"]):
        assert torch.equal(h_o[li], want[li][0].cpu()), li


@pytest.mark.gpu
@pytest.mark.parametrize("host", [False, True])
def test_engine_static_overlapped_step_matches_ordinary(cuda, host):
    """The static view's overlapped step (K1 beside K2, K2 polling K1's
    per-layer flags; only without recall plans) against the ordinary order on
    an identical engine: outputs and CPU-side ids bit for bit, on the device
    path and the host-buffer path; the overlapped side really overlapped."""
    cs = []
    for _ in range(2):  # identical inputs: the same numpy and torch streams
        torch.manual_seed(33)
        cs.append(build(np.random.default_rng(33), L=6, batch=4, recall=False, q_dtype=torch.bfloat16,
                        cpu_dtype=torch.bfloat16))
    cs[0]["eng"].set_overlap(40)
    cs[1]["eng"].set_overlap(0)
    outs = []
    for c in cs:
        if host:
            h = lambda t: t.cpu().pin_memory()  # noqa: E731
            o = [torch.empty(c["q_true"].shape).pin_memory(), torch.empty(c["L"], c["U"] * c["G"], 2).pin_memory(),
                 torch.empty(c["L"], c["U"], c["k"], dtype=torch.int32).pin_memory(),
                 torch.empty(c["L"], c["U"], dtype=torch.int32).pin_memory()]
            res = []
            for step in range(1, 6):
                c["eng"].decode_step_host(step, h(c["q_true"]), h(c["q_pred"]), h(c["cpu_o"]), h(c["cpu_ml"]), *o)
                c["eng"].sync()
                torch.cuda.synchronize()
                res.append([t.clone() for t in o])
        else:
            o = [torch.empty(c["q_true"].shape, device="cuda"), torch.empty(c["L"], c["U"] * c["G"], 2, device="cuda")]
            res = []
            for step in range(1, 6):
                c["eng"].decode_step(step, c["q_true"], c["q_pred"], c["cpu_o"], c["cpu_ml"], *o)
                torch.cuda.synchronize()
                res.append([t.clone() for t in o])
        outs.append(res)
    for step, (a, b) in enumerate(zip(*outs)):
        assert torch.equal(a[0], b[0]) and torch.equal(a[1], b[1]), step
        if host:
            assert torch.equal(a[3], b[3]), step
            for li in range(cs[0]["L"]):
                for u in range(cs[0]["U"]):
                    n = int(a[3][li, u])
                    assert torch.equal(a[2][li, u, :n], b[2][li, u, :n]), (step, li, u)
    n_ov, sms = cs[0]["eng"].overlap_stats()
    assert sms == 40 and n_ov == 4  # every step after the first
    assert cs[1]["eng"].overlap_stats()[0] == 0
    want = reference_step(cs[1])
    for li in range(cs[0]["L"]):  # and the ordinary side is the per-layer ops' result
        assert torch.equal(outs[1][-1][0][li].to(want[li][0].device), want[li][0]), li
