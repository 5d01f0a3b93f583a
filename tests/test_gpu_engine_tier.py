"""Device tier mode of the C++ engine (scout_engine_decode_step_kv): a whole
decode step on the device in the order of ScoutEngine::decode_step
(engine.hpp:220-307): planning view, select + mark, begin_layer's ticket
application, attention + merge, append (open / seal / LRU eviction,
write-through), periodic recall of the CPU-side selected blocks. Compared,
step after step, with a replay of the reference's per-layer order through the
validated single ops and the DeviceTieredCache mirror (itself bit-exact
against the reference TieredKvCache, test_gpu_tier.py)."""
import ctypes as C
import math

import numpy as np
import pytest
import torch

from paper_2603_27138_b200 import _capi as A
from paper_2603_27138_b200 import ops
from paper_2603_27138_b200.engine import DecodeEngine, LayerState
from paper_2603_27138_b200.tier import DeviceTieredCache

pytestmark = pytest.mark.gpu
D, BS = 128, 64


class Side:
    """One side of the comparison: its own pool, digests, host tier and tier state."""

    def __init__(self, L, U, nbs, cap, kv, seed_rows, victim_cache=True):
        dev = torch.device("cuda")
        self.tier = DeviceTieredCache(L, U, nbs, capacity=cap, slots_per_unit=nbs, victim_cache=victim_cache)
        self.tier.pin_layer(0)
        self.pool = ops.alloc_pool(L * U * nbs, kv)
        self.dig = [torch.zeros(U, 2, D, nbs, dtype=kv, device=dev) for _ in range(L)]
        self.host = torch.zeros(L * U * nbs * ops.slot_bytes(kv), dtype=torch.uint8).pin_memory()
        self.n_tokens = torch.zeros(U, dtype=torch.int32, device=dev)
        self.kv = kv
        for layer in range(L):  # prefill: appends that seal (and evict: capacity holds during prefill)
            for k_rows, v_rows in seed_rows[layer]:
                self.tier.append_token(layer, k_rows, v_rows, self.pool, kv, self.dig[layer], host_tier=self.host)
        self.n_tokens.copy_(self.tier.n_tokens[0])


POLICIES = {
    # name: (recall intervals per layer or None, capacity, stagger, external re-placement)
    "reference_every_3": ([3, 3, 3], 8, False, False),
    # capacity == k with stationary queries: the fast set converges to the
    # predicted set, so the seal at step 64 (whose open block, filled with
    # small keys, is never predicted) evicts a block the step just predicted
    # (LRU ties -> lower id), and the reference recalls it right away
    # (predicted \ residency after the append)
    "reference_per_layer_full_capacity": ([1, 2, 1], 6, False, False),
    "no_recall": (None, 8, False, False),
    "no_recall_external_place": (None, 8, False, True),
    "stagger_opt_in": ([3, 3, 3], 8, True, False),
    # GpuSidePolicy::all_resident (engine.hpp:28-29, 253-256): the GPU side
    # attends to the layer's whole fast tier after begin_layer's tickets
    "all_resident_every_3": ([3, 3, 3], 8, False, False),
    "all_resident_no_recall": (None, 8, False, False),
}
ALL_RESIDENT = {"all_resident_every_3", "all_resident_no_recall"}


def fast_tier_lists(rt, i, n_tokens, nbs):
    """residency_set(i) at attention time (the fast tier, ascending ids) with each
    block's pool slot, as [U][nbs] lists for ops.sparse_decode."""
    tier, table = rt.tier[i].cpu().numpy(), rt.table[i].cpu().numpy()
    U = tier.shape[0]
    ids = np.zeros((U, nbs), np.int32)
    slots = np.zeros((U, nbs), np.int32)
    n = np.zeros(U, np.int32)
    for u in range(U):
        nb = (int(n_tokens[u]) + BS - 1) // BS
        f = np.nonzero(tier[u, :nb])[0]
        ids[u, :len(f)] = f
        slots[u, :len(f)] = table[u, f]
        n[u] = len(f)
    to = lambda a: torch.as_tensor(a, device="cuda")  # noqa: E731
    return to(slots), to(ids), to(n)


@pytest.mark.parametrize("policy,kv", [(p, torch.bfloat16) for p in sorted(POLICIES)] +
                         [(p, torch.float32) for p in ("reference_every_3", "all_resident_every_3",
                                                       "reference_per_layer_full_capacity")])
def test_engine_tier_mode_matches_reference_order_replay(cuda, policy, kv):
    """The engine's decode steps against a replay in the reference's per-layer
    order (engine.hpp:219-307) through the validated single ops and the
    DeviceTieredCache mirror, with the recall decision and the recalled set
    coming from the reference itself: maybe_schedule_recall (recall.hpp:114-126)
    through oracle/_ref on (predicted, residency_set after the append).
    external: between two steps the caller re-places layer 1's fast set
    (place_after_prefill) on both sides and tells the engine
    (scout_engine_tier_changed), whose next planning view must then come from
    the new state, not from the view the previous step's post launch wrote.
    kv f32: the engine's f32 KV path (per-layer CUDA-core attention launches
    gated by stream operations, f32 queries and partials)."""
    import py_oracle as P

    intervals, cap, stagger, external = POLICIES[policy]
    rng = np.random.default_rng(21 + len(policy))
    torch.manual_seed(len(policy))
    L, batch, hkv, G, k, nbs, steps = 3, 2, 2, 4, 6, 24, 70
    U = batch * hkv
    qdt = torch.bfloat16 if kv == torch.bfloat16 else torch.float32
    stationary = policy == "reference_per_layer_full_capacity"
    T0 = 64 * 13 if stationary else 64 * 12 + 40
    seed_rows = [[(torch.randn(U, D), torch.randn(U, D)) for _ in range(T0)] for _ in range(L)]
    eng_side, rep = Side(L, U, nbs, cap, kv, seed_rows), Side(L, U, nbs, cap, kv, seed_rows)
    layers = [LayerState(eng_side.dig[i], torch.full((U, nbs), -1, dtype=torch.int32, device="cuda"))
              for i in range(L)]
    eng = DecodeEngine(layers=L, batch=batch, hq=hkv * G, hkv=hkv, k=k, n_tokens=eng_side.n_tokens,
                       pool=eng_side.pool, kv_dtype=kv, layer_states=layers, scale=1 / math.sqrt(D),
                       recall_interval=0, recall_intervals=intervals, recall_stagger=stagger,
                       host_tier=eng_side.host, tier=eng_side.tier, host_blocks=0, q_dtype=qdt,
                       gpu_side_policy="all_resident" if policy in ALL_RESIDENT else
                       "predicted_topk_intersect_resident")
    policy_ref = P.RefRecall(U, intervals) if (intervals and not stagger) else None
    out_o = torch.empty(L, U * G, D, device="cuda")
    out_ml = torch.empty(L, U * G, 2, device="cuda")
    st = torch.cuda.current_stream().cuda_stream
    rt = rep.tier
    n_recalled = evicted_predicted = 0
    q_fixed = torch.randn(L, U * G, D, device="cuda")
    for step in range(1, steps + 1):
        q_true = (q_fixed if stationary else torch.randn(L, U * G, D, device="cuda")).to(qdt)
        q_pred = q_true if stationary else (q_true.float() + 0.3 * torch.randn(L, U * G, D, device="cuda")).to(qdt)
        cpu_o = torch.randn(L, U * G, D, device="cuda")
        cpu_ml = torch.stack([torch.randn(L, U * G, device="cuda"), torch.rand(L, U * G, device="cuda") + 0.1], -1).contiguous()
        k_new = torch.randn(L, U, D, device="cuda") * (0.05 if stationary else 1.0)
        v_new = torch.randn(L, U, D, device="cuda")
        eng.decode_step_kv(step, q_true, q_pred, cpu_o, cpu_ml, k_new, v_new, out_o, out_ml)
        # ---- replay in the reference's per-layer order
        sel = [None] * L
        want = []
        for i in range(L):
            rt.begin_layer(step, i)
            targets = ([0] if i == 0 else []) + ([i + 1] if i + 1 < L else [])
            for t in targets:
                q = q_true[0] if t == 0 else q_pred[t]
                sel[t] = ops.score_topk_split(q, rep.dig[t], rep.n_tokens, k, G, block_table=rt.residency_table(t),
                                              step=step, last_selected=rt.last_sel[t], k_stride=k)
            r = sel[i]
            if policy in ALL_RESIDENT:  # engine.hpp:253-256: gpu_ids = residency_set(i)
                torch.cuda.synchronize()
                a_slots, a_ids, a_n = fast_tier_lists(rt, i, rep.n_tokens.cpu().numpy(), nbs)
                o, ml = ops.sparse_decode(q_true[i], rep.pool, kv, a_slots, a_ids, a_n, rep.n_tokens, G,
                                          cpu_o=cpu_o[i], cpu_ml=cpu_ml[i])
            else:
                o, ml = ops.sparse_decode(q_true[i], rep.pool, kv, r["res_slots"], r["res_ids"], r["n_res"],
                                          rep.n_tokens, G, cpu_o=cpu_o[i], cpu_ml=cpu_ml[i])
            want.append((o, ml))
            rt.append_token(i, k_new[i], v_new[i], rep.pool, kv, rep.dig[i], host_tier=rep.host)
            if not intervals:
                continue
            # engine.hpp:299-307: maybe_schedule_recall(predicted[i], residency_set(i)) after the append
            residency = (rt.residency_table(i) >= 0).cpu().numpy()
            pred = [r["sel_ids"][u, :int(r["n_sel"][u])].cpu().numpy() for u in range(U)]
            res_before = [set(r["res_ids"][u, :int(r["n_res"][u])].cpu().tolist()) for u in range(U)]
            ids = torch.zeros(U, k, dtype=torch.int32)
            n_ids = torch.zeros(U, dtype=torch.int32)
            for u in range(U):
                res_u = np.nonzero(residency[u])[0]
                if stagger:
                    got = np.setdiff1d(pred[u], res_u) if (step + i) % intervals[i] == 0 else None
                else:
                    got = policy_ref.maybe_schedule_recall(u, i, step, pred[u], res_u)
                if got is None or len(got) == 0:
                    continue
                ids[u, :len(got)] = torch.from_numpy(np.asarray(got, np.int32))
                n_ids[u] = len(got)
                n_recalled += len(got)
                evicted_predicted += len(set(int(x) for x in got) & res_before[u])
            if int(n_ids.sum()) == 0:
                continue
            ids_d, n_d = ids.cuda(), n_ids.cuda()
            dst = rt.schedule_recall(i, ids_d, n_d, step, i)
            A.check(A.lib().scout_recall_gather_ids(rep.pool.data_ptr(), ops.dtype_code(kv), rep.host.data_ptr(),
                                                    i * U * nbs, nbs, 0, U, ids_d.data_ptr(), n_d.data_ptr(),
                                                    dst.data_ptr(), k, 1, st))
            rt.check(i)
        rep.n_tokens.copy_(rt.n_tokens[0])
        eng.sync()
        torch.cuda.synchronize()
        for i in range(L):
            assert torch.equal(out_o[i], want[i][0]), (step, i)
            assert torch.equal(out_ml[i], want[i][1]), (step, i)
        assert torch.equal(eng_side.n_tokens, rep.n_tokens)
        for name in ("tier", "last_sel"):
            assert torch.equal(getattr(eng_side.tier, name), getattr(rt, name)), (step, name)
        assert torch.equal(eng_side.tier.ready >= 0, rt.ready >= 0), step
        assert int(eng_side.tier.err.abs().sum()) == 0
        if external and step == steps // 2:
            qx = torch.randn(U * G, D, device="cuda")
            for i in range(L):  # the engine advanced its own token counts, not the mirror's
                eng_side.tier.n_tokens[i].copy_(eng_side.n_tokens)
            for side in (eng_side, rep):
                side.tier.place_after_prefill(1, qx, side.dig[1], G, kv)
            torch.cuda.synchronize()
            assert torch.equal(eng_side.tier.tier, rt.tier)
            eng.tier_changed()
    # the run crossed seals (evictions) and, with recall, flipped tiers back
    assert int(eng_side.n_tokens[0]) == T0 + steps
    nb = (T0 + steps + BS - 1) // BS
    assert int((eng_side.tier.tier[1:, :, :nb - 1] == 0).sum()) > 0  # sealed blocks on the slow tier
    assert (rt.n_tickets > 0) == bool(intervals)
    assert (n_recalled > 0) == bool(intervals)
    if policy == "reference_per_layer_full_capacity":
        assert evicted_predicted > 0  # a seal evicted a just-predicted block and it was recalled
    # digests (incrementally maintained) equal on both sides and the pools hold the same live blocks
    for i in range(L):
        assert torch.equal(eng_side.dig[i], rep.dig[i])


@pytest.mark.parametrize("cpu_dtype,kv", [(torch.float32, torch.bfloat16), (torch.bfloat16, torch.bfloat16),
                                          (torch.float32, torch.float32)])
def test_engine_tier_host_path_matches_device_path(cuda, cpu_dtype, kv):
    """scout_engine_decode_step_kv_host (pinned host inputs and outputs,
    pipelined copies) against scout_engine_decode_step_kv on an identical
    second cache: same outputs, same tier state, step after step (CPU
    partials in f32 and in bf16, the bench's setting)."""
    rng = np.random.default_rng(5)
    L, batch, hkv, G, k, cap, nbs, steps = 3, 2, 2, 4, 6, 8, 24, 40
    U = batch * hkv
    qdt = torch.bfloat16 if kv == torch.bfloat16 else torch.float32
    T0 = 64 * 11 + 50
    seed_rows = [[(torch.randn(U, D), torch.randn(U, D)) for _ in range(T0)] for _ in range(L)]
    sides = [Side(L, U, nbs, cap, kv, seed_rows) for _ in range(2)]
    engs = []
    for sd in sides:
        layers = [LayerState(sd.dig[i], torch.full((U, nbs), -1, dtype=torch.int32, device="cuda")) for i in range(L)]
        engs.append(DecodeEngine(layers=L, batch=batch, hq=hkv * G, hkv=hkv, k=k, n_tokens=sd.n_tokens, pool=sd.pool,
                                 kv_dtype=kv, layer_states=layers, scale=1 / math.sqrt(D), recall_interval=4,
                                 host_tier=sd.host, tier=sd.tier, q_dtype=qdt, host_staging=True,
                                 chunk_layers=2, cpu_dtype=cpu_dtype))
    out = [torch.empty(L, U * G, D, device="cuda"), torch.empty(L, U * G, 2, device="cuda")]
    h_out = [torch.empty(L, U * G, D).pin_memory(), torch.empty(L, U * G, 2).pin_memory()]
    for step in range(1, steps + 1):
        ins = [torch.randn(L, U * G, D, device="cuda").to(qdt), torch.randn(L, U * G, D, device="cuda").to(qdt),
               torch.randn(L, U * G, D, device="cuda").to(cpu_dtype),
               torch.stack([torch.randn(L, U * G, device="cuda"), torch.rand(L, U * G, device="cuda") + 0.1], -1).contiguous(),
               torch.randn(L, U, D, device="cuda"), torch.randn(L, U, D, device="cuda")]
        engs[0].decode_step_kv(step, *ins, *out)
        h_ins = [t.cpu().pin_memory() for t in ins]
        engs[1].decode_step_kv_host(step, *h_ins, *h_out)
        for e in engs:
            e.sync()
        torch.cuda.synchronize()
        assert torch.equal(h_out[0], out[0].cpu()) and torch.equal(h_out[1], out[1].cpu()), step
        for name in ("tier", "last_sel", "table"):
            assert torch.equal(getattr(sides[0].tier, name), getattr(sides[1].tier, name)), (step, name)


@pytest.mark.parametrize("policy", ["reference", "stagger"])
def test_engine_victim_cache_matches_copies(cuda, policy):
    """The device victim cache (warm images in free pool slots) against the
    same engine with every recall copied from the host tier: identical
    outputs and tier state step after step (an image in HBM is the block's
    host-tier image: sealed blocks are immutable and written through), with
    most recalled blocks served warm on the victim side."""
    L, batch, hkv, G, k, cap, nbs, steps = 3, 2, 2, 4, 6, 8, 24, 48
    U = batch * hkv
    kv = torch.bfloat16
    T0 = 64 * 11 + 50
    torch.manual_seed(11)
    seed_rows = [[(torch.randn(U, D), torch.randn(U, D)) for _ in range(T0)] for _ in range(L)]
    sides = [Side(L, U, nbs, cap, kv, seed_rows, victim_cache=vc) for vc in (True, False)]
    engs = []
    for sd in sides:
        layers = [LayerState(sd.dig[i], torch.full((U, nbs), -1, dtype=torch.int32, device="cuda")) for i in range(L)]
        engs.append(DecodeEngine(layers=L, batch=batch, hq=hkv * G, hkv=hkv, k=k, n_tokens=sd.n_tokens, pool=sd.pool,
                                 kv_dtype=kv, layer_states=layers, scale=1 / math.sqrt(D), recall_interval=3,
                                 recall_stagger=policy == "stagger", host_tier=sd.host, tier=sd.tier,
                                 q_dtype=torch.bfloat16))
    outs = [[torch.empty(L, U * G, D, device="cuda"), torch.empty(L, U * G, 2, device="cuda")] for _ in range(2)]
    qs = [torch.randn(L, U * G, D, device="cuda").bfloat16() for _ in range(6)]
    for step in range(1, steps + 1):
        co = torch.randn(L, U * G, D, device="cuda")
        cm = torch.stack([torch.randn(L, U * G, device="cuda"), torch.rand(L, U * G, device="cuda") + 0.1], -1).contiguous()
        kn, vn = torch.randn(L, U, D, device="cuda"), torch.randn(L, U, D, device="cuda")
        for e, o in zip(engs, outs):  # queries cycle: blocks leave the fast tier and come back
            e.decode_step_kv(step, qs[step % 6], qs[(step + 1) % 6], co, cm, kn, vn, *o)
        for e in engs:
            e.sync()
        torch.cuda.synchronize()
        assert torch.equal(outs[0][0], outs[1][0]) and torch.equal(outs[0][1], outs[1][1]), step
        for name in ("tier", "last_sel"):
            assert torch.equal(getattr(sides[0].tier, name), getattr(sides[1].tier, name)), (step, name)
        assert torch.equal(sides[0].tier.ready >= 0, sides[1].tier.ready >= 0), step
    warm, copied = engs[0].recall_stats()
    warm_off, copied_off = engs[1].recall_stats()
    assert warm_off == 0 and copied_off == warm + copied > 0
    assert warm > copied  # the victim side moved only a minority of the recalled blocks
    for e in engs:
        e.check_state()


@pytest.mark.parametrize("recall_mode", [1, 0])
def test_engine_tier_back_to_back_steps_with_recalls(cuda, recall_mode):
    """Steps queued back to back (no host sync), a recall every step: the
    recall copies (SM gather, or the copy engines from the issuer thread) must
    never sit behind the next step's work that waits for them (a K2 flag wait
    would trap after 10 s)."""
    L, batch, hkv, G, k, cap, nbs = 4, 2, 2, 4, 6, 8, 32
    U = batch * hkv
    kv = torch.bfloat16
    T0 = 64 * 14 + 3
    seed_rows = [[(torch.randn(U, D), torch.randn(U, D)) for _ in range(T0)] for _ in range(L)]
    sd = Side(L, U, nbs, cap, kv, seed_rows)
    layers = [LayerState(sd.dig[i], torch.full((U, nbs), -1, dtype=torch.int32, device="cuda")) for i in range(L)]
    eng = DecodeEngine(layers=L, batch=batch, hq=hkv * G, hkv=hkv, k=k, n_tokens=sd.n_tokens, pool=sd.pool,
                       kv_dtype=kv, layer_states=layers, scale=1 / math.sqrt(D), recall_interval=1,
                       host_tier=sd.host, tier=sd.tier, q_dtype=torch.bfloat16, recall_mode=recall_mode)
    qs = [torch.randn(L, U * G, D, device="cuda").bfloat16() for _ in range(4)]
    cpu_o = torch.randn(L, U * G, D, device="cuda")
    cpu_ml = torch.stack([torch.randn(L, U * G, device="cuda"), torch.rand(L, U * G, device="cuda") + 0.1], -1).contiguous()
    kn, vn = torch.randn(L, U, D, device="cuda"), torch.randn(L, U, D, device="cuda")
    out_o = torch.empty(L, U * G, D, device="cuda")
    out_ml = torch.empty(L, U * G, 2, device="cuda")
    for step in range(1, 61):  # drifting queries: every step recalls something
        eng.decode_step_kv(step, qs[step % 4], qs[(step + 1) % 4], cpu_o, cpu_ml, kn, vn, out_o, out_ml)
    eng.sync()
    torch.cuda.synchronize()
    assert int(sd.tier.err.abs().sum()) == 0
    assert torch.isfinite(out_o).all()
    assert int(sd.n_tokens[0]) == T0 + 60


@pytest.mark.parametrize("stagger,gpu_side,kv", [(False, "predicted_topk_intersect_resident", torch.bfloat16),
                                                  (True, "predicted_topk_intersect_resident", torch.bfloat16),
                                                  (False, "all_resident", torch.bfloat16),
                                                  (False, "predicted_topk_intersect_resident", torch.float32)])
def test_engine_layerwise_matches_fused_step(cuda, stagger, gpu_side, kv):
    """scout_engine_decode_layer (one call per layer, inputs given layer by
    layer) against scout_engine_decode_step_kv (all layers at once) on an
    identical second cache: the same outputs bit for bit and the same tier
    state after every step, with recalls in both cadences."""
    L, batch, hkv, G, k, cap, nbs, steps = 4, 2, 2, 4, 6, 8, 24, 40
    U = batch * hkv
    qdt = torch.bfloat16 if kv == torch.bfloat16 else torch.float32
    T0 = 64 * 11 + 50
    torch.manual_seed(7)
    seed_rows = [[(torch.randn(U, D), torch.randn(U, D)) for _ in range(T0)] for _ in range(L)]
    sides = [Side(L, U, nbs, cap, kv, seed_rows) for _ in range(2)]
    engs = []
    for sd in sides:
        layers = [LayerState(sd.dig[i], torch.full((U, nbs), -1, dtype=torch.int32, device="cuda")) for i in range(L)]
        engs.append(DecodeEngine(layers=L, batch=batch, hq=hkv * G, hkv=hkv, k=k, n_tokens=sd.n_tokens, pool=sd.pool,
                                 kv_dtype=kv, layer_states=layers, scale=1 / math.sqrt(D), recall_interval=0,
                                 recall_intervals=[2, 3, 2, 1], recall_stagger=stagger, host_tier=sd.host,
                                 tier=sd.tier, q_dtype=qdt, gpu_side_policy=gpu_side))
    out = [torch.empty(L, U * G, D, device="cuda"), torch.empty(L, U * G, 2, device="cuda")]
    lw = [torch.empty(L, U * G, D, device="cuda"), torch.empty(L, U * G, 2, device="cuda")]
    for step in range(1, steps + 1):
        qt = torch.randn(L, U * G, D, device="cuda").to(qdt)
        qp = (qt.float() + 0.3 * torch.randn(L, U * G, D, device="cuda")).to(qdt)
        co = torch.randn(L, U * G, D, device="cuda")
        cm = torch.stack([torch.randn(L, U * G, device="cuda"), torch.rand(L, U * G, device="cuda") + 0.1], -1).contiguous()
        kn, vn = torch.randn(L, U, D, device="cuda"), torch.randn(L, U, D, device="cuda")
        engs[0].decode_step_kv(step, qt, qp, co, cm, kn, vn, *out)
        for i in range(L):
            engs[1].decode_layer(step, i, qt[i], qp[i + 1] if i + 1 < L else None, co[i], cm[i], kn[i], vn[i],
                                 lw[0][i], lw[1][i])
        for e in engs:
            e.sync()
        torch.cuda.synchronize()
        assert torch.equal(out[0], lw[0]) and torch.equal(out[1], lw[1]), step
        for name in ("tier", "last_sel", "table", "ready"):
            assert torch.equal(getattr(sides[0].tier, name), getattr(sides[1].tier, name)), (step, name)
        assert torch.equal(sides[0].n_tokens, sides[1].n_tokens)
    for e in engs:
        e.check_state()
    with pytest.raises(RuntimeError):  # layers out of order
        engs[1].decode_layer(steps + 1, 2, qt[2], qp[3], None, None, kn[2], vn[2], lw[0][2], lw[1][2])


def test_engine_layerwise_with_query_prediction(cuda):
    """scout_engine_decode_layer_x (K6 inside: q_pred of layer i+1 =
    predict_next_query(rms_normalize(x_i), W_Q^{i+1}), engine.hpp:237) against
    scout_engine_decode_layer fed with the same prediction made outside
    (ops.QueryPredictor, the same tcgen05 kernel): bit-identical outputs and
    tier state, step after step."""
    L, batch, hkv, G, k, cap, nbs, steps, hidden = 4, 2, 2, 4, 6, 8, 24, 24, 256
    U = batch * hkv
    kv = torch.bfloat16
    T0 = 64 * 11 + 50
    torch.manual_seed(13)
    seed_rows = [[(torch.randn(U, D), torch.randn(U, D)) for _ in range(T0)] for _ in range(L)]
    sides = [Side(L, U, nbs, cap, kv, seed_rows) for _ in range(2)]
    engs = []
    for sd in sides:
        layers = [LayerState(sd.dig[i], torch.full((U, nbs), -1, dtype=torch.int32, device="cuda")) for i in range(L)]
        engs.append(DecodeEngine(layers=L, batch=batch, hq=hkv * G, hkv=hkv, k=k, n_tokens=sd.n_tokens, pool=sd.pool,
                                 kv_dtype=kv, layer_states=layers, scale=1 / math.sqrt(D), recall_interval=3,
                                 host_tier=sd.host, tier=sd.tier, q_dtype=torch.bfloat16, hidden=hidden))
    # the engine's K6 grid inside decode_layer_x: one CTA per 128-feature tile (at most 68)
    qp_ctas = min(hkv * G * D // 128, 68)
    wqs = [ops.QueryPredictor((torch.randn(hidden, hkv * G * D, device="cuda") / hidden ** 0.5), batch,
                              max_ctas=qp_ctas) for _ in range(L)]
    outs = [[torch.empty(L, U * G, D, device="cuda"), torch.empty(L, U * G, 2, device="cuda")] for _ in range(2)]
    x_base = torch.randn(L, batch, hidden, device="cuda")
    for step in range(1, steps + 1):
        qt = torch.randn(L, U * G, D, device="cuda").bfloat16()
        xs = x_base + 0.1 * torch.randn(L, batch, hidden, device="cuda")
        co = torch.randn(L, U * G, D, device="cuda")
        cm = torch.stack([torch.randn(L, U * G, device="cuda"), torch.rand(L, U * G, device="cuda") + 0.1], -1).contiguous()
        kn, vn = torch.randn(L, U, D, device="cuda"), torch.randn(L, U, D, device="cuda")
        for i in range(L):
            nxt = i + 1 < L
            engs[0].decode_layer_x(step, i, qt[i], xs[i] if nxt else None, wqs[i + 1] if nxt else None, co[i], cm[i],
                                   kn[i], vn[i], outs[0][0][i], outs[0][1][i])
            qp = wqs[i + 1](xs[i], want=("bf16",)).view(U * G, D) if nxt else None
            engs[1].decode_layer(step, i, qt[i], qp, co[i], cm[i], kn[i], vn[i], outs[1][0][i], outs[1][1][i])
        for e in engs:
            e.sync()
        torch.cuda.synchronize()
        assert torch.equal(outs[0][0], outs[1][0]) and torch.equal(outs[0][1], outs[1][1]), step
        for name in ("tier", "last_sel", "ready"):
            assert torch.equal(getattr(sides[0].tier, name), getattr(sides[1].tier, name)), (step, name)
    for e in engs:
        e.check_state()


def test_engine_cpu_tokens_and_calibration(cuda):
    """scout_engine_cpu_tokens: the last step's CPU-side tokens per layer (the
    RatioTrace sample of engine.hpp:283, summed over the units) equal K1's own
    per-unit counts; a recall-free trace of them calibrates per-layer
    intervals (recall.hpp:66-95) that the engine then runs with."""
    from paper_2603_27138_b200.engine import calibrate_intervals

    L, batch, hkv, G, k, cap, nbs = 3, 2, 2, 4, 6, 8, 24
    U = batch * hkv
    kv = torch.bfloat16
    T0 = 64 * 11 + 50
    torch.manual_seed(17)
    seed_rows = [[(torch.randn(U, D), torch.randn(U, D)) for _ in range(T0)] for _ in range(L)]
    sd = Side(L, U, nbs, cap, kv, seed_rows)
    layers = [LayerState(sd.dig[i], torch.full((U, nbs), -1, dtype=torch.int32, device="cuda")) for i in range(L)]
    mk = lambda **kw: DecodeEngine(layers=L, batch=batch, hq=hkv * G, hkv=hkv, k=k, n_tokens=sd.n_tokens,  # noqa: E731
                                   pool=sd.pool, kv_dtype=kv, layer_states=layers, scale=1 / math.sqrt(D),
                                   host_tier=sd.host, tier=sd.tier, q_dtype=torch.bfloat16, **kw)
    eng = mk(recall_interval=0)
    out = [torch.empty(L, U * G, D, device="cuda"), torch.empty(L, U * G, 2, device="cuda")]
    cm = torch.stack([torch.randn(L, U * G, device="cuda"), torch.rand(L, U * G, device="cuda") + 0.1], -1).contiguous()
    co = torch.randn(L, U * G, D, device="cuda")
    cpu_tr, bud_tr = [], []
    for step in range(1, 13):
        qt = torch.randn(L, U * G, D, device="cuda").bfloat16()
        qp = (qt.float() + 0.3 * torch.randn(L, U * G, D, device="cuda")).bfloat16()
        eng.decode_step_kv(step, qt, qp, co, cm, torch.randn(L, U, D, device="cuda"), torch.randn(L, U, D, device="cuda"),
                           *out)
        c, b = eng.cpu_tokens()
        k1 = eng.k1_outputs()
        assert c == k1["cpu_tokens"].sum(1).tolist() and b == [U * k * 64] * L
        cpu_tr.append(c)
        bud_tr.append(b)
    ivals = calibrate_intervals(np.array(cpu_tr).T, np.array(bud_tr).T, 0.12)
    assert len(ivals) == L and all(1 <= x <= 12 for x in ivals)
    eng.close()
    eng = mk(recall_interval=0, recall_intervals=ivals)
    for step in range(13, 25):
        qt = torch.randn(L, U * G, D, device="cuda").bfloat16()
        eng.decode_step_kv(step, qt, qt, co, cm, torch.randn(L, U, D, device="cuda"), torch.randn(L, U, D, device="cuda"),
                           *out)
    eng.sync()
    eng.check_state()


@pytest.mark.parametrize("kv", [torch.bfloat16, torch.float32])
def test_engine_prefill_matches_mirror_prefill_and_place(cuda, kv):
    """scout_engine_prefill (ScoutEngine::prefill + place_after_prefill,
    engine.hpp:192-201) against the same composition through the tier mirror
    (DeviceTieredCache.prefill per layer, place_after_prefill with K1 on the
    unpinned layers, the promoted blocks gathered from the host tier): the
    same tier state, digests, host images and fast-block contents, with ragged
    per-unit prefill lengths; then identical decode steps with recalls."""
    L, batch, hkv, G, k, cap, nbs, steps = 3, 2, 2, 4, 6, 8, 24, 30
    U = batch * hkv
    qdt = torch.bfloat16 if kv == torch.bfloat16 else torch.float32
    T = 64 * 13 + 17
    torch.manual_seed(23)
    n_tok = torch.tensor([T, 64 * 12, 64 * 9 + 63, 64 * 11 + 1], dtype=torch.int32, device="cuda")
    k_rows = torch.randn(L, U, T, D, device="cuda")
    v_rows = torch.randn(L, U, T, D, device="cuda")
    q_place = torch.randn(L, U * G, D, device="cuda").to(qdt)
    dev = torch.device("cuda")
    st = torch.cuda.current_stream().cuda_stream
    sides, engs = [], []
    for _ in range(2):
        tier = DeviceTieredCache(L, U, nbs, capacity=cap, slots_per_unit=nbs)
        tier.pin_layer(0)
        sd = type("S", (), {})()
        sd.tier, sd.pool = tier, ops.alloc_pool(L * U * nbs, kv)
        sd.dig = [torch.zeros(U, 2, D, nbs, dtype=kv, device=dev) for _ in range(L)]
        sd.host = torch.zeros(L * U * nbs * ops.slot_bytes(kv), dtype=torch.uint8).pin_memory()
        sd.n_tokens = torch.zeros(U, dtype=torch.int32, device=dev)
        layers = [LayerState(sd.dig[i], torch.full((U, nbs), -1, dtype=torch.int32, device=dev)) for i in range(L)]
        engs.append(DecodeEngine(layers=L, batch=batch, hq=hkv * G, hkv=hkv, k=k, n_tokens=sd.n_tokens, pool=sd.pool,
                                 kv_dtype=kv, layer_states=layers, scale=1 / math.sqrt(D), recall_interval=3,
                                 host_tier=sd.host, tier=tier, q_dtype=qdt))
        sides.append(sd)
    m = sides[0]  # the mirror composition
    for i in range(L):
        m.tier.prefill(i, k_rows[i], v_rows[i], n_tok, m.pool, kv, m.dig[i], host_tier=m.host)
    for i in range(1, L):
        _, fill = m.tier.place_after_prefill(i, q_place[i], m.dig[i], G, kv)
        r = ops.score_topk_split(q_place[i], m.dig[i], ((m.tier.n_tokens[i] // BS) * BS).contiguous(), cap, G)
        A.check(A.lib().scout_recall_gather_ids(m.pool.data_ptr(), ops.dtype_code(kv), m.host.data_ptr(), i * U * nbs,
                                                nbs, 0, U, r["sel_ids"].data_ptr(), r["n_sel"].data_ptr(),
                                                fill.data_ptr(), cap, 0, st))
    m.n_tokens.copy_(n_tok)
    engs[1].prefill(k_rows, v_rows, n_tok, q_place)
    torch.cuda.synchronize()
    e = sides[1]
    assert torch.equal(e.n_tokens, n_tok)
    for name in ("tier", "table", "last_sel", "free_head", "free_owner", "warm"):
        a, b = getattr(m.tier, name), getattr(e.tier, name)
        if a is not None:
            assert torch.equal(a, b), name
    for i in range(L):
        assert torch.equal(m.dig[i], e.dig[i]), i
    assert torch.equal(m.host, e.host)
    # the fast blocks' contents: every block on the fast tier holds its rows
    sb = ops.slot_bytes(kv)
    pm, pe = m.pool.view(torch.uint8).view(-1, sb), e.pool.view(torch.uint8).view(-1, sb)
    tab = m.tier.table.cpu()
    fast = m.tier.tier.cpu()
    for i in range(L):
        for u in range(U):
            nb = (int(n_tok[u]) + BS - 1) // BS
            for b in range(nb):
                if fast[i, u, b]:
                    s = int(tab[i, u, b])
                    assert torch.equal(pm[s], pe[s]), (i, u, b)
    assert int(e.tier.err.abs().sum()) == 0
    with pytest.raises(A.ScoutError):  # engine.hpp:194: prefill already done
        engs[1].prefill(k_rows, v_rows, n_tok, q_place)
    # identical decode steps from the two states
    outs = [[torch.empty(L, U * G, D, device="cuda"), torch.empty(L, U * G, 2, device="cuda")] for _ in range(2)]
    for step in range(1, steps + 1):
        qt = torch.randn(L, U * G, D, device="cuda").to(qdt)
        qp = (qt.float() + 0.3 * torch.randn(L, U * G, D, device="cuda")).to(qdt)
        co = torch.randn(L, U * G, D, device="cuda")
        cm = torch.stack([torch.randn(L, U * G, device="cuda"), torch.rand(L, U * G, device="cuda") + 0.1], -1).contiguous()
        kn, vn = torch.randn(L, U, D, device="cuda"), torch.randn(L, U, D, device="cuda")
        for eng, o in zip(engs, outs):
            eng.decode_step_kv(step, qt, qp, co, cm, kn, vn, *o)
        for eng in engs:
            eng.sync()
        torch.cuda.synchronize()
        assert torch.equal(outs[0][0], outs[1][0]) and torch.equal(outs[0][1], outs[1][1]), step
        for name in ("tier", "last_sel"):
            assert torch.equal(getattr(m.tier, name), getattr(e.tier, name)), (step, name)
    for eng in engs:
        eng.check_state()


def test_engine_prefill_rejects_bad_calls(cuda):
    """scout_engine_prefill's argument checks: a prefill longer than the rows
    it is given fails loudly (the tier's sticky error, reported by the call)."""
    L, batch, hkv, G, k, cap, nbs = 2, 1, 2, 4, 6, 8, 16
    U = batch * hkv
    kv = torch.bfloat16
    tier = DeviceTieredCache(L, U, nbs, capacity=cap, slots_per_unit=nbs)
    tier.pin_layer(0)
    pool = ops.alloc_pool(L * U * nbs, kv)
    dig = [torch.zeros(U, 2, D, nbs, dtype=kv, device="cuda") for _ in range(L)]
    host = torch.zeros(L * U * nbs * ops.slot_bytes(kv), dtype=torch.uint8).pin_memory()
    n_tokens = torch.zeros(U, dtype=torch.int32, device="cuda")
    layers = [LayerState(dig[i], torch.full((U, nbs), -1, dtype=torch.int32, device="cuda")) for i in range(L)]
    eng = DecodeEngine(layers=L, batch=batch, hq=hkv * G, hkv=hkv, k=k, n_tokens=n_tokens, pool=pool, kv_dtype=kv,
                       layer_states=layers, scale=1 / math.sqrt(D), recall_interval=0, host_tier=host, tier=tier,
                       q_dtype=torch.bfloat16)
    rows = torch.randn(L, U, 100, D, device="cuda")
    with pytest.raises(ValueError):
        eng.prefill(rows, rows, torch.tensor([100, 101], dtype=torch.int32), None)


@pytest.mark.parametrize("host", [False, True])
def test_engine_overlapped_step_matches_ordinary(cuda, host):
    """The overlapped step (K1 beside K2 on a share of the SMs, K2 polling
    K1's per-layer flags) against the ordinary order (K1, then K2) on an
    identical second cache: the same outputs, CPU-side ids and tier state bit
    for bit, step after step, through recalls (steps with a due ticket run in
    the ordinary order on both); the overlapped side really overlapped."""
    L, batch, hkv, G, k, cap, nbs, steps = 4, 2, 2, 4, 6, 8, 24, 40
    U = batch * hkv
    kv = torch.bfloat16
    T0 = 64 * 11 + 50
    torch.manual_seed(29)
    seed_rows = [[(torch.randn(U, D), torch.randn(U, D)) for _ in range(T0)] for _ in range(L)]
    sides = [Side(L, U, nbs, cap, kv, seed_rows) for _ in range(2)]
    engs = []
    for sd in sides:
        layers = [LayerState(sd.dig[i], torch.full((U, nbs), -1, dtype=torch.int32, device="cuda")) for i in range(L)]
        engs.append(DecodeEngine(layers=L, batch=batch, hq=hkv * G, hkv=hkv, k=k, n_tokens=sd.n_tokens, pool=sd.pool,
                                 kv_dtype=kv, layer_states=layers, scale=1 / math.sqrt(D), recall_interval=5,
                                 host_tier=sd.host, tier=sd.tier, q_dtype=torch.bfloat16, host_staging=host,
                                 chunk_layers=2))
    engs[0].set_overlap(40)
    engs[1].set_overlap(0)
    outs = [[torch.empty(L, U * G, D, device="cuda"), torch.empty(L, U * G, 2, device="cuda")] for _ in range(2)]
    h_outs = [[torch.empty(L, U * G, D).pin_memory(), torch.empty(L, U * G, 2).pin_memory(),
               torch.empty(L, U, k, dtype=torch.int32).pin_memory(), torch.empty(L, U, dtype=torch.int32).pin_memory()]
              for _ in range(2)]
    for step in range(1, steps + 1):
        ins = [torch.randn(L, U * G, D, device="cuda").bfloat16(), torch.randn(L, U * G, D, device="cuda").bfloat16(),
               torch.randn(L, U * G, D, device="cuda"),
               torch.stack([torch.randn(L, U * G, device="cuda"), torch.rand(L, U * G, device="cuda") + 0.1],
                           -1).contiguous(),
               torch.randn(L, U, D, device="cuda"), torch.randn(L, U, D, device="cuda")]
        if host:
            h_ins = [t.cpu().pin_memory() for t in ins]
            for e, ho in zip(engs, h_outs):
                e.decode_step_kv_host(step, *h_ins, ho[0], ho[1], ho[2], ho[3])
        else:
            for e, o in zip(engs, outs):
                e.decode_step_kv(step, *ins, *o)
        for e in engs:
            e.sync()
        torch.cuda.synchronize()
        if host:
            a, b = h_outs
            assert torch.equal(a[0], b[0]) and torch.equal(a[1], b[1]) and torch.equal(a[3], b[3]), step
            for li in range(L):  # the CPU-side ids: the first n_cpu of each row are defined
                for u in range(U):
                    n = int(a[3][li, u])
                    assert torch.equal(a[2][li, u, :n], b[2][li, u, :n]), (step, li, u)
        else:
            assert torch.equal(outs[0][0], outs[1][0]) and torch.equal(outs[0][1], outs[1][1]), step
        for name in ("tier", "last_sel", "table"):
            assert torch.equal(getattr(sides[0].tier, name), getattr(sides[1].tier, name)), (step, name)
    n_ov, sms = engs[0].overlap_stats()
    assert sms == 40 and n_ov >= steps // 2  # every step but the first and those with a due ticket
    assert engs[1].overlap_stats()[0] == 0
    for e in engs:
        e.check_state()
