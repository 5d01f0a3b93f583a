"""K5 device tier bookkeeping vs the reference TieredKvCache (kv_store.hpp,
compiled unchanged into oracle/_ref): the reference's own kv_store test cases
restated at block size 64, random op sequences (append / seal / evict,
mark_selected, schedule_recall incl. rejected tickets, begin_layer, the
residency planning view) compared block by block after every operation, and
place_after_prefill with K1's selection."""
import numpy as np
import pytest
import torch

import py_oracle as P
from paper_2603_27138_b200 import ops
from paper_2603_27138_b200.tier import DeviceTieredCache

pytestmark = pytest.mark.gpu
BS = 64


def _ids(rows, U):
    k = max(1, max((len(r) for r in rows), default=1))
    ids = np.zeros((U, k), np.int32)
    n = np.zeros(U, np.int32)
    for u, r in enumerate(rows):
        ids[u, :len(r)] = r
        n[u] = len(r)
    return torch.from_numpy(ids), torch.from_numpy(n)


def _compare(dev: DeviceTieredCache, refs, L):
    tier, ls, rd = dev.tier.cpu().numpy(), dev.last_sel.cpu().numpy(), dev.ready.cpu().numpy()
    for layer in range(L):
        tab = dev.residency_table(layer).cpu().numpy()
        for u, r in enumerate(refs):
            t, l, f = r.state(layer)
            n = len(t)
            assert np.array_equal(tier[layer, u, :n], t), (layer, u, "tier")
            assert np.array_equal(ls[layer, u, :n].astype(np.int64), l), (layer, u, "last_selected")
            assert np.array_equal((rd[layer, u, :n] >= 0).astype(np.int32), f), (layer, u, "in flight")
            assert np.array_equal(np.nonzero(tab[u] >= 0)[0], r.residency_set(layer)), (layer, u, "residency")


def _append_all(dev, refs, layer):
    sealed_ref = [r.append_token(layer, np.zeros(1), np.zeros(1)) for r in refs]
    _, sealed = dev.append_token(layer)
    assert [s if s is not None else -1 for s in sealed_ref] == sealed.cpu().tolist()


def test_tier_kv_store_cases(cuda):
    """test_kv_store.cpp:47-110 at block size 64: LRU eviction with the id
    tie-break, the open block outside capacity, recall visibility at (m+1, i)
    (planning view from (m, i+1)), and rejected recall requests."""
    dev = DeviceTieredCache(2, 1, 16, capacity=2, slots_per_unit=8)
    ref = P.RefCache(2, 1, 2)
    for _ in range(3 * BS):
        _append_all(dev, [ref], 0)
    _compare(dev, [ref], 2)
    assert dev.tier[0, 0, :3].tolist() == [0, 1, 1]
    dev.mark_selected(0, *_ids([[1]], 1), 5)
    ref.mark_selected(0, [1], 5)
    for _ in range(BS):
        _append_all(dev, [ref], 0)
    assert dev.tier[0, 0, :4].tolist() == [0, 1, 0, 1]
    _compare(dev, [ref], 2)
    # recall visibility
    dev.begin_layer(1, 0), ref.begin_layer(1, 0)
    dev.schedule_recall(0, *_ids([[0]], 1), 1, 0), ref.schedule_recall(0, [0], 1, 0)
    _compare(dev, [ref], 2)
    assert dev.residency_table(0)[0, 0].item() < 0
    dev.begin_layer(1, 1), ref.begin_layer(1, 1)
    assert dev.residency_table(0)[0, 0].item() >= 0 and dev.tier[0, 0, 0].item() == 0
    _compare(dev, [ref], 2)
    dev.mark_selected(0, *_ids([[0, 3]], 1), 6), ref.mark_selected(0, [0, 3], 6)
    assert dev.begin_layer(2, 0) == 1 and ref.begin_layer(2, 0) == 1
    _compare(dev, [ref], 2)
    assert dev.tier[0, 0, :4].tolist() == [1, 0, 0, 1]
    # rejected requests: already fast, unsealed (the open block), already in flight
    _append_all(dev, [ref], 0)  # opens block 4
    for bad in ([0], [4]):
        dev.schedule_recall(0, *_ids([bad], 1), 2, 0)
        with pytest.raises(ValueError):
            ref.schedule_recall(0, bad, 2, 0)
        with pytest.raises(ValueError):
            dev.check(0)
    dev.schedule_recall(0, *_ids([[1]], 1), 2, 0), ref.schedule_recall(0, [1], 2, 0)
    dev.check(0)
    dev.schedule_recall(0, *_ids([[1]], 1), 2, 0)
    with pytest.raises(ValueError):
        dev.check(0)
    _compare(dev, [ref], 2)


@pytest.mark.parametrize("seed", [0, 1, 2])
def test_tier_random_ops_vs_reference(cuda, seed):
    rng = np.random.default_rng(seed)
    L, U, cap, nbs = 3, 6, 4, 24
    dev = DeviceTieredCache(L, U, nbs, capacity=cap, slots_per_unit=nbs)
    refs = [P.RefCache(L, 1, cap) for _ in range(U)]
    dev.pin_layer(0)
    for r in refs:
        r.pin_layer(0)
    for layer in range(L):
        for _ in range(5 * BS + 10):
            _append_all(dev, refs, layer)
    _compare(dev, refs, L)
    for step in range(1, 9):
        for layer in range(L):
            dev.begin_layer(step, layer)
            for r in refs:
                r.begin_layer(step, layer)
            _compare(dev, refs, L)
            # mark_selected on the next layer (the layer-ahead selection)
            tgt = (layer + 1) % L
            nb = (int(dev.n_tokens[tgt, 0]) + BS - 1) // BS
            marks = [sorted(rng.choice(nb, size=3, replace=False).tolist()) for _ in range(U)]
            dev.mark_selected(tgt, *_ids(marks, U), step)
            for r, m in zip(refs, marks):
                r.mark_selected(tgt, m, step)
            # the layer's tokens (append after attention, engine.hpp:289); some appends seal
            for _ in range(int(rng.integers(1, 40))):
                _append_all(dev, refs, layer)
            _compare(dev, refs, L)
            # recall: slow sealed blocks not in flight, sometimes with a fast id (rejected)
            rows, bad_units = [], []
            for u, r in enumerate(refs):
                t, _, f = r.state(layer)
                ntok = int(dev.n_tokens[layer, u])
                cand = [b for b in range(len(t)) if not t[b] and not f[b] and (b + 1) * BS <= ntok]
                n = min(len(cand), int(rng.integers(0, 4)))
                pick = sorted(rng.choice(cand, size=n, replace=False).tolist()) if n else []
                if pick and rng.random() < 0.2:
                    fast = [b for b in range(len(t)) if t[b]]
                    pick = sorted(set(pick) | {fast[0]})
                    bad_units.append(u)
                rows.append(pick)
            dev.schedule_recall(layer, *_ids(rows, U), step, layer)
            for u, (r, pick) in enumerate(zip(refs, rows)):
                if not pick:
                    continue
                if u in bad_units:
                    with pytest.raises(ValueError):
                        r.schedule_recall(layer, pick, step, layer)
                else:
                    r.schedule_recall(layer, pick, step, layer)
            err = dev.err[layer].cpu().numpy()
            assert sorted(np.nonzero(err)[0].tolist()) == bad_units
            dev.err[layer].zero_()
            _compare(dev, refs, L)
    # slot bookkeeping: fast / in-flight blocks hold distinct slots of their own
    # range, and with the free ring they account for every slot exactly once
    _check_slots(dev, L, U, nbs)


def _check_slots(dev, L, U, nbs):
    tab = dev.table.cpu().numpy()
    tier, warm, owner = dev.tier.cpu().numpy(), dev.warm.cpu().numpy(), dev.free_owner.cpu().numpy()
    head, nf = dev.free_head.cpu().numpy(), dev.n_free.cpu().numpy()
    for layer in range(L):
        for u in range(U):
            nb = (int(dev.n_tokens[layer, u]) + BS - 1) // BS
            used = tab[layer, u, :nb][tab[layer, u, :nb] >= 0].tolist()
            free = dev.free_ring(layer, u)
            base = dev.layer_base[layer] + u * dev.spu_l[layer]
            assert sorted(used + free) == list(range(base, base + dev.spu_l[layer]))
            # victim cache: a warm block is slow, and its ring entry names it
            pos = {(int(head[layer, u]) + i) % dev.spu for i in range(int(nf[layer, u]))}
            for b in np.nonzero(warm[layer, u] >= 0)[0].tolist():
                p = int(warm[layer, u, b])
                assert p in pos and owner[layer, u, p] == b and tier[layer, u, b] == 0 and tab[layer, u, b] < 0


def test_tier_victim_cache_warm_recall(cuda):
    """Device victim cache: an evicted block's slot keeps its image at the
    back of the FIFO free ring; recalling the block takes the same slot back
    with nothing to copy (dst = -2 - slot). The tier state stays the
    reference's after every operation."""
    dev = DeviceTieredCache(1, 1, 16, capacity=2, slots_per_unit=4)
    ref = P.RefCache(1, 1, 2)
    for _ in range(3 * BS):  # blocks 0, 1, 2 take slots 0, 1, 2; sealing 2 evicts 0 (LRU tie -> lower id)
        _append_all(dev, [ref], 0)
    _compare(dev, [ref], 1)
    assert dev.tier[0, 0, :3].tolist() == [0, 1, 1]
    assert int(dev.warm[0, 0, 0]) >= 0 and dev.free_ring(0, 0) == [3, 0]
    dst = dev.schedule_recall(0, *_ids([[0]], 1), 0, 0)
    ref.schedule_recall(0, [0], 0, 0)
    assert int(dst[0, 0]) == -2 - 0  # warm: its own slot, no bytes to move
    assert int(dev.table[0, 0, 0]) == 0 and int(dev.warm[0, 0, 0]) == -1 and dev.free_ring(0, 0) == [3]
    _compare(dev, [ref], 1)
    _check_slots(dev, 1, 1, 16)


def test_tier_victim_cache_reused_slot_is_a_miss(cuda):
    """A warm image is forgotten when the ring hands its slot out again: the
    recall then gets the oldest free slot (dst >= 0, an H2D copy)."""
    dev = DeviceTieredCache(1, 1, 16, capacity=2, slots_per_unit=4)
    ref = P.RefCache(1, 1, 2)
    for _ in range(4 * BS + 1):  # ring after: block 3 took slot 3, its seal evicted 1; block 4 took slot 0
        _append_all(dev, [ref], 0)
    _compare(dev, [ref], 1)
    assert dev.tier[0, 0, :5].tolist() == [0, 0, 1, 1, 1]
    assert int(dev.warm[0, 0, 0]) == -1 and int(dev.warm[0, 0, 1]) >= 0 and dev.free_ring(0, 0) == [1]
    dst = dev.schedule_recall(0, *_ids([[0]], 1), 0, 0)
    ref.schedule_recall(0, [0], 0, 0)
    assert int(dst[0, 0]) == 1  # block 1's slot, whose image is now forgotten
    assert int(dev.warm[0, 0, 1]) == -1 and dev.free_ring(0, 0) == []
    _compare(dev, [ref], 1)
    _check_slots(dev, 1, 1, 16)


def test_tier_place_after_prefill_vs_reference(cuda):
    """place_after_prefill (kv_store.hpp:271-283) after a prefill: the
    reference evicts during the prefill appends and then re-places by the last
    prefill query; the device prefills the whole layer into HBM (no capacity)
    and places once. Final tiers and marks agree; digests are bit-exact."""
    rng = np.random.default_rng(11)
    U, cap, nbs, T = 4, 5, 16, 64 * 12 + 9
    dev = DeviceTieredCache(2, U, nbs, capacity=cap, slots_per_unit=nbs)
    refs = [P.RefCache(2, 128, cap) for _ in range(U)]
    dev.capacity[1] = 0  # prefill: every block in HBM
    pool = ops.alloc_pool(2 * U * nbs, torch.float32)
    dig = torch.zeros((U, 2, 128, nbs), dtype=torch.float32, device="cuda")
    for _ in range(T):
        k = rng.standard_normal((U, 128)).astype(np.float32)
        for u, r in enumerate(refs):
            r.append_token(1, k[u].astype(np.float64), np.zeros(128))
        dev.append_token(1, torch.from_numpy(k), torch.zeros(U, 128), pool, torch.float32, dig)
    for u, r in enumerate(refs):
        want, n = r.digests(1, nbs)
        assert np.array_equal(dig[u, :, :, :n].double().cpu().numpy(), want[:, :, :n])
    q = rng.standard_normal((U, 128)).astype(np.float32)
    dev.capacity[1] = cap
    keep, fill = dev.place_after_prefill(1, torch.from_numpy(q).cuda(), dig, 1)
    for u, r in enumerate(refs):
        r.place_after_prefill(1, q[u].astype(np.float64))
    _compare(dev, refs, 2)
    assert (fill[:, :cap] == -1).all()  # every kept block was already in HBM
    assert (dev.n_free[1].cpu().numpy() == nbs - (cap + 1)).all()  # kept + open block hold slots


@pytest.mark.parametrize("kv", [torch.bfloat16, torch.float32])
@pytest.mark.parametrize("T,cap", [(1, 3), (63, 3), (64, 3), (65, 2), (9 * BS + 17, 3), (12 * BS, 4), (9 * BS + 17, 0),
                                   (14 * BS + 5, 3)])
def test_tier_prefill_matches_token_appends(cuda, kv, T, cap):
    """scout_tier_prefill (one pass) against T append_token calls (the K0 / K5
    append path, itself bit-exact against the reference TieredKvCache): the
    same tier state (and the reference's, compared block by block), the same
    digests bit for bit, the fast blocks' rows in their slots, every sealed
    block's host image; warm images hold their block's rows. cap 0: a pinned
    layer."""
    U, nbs, spu = 3, 24, 10
    dev = torch.device("cuda")
    sb = ops.slot_bytes(kv)
    k_rows = torch.randn(U, T, 128, device=dev)
    v_rows = torch.randn(U, T, 128, device=dev)
    sides = []
    for _ in range(2):
        tc = DeviceTieredCache(1, U, nbs, capacity=max(cap, 1), slots_per_unit=nbs if cap == 0 else spu)
        if cap == 0:
            tc.pin_layer(0)
        pool = ops.alloc_pool(tc.n_slots, kv)
        pool.zero_()
        dig = torch.zeros(U, 2, 128, nbs, dtype=kv, device=dev)
        host = torch.zeros(U * nbs * sb, dtype=torch.uint8).pin_memory()
        sides.append((tc, pool, dig, host))
    tc, pool, dig, host = sides[0]
    for t in range(T):
        tc.append_token(0, k_rows[:, t], v_rows[:, t], pool, kv, dig, host_tier=host)
    tc2, pool2, dig2, host2 = sides[1]
    tc2.prefill(0, k_rows, v_rows, torch.full((U,), T, dtype=torch.int32), pool2, kv, dig2, host_tier=host2)
    torch.cuda.synchronize()
    ref = P.RefCache(1, 1, max(cap, 1))
    if cap == 0:
        ref.pin_layer(0)
    for _ in range(T):
        ref.append_token(0, np.zeros(1), np.zeros(1))
    for side in (tc, tc2):
        _compare(side, [ref] * U, 1)
    assert torch.equal(tc.tier, tc2.tier) and torch.equal(tc.last_sel, tc2.last_sel) and torch.equal(tc.ready, tc2.ready)
    nb = (T + BS - 1) // BS
    assert torch.equal(dig[..., :nb], dig2[..., :nb])
    assert torch.equal(host, host2)  # the sealed blocks' images (the open one is not written through)
    _check_slots(tc2, 1, U, nbs)
    pv, pv2 = pool.view(-1, sb), pool2.view(-1, sb)
    for u in range(U):
        for b in range(nb):
            rows = min(BS, T - b * BS)
            s1, s2 = int(tc.table[0, u, b]), int(tc2.table[0, u, b])
            assert (s1 >= 0) == (s2 >= 0)
            if s2 >= 0:  # a fast block: its rows in its slot
                k1, v1 = ops.kv_read_tokens(pool, kv, [s1] * rows, list(range(rows)))
                k2, v2 = ops.kv_read_tokens(pool2, kv, [s2] * rows, list(range(rows)))
                assert torch.equal(k1, k2) and torch.equal(v1, v2), (u, b)
            p = int(tc2.warm[0, u, b])
            if p >= 0:  # a warm image: the block's host image, byte for byte
                slot = int(tc2.free_slots[0, u, p])
                assert torch.equal(pv2[slot].cpu(), host2.view(-1, sb)[u * nbs + b]), (u, b)


def test_tier_prefill_rejects_counts_beyond_rows(cuda):
    """A token count beyond the rows given (or the stride) is the unit's
    invalid-argument error, and no row is read past the end."""
    dev = torch.device("cuda")
    tc = DeviceTieredCache(1, 2, 8, capacity=2, slots_per_unit=8)
    pool = ops.alloc_pool(tc.n_slots, torch.bfloat16)
    dig = torch.zeros(2, 2, 128, 8, dtype=torch.bfloat16, device=dev)
    k = torch.randn(2, 100, 128, device=dev)
    with pytest.raises(ValueError):
        tc.prefill(0, k, k, torch.tensor([100, 101], dtype=torch.int32), pool, torch.bfloat16, dig)
