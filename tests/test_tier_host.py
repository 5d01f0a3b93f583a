"""DeviceTieredCache's host-side bookkeeping on CPU tensors (no kernel runs):
adopt() lays out the free-slot ring of the device victim cache -- empty slots
first, then the caller's warm images ordered by warm_rank (lower = reused
first), the fast blocks' slots outside the ring -- with every warm block's
ring position pointing at an entry that names it."""
import torch

from paper_2603_27138_b200.tier import DeviceTieredCache


def _cache(L=2, U=2, nbs=16, cap=3, spu=8):
    return DeviceTieredCache(L, U, nbs, capacity=cap, slots_per_unit=spu, device="cpu")


def test_adopt_ring_order_and_warm_positions():
    c = _cache()
    U, nbs, spu = 2, 16, 8
    n_tokens = torch.full((U,), 10 * 64, dtype=torch.int32)
    layer = 1
    base = [c.layer_base[layer] + u * spu for u in range(U)]
    table = torch.full((U, nbs), -1, dtype=torch.int32)
    warm = torch.full((U, nbs), -1, dtype=torch.int32)
    rank = torch.zeros(U, nbs, dtype=torch.int64)
    for u in range(U):
        for i, b in enumerate((2, 5, 9)):  # fast blocks in slots 0..2
            table[u, b] = base[u] + i
        for i, (b, r) in enumerate(((1, 2), (4, 0), (7, 1))):  # warm images in slots 3..5, ranks
            warm[u, b] = base[u] + 3 + i
            rank[u, b] = r
    c.adopt(layer, table, n_tokens, warm=warm, warm_rank=rank)
    for u in range(U):
        ring = c.free_ring(layer, u)
        # empty slots 6, 7 first, then the warm slots by rank: block 4 (slot 4), 7 (slot 5), 1 (slot 3)
        assert ring == [base[u] + 6, base[u] + 7, base[u] + 4, base[u] + 5, base[u] + 3]
        assert int(c.n_free[layer, u]) == 5 and int(c.free_head[layer, u]) == 0
        for b, slot in ((4, 4), (7, 5), (1, 3)):
            p = int(c.warm[layer, u, b])
            assert int(c.free_slots[layer, u, p]) == base[u] + slot and int(c.free_owner[layer, u, p]) == b
        assert int((c.warm[layer, u] >= 0).sum()) == 3
        assert c.tier[layer, u].nonzero().flatten().tolist() == [2, 5, 9]


def test_adopt_without_victim_cache_and_forget_warm():
    c = DeviceTieredCache(1, 1, 16, capacity=2, slots_per_unit=6, device="cpu", victim_cache=False)
    table = torch.full((1, 16), -1, dtype=torch.int32)
    table[0, 3] = c.layer_base[0] + 2
    warm = torch.full((1, 16), -1, dtype=torch.int32)
    warm[0, 5] = c.layer_base[0] + 4
    c.adopt(0, table, torch.full((1,), 8 * 64, dtype=torch.int32), warm=warm)
    # victim cache off: the warm table is ignored, every other slot is plainly free
    assert c.free_ring(0, 0) == [0, 1, 3, 4, 5]
    assert int((c.warm >= 0).sum()) == 0 and int((c.free_owner >= 0).sum()) == 0
    d = c.layer_desc(0)
    assert not d.free_owner and not d.warm and d.free_head
    c2 = _cache()
    c2.warm.fill_(3)
    c2.free_owner.fill_(1)
    c2.forget_warm()
    assert int((c2.warm >= 0).sum()) == 0 and int((c2.free_owner >= 0).sum()) == 0
