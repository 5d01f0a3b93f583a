"""Device-resident TieredKvCache (the host-side mirror of the reference class
over the K5 C ABI).

`DeviceTieredCache` keeps the reference's API (proj/include/scout/kv_store.hpp:
append_token :90, residency_set :156, schedule_recall :175, begin_layer :201,
mark_selected :222, place_after_prefill :271, pin_layer :79) for n_units units
at once ("unit" = (request, KV head)); every unit is one reference cache and
all of them share the writer clock. The tier state lives in HBM and is only
touched by the K5 kernels; the host keeps the two things the reference keeps
on its clock side: the (step, layer) clock and the ledger of in-flight
tickets per layer (which layers begin_layer must visit).
"""
from __future__ import annotations

import ctypes as C

import torch

from . import _capi as A
from . import ops

BS = A.BLOCK_SIZE


class DeviceTieredCache:
    def __init__(self, layers: int, n_units: int, nb_stride: int, capacity: int, slots_per_unit,
                 device="cuda", slot_base: int = 0, victim_cache: bool = True):
        """slots_per_unit: pool slots each (layer, unit) owns, an int or one per
        layer (a pinned layer needs every block, the others capacity plus
        room for in-flight recalls and the open block; slots beyond that hold
        warm images of slow blocks). victim_cache: a recall of a block whose
        image still sits in a free slot takes that slot back and moves no
        bytes (scout_tier_layer.free_owner / warm); the tier state is the
        reference's either way."""
        self.L, self.U, self.nbs = layers, n_units, nb_stride
        spu = [int(slots_per_unit)] * layers if isinstance(slots_per_unit, int) else [int(x) for x in slots_per_unit]
        self.spu_l = spu
        self.spu = max(spu)
        self.dev = torch.device(device)
        dev, U, nbs = self.dev, n_units, nb_stride
        i32 = dict(dtype=torch.int32, device=dev)
        self.table = torch.full((layers, U, nbs), -1, **i32)
        self.tier = torch.zeros((layers, U, nbs), dtype=torch.uint8, device=dev)
        self.last_sel = torch.zeros((layers, U, nbs), **i32)
        self.ready = torch.full((layers, U, nbs), -1, **i32)
        self.ticket = torch.zeros((layers, U, nbs), **i32)
        # layer l, unit u owns pool slots layer_base[l] + u*spu[l] + [0, spu[l]); the free
        # slots form a FIFO ring per unit (head, n_free), lowest slot first
        self.layer_base = [slot_base + U * sum(spu[:l]) for l in range(layers)]
        self.free_slots = torch.zeros((layers, U, self.spu), **i32)
        for l in range(layers):
            base = self.layer_base[l] + torch.arange(U, **i32).view(U, 1) * spu[l]
            self.free_slots[l, :, :spu[l]] = base + torch.arange(spu[l], **i32).view(1, -1)
        self.n_free = torch.tensor(spu, **i32).view(layers, 1).repeat(1, U).contiguous()
        self.free_head = torch.zeros((layers, U), **i32)
        # device victim cache: a free slot that still holds an evicted block's image
        # (free_owner), and each slow block's ring position of such an image (warm)
        self.victim_cache = bool(victim_cache)
        self.free_owner = torch.full((layers, U, self.spu), -1, **i32)
        self.warm = torch.full((layers, U, nbs), -1, **i32)
        self.n_slots = U * sum(spu)
        self.err = torch.zeros((layers, U), **i32)
        self.n_tokens = torch.zeros((layers, U), **i32)
        self.capacity = [capacity] * layers
        self.clock_step, self.clock_layer = 0, 0
        self.pending: list[list[int]] = [[] for _ in range(layers)]  # ready ticks of in-flight tickets
        self.n_tickets = 0

    # -------------------------------------------------------------- helpers
    def tick(self, step: int, layer: int) -> int:
        return step * self.L + layer

    def layer_desc(self, layer: int) -> A.TierLayer:
        d = A.TierLayer()
        for name in ("table", "tier", "last_sel", "ready", "ticket", "free_slots", "n_free", "err", "free_head"):
            setattr(d, name, getattr(self, name)[layer].data_ptr())
        if self.victim_cache:
            d.free_owner = self.free_owner[layer].data_ptr()
            d.warm = self.warm[layer].data_ptr()
        d.capacity = self.capacity[layer]
        # the free stacks' row stride: the tensor is [L][U][max spu] whatever this
        # layer's own slot count (a layer owning fewer slots just never fills it)
        d.slots_per_unit = self.spu
        return d

    def next_run_of(self, layer: int) -> int:  # kv_store.hpp:328-331
        if self.clock_layer <= layer:
            return self.tick(self.clock_step, layer)
        return self.tick(self.clock_step + 1, layer)

    def check(self, layer: int):
        """Raise like the reference would (std::invalid_argument / logic errors
        surface as the units' sticky error codes)."""
        e = self.err[layer]
        bad = torch.nonzero(e).flatten().tolist()
        if bad:
            code = int(e[bad[0]])
            self.err[layer].zero_()
            if code == A.SCOUT_ERR_INVALID_ARGUMENT:
                raise ValueError(f"tier layer {layer}: invalid argument in units {bad}")
            raise RuntimeError(f"tier layer {layer}: out of pool slots in units {bad}")

    def adopt(self, layer: int, table: torch.Tensor, n_tokens: torch.Tensor, warm: torch.Tensor | None = None,
              warm_rank: torch.Tensor | None = None):
        """Start a layer from a placed state (a prefill done elsewhere): the
        blocks with a slot in table [U][nbs] are fast, the rest of the first
        n_tokens' blocks slow; every other slot of the (layer, unit) range goes
        on the free ring. warm [U][nbs] (optional, victim cache): slot of the
        range in which the caller left a slow block's image; those slots join
        the ring after the empty ones, ordered by warm_rank [U][nbs] (lower
        is reused first; default: block id). Marks start at 0."""
        U, spu = self.U, self.spu_l[layer]
        dev = self.dev
        table = table.to(device=dev, dtype=torch.int32)
        self.table[layer].copy_(table)
        self.tier[layer].copy_((table >= 0).to(torch.uint8))
        self.last_sel[layer].zero_()
        self.ready[layer].fill_(-1)
        self.n_tokens[layer].copy_(n_tokens)
        self.warm[layer].fill_(-1)
        self.free_owner[layer].fill_(-1)
        self.free_head[layer].zero_()
        base = self.layer_base[layer] + torch.arange(U, device=dev, dtype=torch.int32).view(U, 1) * spu
        cand = base + torch.arange(spu, device=dev, dtype=torch.int32).view(1, -1)  # [U][spu]
        # sort key per slot of the range: 0 empty, 1 + rank a warm image, USED a fast block's
        USED = 1 << 40
        key = torch.zeros((U, spu), dtype=torch.int64, device=dev)
        owner = torch.full((U, spu), -1, dtype=torch.int32, device=dev)
        rel = (table - base).long()
        ok = (table >= 0) & (rel >= 0) & (rel < spu)
        uu, bb = ok.nonzero(as_tuple=True)
        key[uu, rel[uu, bb]] = USED
        if warm is not None and self.victim_cache:
            warm = warm.to(device=dev, dtype=torch.int32)
            wrel = (warm - base).long()
            wok = (warm >= 0) & (table < 0) & (wrel >= 0) & (wrel < spu)
            uu, bb = wok.nonzero(as_tuple=True)
            rk = warm_rank[uu, bb].to(dev).long() if warm_rank is not None else bb.long()
            key[uu, wrel[uu, bb]] = 1 + rk
            owner[uu, wrel[uu, bb]] = bb.to(torch.int32)
        order = torch.sort(key, dim=1, stable=True).indices  # empty, warm by rank, then used
        nfree = (key < USED).sum(1)
        self.free_slots[layer, :, :spu] = cand.gather(1, order)
        ring_owner = owner.gather(1, order)
        pos = torch.arange(spu, device=dev).view(1, -1).expand(U, spu)
        ring_owner = torch.where(pos < nfree.view(U, 1), ring_owner, torch.full_like(ring_owner, -1))
        self.free_owner[layer, :, :spu] = ring_owner
        uu, pp = (ring_owner >= 0).nonzero(as_tuple=True)
        self.warm[layer][uu, ring_owner[uu, pp].long()] = pp.to(torch.int32)
        self.n_free[layer] = nfree.to(torch.int32)

    def forget_warm(self):
        """Drop every warm image (after engines ran with victim_cache off: the
        ring reused slots without updating the warm positions)."""
        self.warm.fill_(-1)
        self.free_owner.fill_(-1)

    def free_ring(self, layer: int, unit: int) -> list:
        """The unit's free slots, oldest (next to be reused) first."""
        n, h = int(self.n_free[layer, unit]), int(self.free_head[layer, unit])
        fs = self.free_slots[layer, unit].tolist()
        return [fs[(h + i) % self.spu] for i in range(n)]

    # ------------------------------------------------------------- reference API
    def pin_layer(self, layer: int):
        self.capacity[layer] = 0

    def append_token(self, layer: int, k_rows=None, v_rows=None, pool=None, kv_dtype=None, digests=None,
                     method=0, host_tier=None, host_blocks=0):
        """One token for every unit. Without a pool only the bookkeeping runs;
        with host_tier, sealed blocks are written through to their host images
        ((layer*U + unit)*nb_stride + id, modulo host_blocks)."""
        lib, st = A.lib(), torch.cuda.current_stream(self.dev).cuda_stream
        open_slot = torch.empty(self.U, dtype=torch.int32, device=self.dev)
        sealed = torch.empty(self.U, dtype=torch.int32, device=self.dev)
        nt = self.n_tokens[layer]
        desc = self.layer_desc(layer)
        A.check(lib.scout_tier_append(C.byref(desc), self.U, self.nbs, nt.data_ptr(), self.clock_step,
                                      open_slot.data_ptr(), sealed.data_ptr(), st))
        if pool is not None:
            ops.kv_append(pool, kv_dtype, method, open_slot, nt, k_rows, v_rows, digests, self.nbs, advance=True)
            if host_tier is not None:
                A.check(lib.scout_kv_writeback(pool.data_ptr(), ops.dtype_code(kv_dtype), host_tier.data_ptr(),
                                               layer * self.U * self.nbs, self.nbs, int(host_blocks), self.U,
                                               open_slot.data_ptr(), sealed.data_ptr(), st))
        else:
            nt.add_(1)
        return open_slot, sealed

    def prefill(self, layer: int, k_rows: torch.Tensor, v_rows: torch.Tensor, n_tokens: torch.Tensor, pool,
                kv_dtype, digests, host_tier=None, host_blocks=0) -> torch.Tensor:
        """The state n_tokens[u] append_token calls leave on a fresh layer
        (kv_store.hpp:90-117), in one pass (scout_tier_prefill): k_rows /
        v_rows [U][T][128] f32, the pool slots of the fast (and warm) blocks,
        min/max digests, sealed blocks written through to host_tier at the
        append path's image indices. Returns blk_slot [U][nb_stride]."""
        U, nbs = self.U, self.nbs
        k = k_rows.to(device=self.dev, dtype=torch.float32).contiguous()
        v = v_rows.to(device=self.dev, dtype=torch.float32).contiguous()
        self.n_tokens[layer].copy_(n_tokens.to(device=self.dev, dtype=torch.int32))
        blk = torch.empty((U, nbs), dtype=torch.int32, device=self.dev)
        desc = self.layer_desc(layer)
        A.check(A.lib().scout_tier_prefill(C.byref(desc), U, nbs, self.n_tokens[layer].data_ptr(), self.clock_step,
                                           k.data_ptr(), v.data_ptr(), int(k.shape[1]), pool.data_ptr(),
                                           ops.dtype_code(kv_dtype), digests.data_ptr(),
                                           None if host_tier is None else host_tier.data_ptr(),
                                           layer * U * nbs, int(host_blocks), blk.data_ptr(),
                                           torch.cuda.current_stream(self.dev).cuda_stream))
        self.check(layer)
        return blk

    def begin_layer(self, step: int, layer: int) -> int:
        """Advance the clock and apply every due ticket (kv_store.hpp:201-218)."""
        self.clock_step, self.clock_layer = step, layer
        now = self.tick(step, layer)
        lib, st = A.lib(), torch.cuda.current_stream(self.dev).cuda_stream
        applied = 0
        for l in range(self.L):
            due = [t for t in self.pending[l] if t <= now]
            if not due:
                continue
            self.pending[l] = [t for t in self.pending[l] if t > now]
            desc = self.layer_desc(l)
            A.check(lib.scout_tier_apply(C.byref(desc), self.U, self.nbs, self.n_tokens[l].data_ptr(), now, None, st))
            applied += len(due)
        return applied

    def schedule_recall(self, layer: int, ids: torch.Tensor, n_ids: torch.Tensor, issue_step: int,
                        issue_layer: int) -> torch.Tensor:
        """ids [U][k] ascending per unit (n_ids[u] valid; 0 = no recall for the
        unit). Returns the destination pool slots [U][k] for the H2D copies."""
        ids = ids.to(device=self.dev, dtype=torch.int32).contiguous()
        n_ids = n_ids.to(device=self.dev, dtype=torch.int32).contiguous()
        k = ids.shape[1]
        dst = torch.empty_like(ids)
        ready = self.tick(issue_step + 1, issue_layer)
        desc = self.layer_desc(layer)
        A.check(A.lib().scout_tier_schedule_recall(C.byref(desc), self.U, self.nbs, self.n_tokens[layer].data_ptr(),
                                                   ids.data_ptr(), n_ids.data_ptr(), k, ready, self.n_tickets,
                                                   dst.data_ptr(), torch.cuda.current_stream(self.dev).cuda_stream))
        self.n_tickets += 1
        self.pending[layer].append(ready)
        return dst

    def mark_selected(self, layer: int, ids: torch.Tensor, n_ids: torch.Tensor, step: int):
        ids = ids.to(device=self.dev, dtype=torch.int32).contiguous()
        n_ids = n_ids.to(device=self.dev, dtype=torch.int32).contiguous()
        desc = self.layer_desc(layer)
        A.check(A.lib().scout_tier_mark(C.byref(desc), self.U, self.nbs, ids.data_ptr(), n_ids.data_ptr(),
                                        ids.shape[1], step, torch.cuda.current_stream(self.dev).cuda_stream))

    def residency_table(self, layer: int) -> torch.Tensor:
        """residency_set (kv_store.hpp:156-170) as K1's block table [U][nb_stride]."""
        out = torch.empty((self.U, self.nbs), dtype=torch.int32, device=self.dev)
        desc = self.layer_desc(layer)
        A.check(A.lib().scout_tier_plan(C.byref(desc), self.U, self.nbs, self.n_tokens[layer].data_ptr(),
                                        self.next_run_of(layer), out.data_ptr(),
                                        torch.cuda.current_stream(self.dev).cuda_stream))
        return out

    def place_after_prefill(self, layer: int, q: torch.Tensor, digests: torch.Tensor, group: int, kv_dtype=None):
        """Keep the top-capacity sealed blocks of every unit fast (kv_store.hpp:271-283):
        K1 over the sealed blocks (n_tokens rounded down to whole blocks)."""
        if self.capacity[layer] <= 0:
            return
        sealed_tok = (self.n_tokens[layer] // BS) * BS
        r = ops.score_topk_split(q, digests, sealed_tok.contiguous(), self.capacity[layer], group)
        desc = self.layer_desc(layer)
        fill = torch.empty_like(r["sel_ids"])
        A.check(A.lib().scout_tier_place(C.byref(desc), self.U, self.nbs, self.n_tokens[layer].data_ptr(),
                                         r["sel_ids"].data_ptr(), r["n_sel"].data_ptr(), r["sel_ids"].shape[1],
                                         fill.data_ptr(), torch.cuda.current_stream(self.dev).cuda_stream))
        return r["sel_ids"], fill
