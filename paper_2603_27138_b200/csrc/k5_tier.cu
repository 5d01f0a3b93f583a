// K5 — device-resident tier bookkeeping.
//
// The GPU mirror of TieredKvCache's per-layer state (reference
// proj/include/scout/kv_store.hpp:296-305): tier flag, last_selected mark,
// in-flight recall ticket and the pool slot of every block of every unit,
// plus a per-(layer, unit) stack of free pool slots. It replaces the
// reference's host bookkeeping on the decode path:
//   append_token's block open / seal        kv_store.hpp:90-117
//   residency_set (the planning view)       kv_store.hpp:156-170
//   schedule_recall                         kv_store.hpp:175-197
//   begin_layer (apply due recalls)         kv_store.hpp:201-218
//   enforce_capacity (LRU, ties -> lower id) kv_store.hpp:333-345
//   place_after_prefill                     kv_store.hpp:271-283
// mark_selected (kv_store.hpp:222-228) is K1's last_selected output.
// One CTA per unit; the LRU victim search is a block-wide argmin over the
// (last_selected, id) key, one round per evicted block (the excess is the
// handful of blocks a recall or a seal adds, so rounds are few).
#include "scout_common.cuh"

#include <climits>

using namespace scout_dev;

namespace {

constexpr int TT = 128;  // threads per unit
constexpr int TW = TT / 32;

struct TierSm {
    unsigned long long red[TW];
    int cnt[TW];
    int n_free;
    int err;
};

__device__ __forceinline__ int n_blocks_of(int ntok) { return (ntok + BS - 1) / BS; }
// a block is sealed once it holds B rows (kv_store.hpp:111)
__device__ __forceinline__ bool sealed(int id, int ntok) { return (id + 1) * BS <= ntok; }

__device__ int block_sum(int v, TierSm& S) {
    const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
#pragma unroll
    for (int o = 16; o; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
    if (lane == 0) S.cnt[w] = v;
    __syncthreads();
    int t = 0;
#pragma unroll
    for (int i = 0; i < TW; ++i) t += S.cnt[i];
    __syncthreads();
    return t;
}

__device__ unsigned long long block_min(unsigned long long v, TierSm& S) {
    const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
#pragma unroll
    for (int o = 16; o; o >>= 1) {
        const unsigned long long y = __shfl_xor_sync(0xffffffffu, v, o);
        v = y < v ? y : v;
    }
    if (lane == 0) S.red[w] = v;
    __syncthreads();
    unsigned long long t = S.red[0];
#pragma unroll
    for (int i = 1; i < TW; ++i) t = S.red[i] < t ? S.red[i] : t;
    __syncthreads();
    return t;
}

struct Unit {
    int32_t* table;
    uint8_t* tier;
    int32_t* last_sel;
    int32_t* ready;
    int32_t* ticket;
    int32_t* free_slots;
    int32_t* n_free;
    int32_t* err;
    int32_t* head;   // free ring head
    int32_t* owner;  // [S] block whose image the ring entry's slot holds (nullptr: no victim cache)
    int32_t* warm;   // [nbs] ring position of a slow block's image, -1
    int S;           // ring size
};

__device__ Unit unit_of(const scout_tier_layer& L, int u, int nbs) {
    const size_t o = static_cast<size_t>(u) * nbs, r = static_cast<size_t>(u) * L.slots_per_unit;
    const bool vc = L.free_owner && L.warm;
    return Unit{L.table + o, L.tier + o, L.last_sel + o, L.ready + o, L.ticket + o, L.free_slots + r, L.n_free + u,
                L.err + u, L.free_head + u, vc ? L.free_owner + r : nullptr, vc ? L.warm + o : nullptr,
                L.slots_per_unit};
}

// ---- the free ring (one thread of the unit's CTA at a time). FIFO: a slot
// freed by an eviction waits as long as possible before it is reused, so its
// image (the evicted block's) serves as long as possible as a warm copy.
// The oldest entry is taken; its slot's image, if any, is forgotten.
__device__ int ring_pop(const Unit& U) {
    const int n = *U.n_free;
    if (n <= 0) return -1;
    const int h = *U.head;
    const int slot = U.free_slots[h];
    if (U.owner) {
        const int o = U.owner[h];
        if (o >= 0 && U.warm[o] == h) U.warm[o] = -1;
    }
    *U.head = h + 1 == U.S ? 0 : h + 1;
    *U.n_free = n - 1;
    return slot;
}
// a freed slot goes to the back; owner >= 0: it holds that (now slow) block's image
__device__ bool ring_push(const Unit& U, int slot, int owner) {
    const int n = *U.n_free;
    if (n >= U.S) return false;
    int p = *U.head + n;
    if (p >= U.S) p -= U.S;
    U.free_slots[p] = slot;
    if (U.owner) {
        U.owner[p] = owner;
        if (owner >= 0) U.warm[owner] = p;
    }
    *U.n_free = n + 1;
    return true;
}
// block b's warm image leaves the ring with its slot (-1: b has none); the
// oldest entry fills the hole
__device__ int ring_take(const Unit& U, int b) {
    if (!U.owner) return -1;
    const int p = U.warm[b];
    if (p < 0) return -1;
    const int slot = U.free_slots[p];
    U.warm[b] = -1;
    const int h = *U.head;
    if (p != h) {
        const int s2 = U.free_slots[h], o2 = U.owner[h];
        U.free_slots[p] = s2;
        U.owner[p] = o2;
        if (o2 >= 0) U.warm[o2] = p;
    }
    *U.head = h + 1 == U.S ? 0 : h + 1;
    *U.n_free -= 1;
    return slot;
}

// schedule_recall's slot assignment for a validated ticket (thread 0): warm
// blocks take their own slot back first (dst = -2 - slot: no bytes to move),
// then the others take the oldest free slots (dst = slot: the H2D copy's
// destination). n <= n_free was checked, and every recalled block consumes
// exactly one ring entry, so no pop can fail. Returns the warm count.
__device__ int assign_recall_slots(const Unit& U, const int32_t* ids, int n, int32_t* dst) {
    int hits = 0;
    for (int i = 0; i < n; ++i) {
        const int b = ids[i];
        const int s = ring_take(U, b);
        dst[i] = s >= 0 ? -2 - s : -1;
        if (s >= 0) {
            U.table[b] = s;
            ++hits;
        }
    }
    if (hits < n)
        for (int i = 0; i < n; ++i) {
            if (dst[i] != -1) continue;
            const int b = ids[i];
            const int s = ring_pop(U);
            U.table[b] = s;
            dst[i] = s;
        }
    return hits;
}

__device__ bool find_sorted_dev(const int32_t* v, int n, int x) {
    int lo = 0, hi = n;
    while (lo < hi) {
        const int mid = (lo + hi) >> 1;
        if (v[mid] < x) lo = mid + 1;
        else hi = mid;
    }
    return lo < n && v[lo] == x;
}

__device__ void set_err(Unit& U, int code) {
    if (*U.err == 0) *U.err = code;
}

// enforce_capacity (kv_store.hpp:333-345): while more sealed fast blocks than
// capacity, demote the least recently selected one (ties -> lower id) and
// return its slot to the free stack.
__device__ void enforce_capacity(const scout_tier_layer& L, Unit& U, int nb, int ntok, TierSm& S) {
    if (L.capacity <= 0) return;  // pinned layer
    int mine = 0;
    for (int b = threadIdx.x; b < nb; b += TT) mine += (U.tier[b] && sealed(b, ntok));
    int excess = block_sum(mine, S) - L.capacity;
    while (excess > 0) {
        unsigned long long key = ~0ull;
        for (int b = threadIdx.x; b < nb; b += TT)
            if (U.tier[b] && sealed(b, ntok)) {
                const unsigned long long k =
                    (static_cast<unsigned long long>(static_cast<uint32_t>(U.last_sel[b])) << 32) | static_cast<uint32_t>(b);
                key = k < key ? k : key;
            }
        key = block_min(key, S);
        if (threadIdx.x == 0) {
            const int v = static_cast<int>(key & 0xFFFFFFFFu);
            U.tier[v] = 0;
            ring_push(U, U.table[v], v);  // the slot keeps v's image: a warm copy
            U.table[v] = -1;
        }
        __syncthreads();
        --excess;
    }
}

// append_token's bookkeeping (kv_store.hpp:95-115) for one layer: n_tokens is
// the count BEFORE the append. A new block takes a slot from the free stack,
// is fast and marked with the clock step; the append that fills it seals it
// (mark = clock step again) and enforces capacity.
__global__ void __launch_bounds__(TT) tier_append_kernel(const scout_tier_layer L, int nbs, const int32_t* n_tokens,
                                                         int clock_step, int32_t* open_slot, int32_t* sealed_id) {
    __shared__ TierSm S;
    const int u = blockIdx.x;
    Unit U = unit_of(L, u, nbs);
    const int pos = n_tokens[u];
    const int id = pos / BS;
    if (threadIdx.x == 0) {
        if (id >= nbs) {
            set_err(U, SCOUT_ERR_INVALID_ARGUMENT);
            S.err = 1;
        } else {
            S.err = 0;
            if (pos % BS == 0) {
                const int slot = ring_pop(U);
                if (slot < 0) {
                    set_err(U, SCOUT_ERR_LOGIC);  // no pool slot for the new open block
                    S.err = 1;
                } else {
                    U.table[id] = slot;
                    U.tier[id] = 1;
                    U.ready[id] = -1;
                    U.last_sel[id] = clock_step;
                }
            }
        }
        if (open_slot) open_slot[u] = S.err ? -1 : U.table[id];
        if (sealed_id) sealed_id[u] = (!S.err && (pos + 1) % BS == 0) ? id : -1;
    }
    __syncthreads();
    if (S.err || (pos + 1) % BS != 0) return;
    if (threadIdx.x == 0) U.last_sel[id] = clock_step;
    __syncthreads();
    enforce_capacity(L, U, id + 1, pos + 1, S);
}

// begin_layer's application for one layer (kv_store.hpp:201-218): every
// in-flight block whose ready tick <= due_tick becomes fast; tickets are
// applied in issue order (ticket number), each followed by enforce_capacity.
__device__ void apply_unit(const scout_tier_layer& L, int u, int nbs, const int32_t* n_tokens, int due_tick,
                           int32_t* n_applied, TierSm& S) {
    Unit U = unit_of(L, u, nbs);
    const int ntok = n_tokens[u];
    const int nb = min(n_blocks_of(ntok), nbs);
    int applied = 0;
    for (;;) {
        unsigned long long t = ~0ull;
        for (int b = threadIdx.x; b < nb; b += TT)
            if (U.ready[b] >= 0 && U.ready[b] <= due_tick) {
                const unsigned long long k = static_cast<uint32_t>(U.ticket[b]);
                t = k < t ? k : t;
            }
        t = block_min(t, S);
        if (t == ~0ull) break;
        int mine = 0;
        for (int b = threadIdx.x; b < nb; b += TT)
            if (U.ready[b] >= 0 && U.ready[b] <= due_tick && static_cast<uint32_t>(U.ticket[b]) == t) {
                U.tier[b] = 1;
                U.ready[b] = -1;
                ++mine;
            }
        applied += block_sum(mine, S);
        enforce_capacity(L, U, nb, ntok, S);
    }
    if (threadIdx.x == 0 && n_applied) n_applied[u] = applied;
}

__global__ void __launch_bounds__(TT) tier_apply_kernel(const scout_tier_layer L, int nbs, const int32_t* n_tokens,
                                                        int due_tick, int32_t* n_applied) {
    __shared__ TierSm S;
    apply_unit(L, blockIdx.x, nbs, n_tokens, due_tick, n_applied, S);
}

// schedule_recall (kv_store.hpp:175-197): ids must be sealed, slow and not in
// flight, else the unit's whole ticket is rejected (the reference throws
// before changing anything). Accepted blocks get a pool slot (the H2D
// destination, dst_slots) and the ready tick; n_ids[u] == 0 skips the unit.
__global__ void __launch_bounds__(TT) tier_recall_kernel(const scout_tier_layer L, int nbs, const int32_t* n_tokens,
                                                         const int32_t* ids, const int32_t* n_ids, int k_stride,
                                                         int ready_tick, int ticket, int32_t* dst_slots) {
    __shared__ TierSm S;
    const int u = blockIdx.x;
    Unit U = unit_of(L, u, nbs);
    const int n = n_ids[u];
    if (n <= 0) return;
    const int ntok = n_tokens[u];
    const int nb = min(n_blocks_of(ntok), nbs);
    const int32_t* my = ids + static_cast<size_t>(u) * k_stride;
    int bad = 0;
    for (int i = threadIdx.x; i < n; i += TT) {
        const int id = my[i];
        if (id < 0 || id >= nb || !sealed(id, ntok) || U.tier[id] || U.ready[id] >= 0 ||
            (i > 0 && my[i - 1] >= id))  // ids must be a sorted set
            bad = 1;
    }
    bad = block_sum(bad, S);
    if (threadIdx.x == 0) {
        S.err = 0;
        if (bad) {
            set_err(U, SCOUT_ERR_INVALID_ARGUMENT);
            S.err = 1;
        } else if (*U.n_free < n) {
            set_err(U, SCOUT_ERR_LOGIC);  // not enough free pool slots for the ticket
            S.err = 1;
        } else {
            assign_recall_slots(U, my, n, dst_slots + static_cast<size_t>(u) * k_stride);
        }
    }
    __syncthreads();
    if (S.err) {
        for (int i = threadIdx.x; i < n; i += TT) dst_slots[static_cast<size_t>(u) * k_stride + i] = -1;
        return;
    }
    for (int i = threadIdx.x; i < n; i += TT) {
        const int id = my[i];
        U.ready[id] = ready_tick;
        U.ticket[id] = ticket;
    }
}

// residency_set (kv_store.hpp:156-170) as K1's block table: the slot of every
// fast block and of every in-flight block ready by the layer's next run.
__global__ void __launch_bounds__(TT) tier_plan_kernel(const scout_tier_layer L, int nbs, const int32_t* n_tokens,
                                                       int next_tick, int32_t* block_table) {
    const int u = blockIdx.x;
    const size_t o = static_cast<size_t>(u) * nbs;
    const int nb = min(n_blocks_of(n_tokens[u]), nbs);
    for (int b = threadIdx.x; b < nbs; b += TT) {
        int v = -1;
        if (b < nb) {
            const int r = L.ready[o + b];
            if (L.tier[o + b] || (r >= 0 && r <= next_tick)) v = L.table[o + b];
        }
        block_table[o + b] = v;
    }
}

// place_after_prefill (kv_store.hpp:271-283): sealed blocks in keep (K1's
// top-capacity selection over the sealed blocks, ascending ids) are fast, the
// other sealed blocks go slow and free their slots (which keep their images:
// warm copies); a kept block that was slow takes its warm slot back
// (fill_slots[u][i] = -2 - slot, nothing to copy) or the oldest free slot
// (fill_slots[u][i] = slot, for the H2D fill of its image), else -1. Pinned
// layers keep all.
__global__ void __launch_bounds__(TT) tier_place_kernel(const scout_tier_layer L, int nbs, const int32_t* n_tokens,
                                                        const int32_t* keep, const int32_t* n_keep, int k_stride,
                                                        int32_t* fill_slots) {
    __shared__ TierSm S;
    if (L.capacity <= 0) return;
    const int u = blockIdx.x, lane = threadIdx.x & 31, w = threadIdx.x >> 5;
    Unit U = unit_of(L, u, nbs);
    const int ntok = n_tokens[u];
    const int nb = min(n_blocks_of(ntok), nbs);
    const int32_t* kp = keep + static_cast<size_t>(u) * k_stride;
    const int nk = n_keep[u];
    const int head = *U.head, n0 = *U.n_free;
    // demote the sealed blocks outside keep; the fast ones' slots join the
    // ring in id order (an order-preserving compaction per round)
    int pushed = 0;
    for (int base = 0; base < nb; base += TT) {
        const int b = base + static_cast<int>(threadIdx.x);
        bool freed = false;
        if (b < nb && sealed(b, ntok) && !find_sorted_dev(kp, nk, b)) {
            freed = U.tier[b] && U.table[b] >= 0;
            if (!freed) U.table[b] = -1;
            U.tier[b] = 0;
        }
        const unsigned bal = __ballot_sync(0xffffffffu, freed);
        if (lane == 0) S.cnt[w] = __popc(bal);
        __syncthreads();
        int off = pushed, tot = 0;
#pragma unroll
        for (int i = 0; i < TW; ++i) {
            off += i < w ? S.cnt[i] : 0;
            tot += S.cnt[i];
        }
        if (freed) {
            const int q = n0 + off + __popc(bal & ((1u << lane) - 1u));
            if (q < U.S) {
                const int p = (head + q) % U.S;
                U.free_slots[p] = U.table[b];
                if (U.owner) {
                    U.owner[p] = b;
                    U.warm[b] = p;
                }
            }
            U.table[b] = -1;
        }
        pushed += tot;
        __syncthreads();
    }
    // promote the kept blocks that were slow (one thread: the ring's order)
    if (threadIdx.x == 0) {
        *U.n_free = min(n0 + pushed, U.S);
        int err = 0;
        for (int i = 0; i < nk; ++i) {
            const int b = kp[i];
            int fill = -1;
            if (b >= 0 && b < nb && !U.tier[b]) {
                int s = ring_take(U, b);
                if (s >= 0) {
                    fill = -2 - s;
                } else {
                    s = ring_pop(U);
                    fill = s;
                }
                if (s >= 0) {
                    U.table[b] = s;
                    U.tier[b] = 1;
                    U.ready[b] = -1;
                } else {
                    err = 1;
                }
            }
            if (fill_slots) fill_slots[static_cast<size_t>(u) * k_stride + i] = fill;
        }
        if (err) set_err(U, SCOUT_ERR_LOGIC);
    }
}

// mark_selected (kv_store.hpp:222-228) for explicit id lists (K1 marks its
// own selections through last_selected).
__global__ void __launch_bounds__(TT) tier_mark_kernel(const scout_tier_layer L, int nbs, const int32_t* ids,
                                                       const int32_t* n_ids, int k_stride, int step) {
    const int u = blockIdx.x;
    const int n = n_ids[u];
    for (int i = threadIdx.x; i < n; i += TT) {
        const int id = ids[static_cast<size_t>(u) * k_stride + i];
        if (id >= 0 && id < nbs) L.last_sel[static_cast<size_t>(u) * nbs + id] = step;
    }
}

// ---- bulk prefill (the caller side of the decode path): the state T_u
// append_token calls at clock_step leave (kv_store.hpp:90-117) on a fresh
// layer, in one pass. Sealed blocks beyond capacity went slow in id order (all
// carry the same mark, so the LRU tie-break evicts the lowest id first); the
// last `capacity` sealed blocks and the open block are fast. The fast blocks
// take the ring's first entries; the highest-id slow blocks keep warm images
// in its last entries (eviction order: lowest id reused first). blk_slot[u][b]
// is the slot that receives block b's rows (fast or warm), else -1.
__global__ void __launch_bounds__(TT) tier_prefill_state_kernel(const scout_tier_layer L, int nbs,
                                                                 const int32_t* n_tokens, int max_tokens,
                                                                 int clock_step, int32_t* blk_slot) {
    const int u = blockIdx.x;
    Unit U = unit_of(L, u, nbs);
    const int T = n_tokens[u];
    const int nb = n_blocks_of(T), ns = T / BS;
    const int first_fast = L.capacity <= 0 ? 0 : max(0, ns - L.capacity);
    int32_t* bs = blk_slot + static_cast<size_t>(u) * nbs;
    for (int b = threadIdx.x; b < nbs; b += TT) {
        U.tier[b] = b < nb && b >= first_fast;
        U.last_sel[b] = b < nb ? clock_step : 0;
        U.ready[b] = -1;
        U.ticket[b] = 0;
        U.table[b] = -1;
        if (U.owner) U.warm[b] = -1;
        bs[b] = -1;
    }
    __syncthreads();
    if (threadIdx.x != 0) return;
    if (T < 0 || T > max_tokens || nb > nbs || nb - first_fast > *U.n_free) {
        set_err(U, nb - first_fast > *U.n_free && T <= max_tokens && nb <= nbs && T >= 0 ? SCOUT_ERR_LOGIC
                                                                                       : SCOUT_ERR_INVALID_ARGUMENT);
        return;
    }
    int h = *U.head, n = *U.n_free;
    for (int b = first_fast; b < nb; ++b) {
        const int slot = U.free_slots[h];
        if (U.owner) U.owner[h] = -1;
        U.table[b] = slot;
        bs[b] = slot;
        h = h + 1 == U.S ? 0 : h + 1;
        --n;
    }
    *U.head = h;
    *U.n_free = n;
    if (!U.owner) return;
    const int w = min(n, first_fast);  // warm images: slow blocks first_fast - w .. first_fast - 1
    for (int i = 0; i < n; ++i) {
        int p = h + i;
        if (p >= U.S) p -= U.S;
        const int o = i - (n - w);  // the last w entries
        if (o >= 0) {
            const int b = first_fast - w + o;
            U.owner[p] = b;
            U.warm[b] = p;
            bs[b] = U.free_slots[p];
        } else {
            U.owner[p] = -1;
        }
    }
}

// the prefill's rows: one CTA per (block, unit), thread = channel. The block's
// image is assembled in shared memory in the pool's slot layout, copied into
// its slot (fast or warm) and, once sealed, to its host-tier image
// (write-through); the min / max digest folds its rows in order as
// build_digest does (digest.hpp:34-60).
template <typename T>
__global__ void __launch_bounds__(TT) tier_prefill_data_kernel(const int32_t* n_tokens, const float* k_rows,
                                                                const float* v_rows, int max_tokens,
                                                                const int32_t* blk_slot, int nbs, uint8_t* pool,
                                                                void* digests, uint8_t* host_tier,
                                                                long long host_base, long long host_blocks) {
    extern __shared__ __align__(16) uint8_t img[];
    const int b = blockIdx.x, u = blockIdx.y, c = threadIdx.x;
    const int Tu = n_tokens[u];
    if (b * BS >= Tu || Tu > max_tokens || b >= nbs) return;  // (an oversized count is the state kernel's error)
    const int rows = min(BS, Tu - b * BS);
    constexpr size_t tile = static_cast<size_t>(BS) * D;
    constexpr size_t sbytes = 2 * tile * sizeof(T);
    T* im = reinterpret_cast<T*>(img);
    for (int i = c; i < static_cast<int>(sbytes / 16); i += TT) reinterpret_cast<int4*>(img)[i] = make_int4(0, 0, 0, 0);
    __syncthreads();
    float lo = 0.f, hi = 0.f;
    const size_t r0 = (static_cast<size_t>(u) * max_tokens + static_cast<size_t>(b) * BS) * D + c;
    for (int r = 0; r < rows; ++r) {
        T kq, vq;
        float kv;
        if constexpr (sizeof(T) == 2) {
            kq = __float2bfloat16_rn(k_rows[r0 + static_cast<size_t>(r) * D]);
            vq = __float2bfloat16_rn(v_rows[r0 + static_cast<size_t>(r) * D]);
            kv = __bfloat162float(kq);
            const int off = bf16_tile_offset(r, c);
            im[off] = kq;
            im[tile + off] = vq;
        } else {
            kq = k_rows[r0 + static_cast<size_t>(r) * D];
            vq = v_rows[r0 + static_cast<size_t>(r) * D];
            kv = kq;
            im[r * D + c] = kq;
            im[tile + r * D + c] = vq;
        }
        if (r == 0) {
            lo = kv;
            hi = kv;
        } else {  // std::min / std::max fold (digest.hpp:45-46)
            if (kv < lo) lo = kv;
            if (hi < kv) hi = kv;
        }
    }
    T* dig = static_cast<T*>(digests) + static_cast<size_t>(u) * 2 * D * nbs;
    if constexpr (sizeof(T) == 2) {
        dig[static_cast<size_t>(c) * nbs + b] = __float2bfloat16_rn(lo);
        dig[static_cast<size_t>(D + c) * nbs + b] = __float2bfloat16_rn(hi);
    } else {
        dig[static_cast<size_t>(c) * nbs + b] = lo;
        dig[static_cast<size_t>(D + c) * nbs + b] = hi;
    }
    __syncthreads();
    const int slot = blk_slot[static_cast<size_t>(u) * nbs + b];
    const int4* src = reinterpret_cast<const int4*>(img);
    if (slot >= 0) {
        int4* dst = reinterpret_cast<int4*>(pool + static_cast<size_t>(slot) * sbytes);
        for (int i = c; i < static_cast<int>(sbytes / 16); i += TT) dst[i] = src[i];
    }
    if (rows == BS && host_tier) {
        long long hidx = host_base + static_cast<long long>(u) * nbs + b;
        if (host_blocks > 0) hidx %= host_blocks;
        int4* dst = reinterpret_cast<int4*>(host_tier + static_cast<size_t>(hidx) * sbytes);
        for (int i = c; i < static_cast<int>(sbytes / 16); i += TT) dst[i] = src[i];
    }
}

int check_layer(const scout_tier_layer* L, int n_units, int nbs, const char* what) {
    using namespace scout_host;
    if (!L || n_units < 0 || nbs <= 0 ||
        (n_units > 0 && (!L->table || !L->tier || !L->last_sel || !L->ready || !L->ticket || !L->free_slots ||
                         !L->n_free || !L->err || !L->free_head || L->slots_per_unit <= 0 ||
                         (L->free_owner == nullptr) != (L->warm == nullptr)))) {
        set_error(SCOUT_ERR_INVALID_ARGUMENT, "%s: bad tier layer", what);
        return SCOUT_ERR_INVALID_ARGUMENT;
    }
    return SCOUT_OK;
}

}  // namespace

extern "C" int scout_tier_append(const scout_tier_layer* L, int n_units, int nb_stride, const int32_t* n_tokens,
                                 int clock_step, int32_t* open_slot, int32_t* sealed_id, void* stream) {
    int rc = check_layer(L, n_units, nb_stride, "scout_tier_append");
    if (rc != SCOUT_OK || n_units == 0) return rc;
    tier_append_kernel<<<n_units, TT, 0, static_cast<cudaStream_t>(stream)>>>(*L, nb_stride, n_tokens, clock_step,
                                                                              open_slot, sealed_id);
    return scout_host::check_launch("scout_tier_append");
}

extern "C" int scout_tier_apply(const scout_tier_layer* L, int n_units, int nb_stride, const int32_t* n_tokens,
                                int due_tick, int32_t* n_applied, void* stream) {
    int rc = check_layer(L, n_units, nb_stride, "scout_tier_apply");
    if (rc != SCOUT_OK || n_units == 0) return rc;
    tier_apply_kernel<<<n_units, TT, 0, static_cast<cudaStream_t>(stream)>>>(*L, nb_stride, n_tokens, due_tick,
                                                                             n_applied);
    return scout_host::check_launch("scout_tier_apply");
}

extern "C" int scout_tier_schedule_recall(const scout_tier_layer* L, int n_units, int nb_stride,
                                          const int32_t* n_tokens, const int32_t* ids, const int32_t* n_ids,
                                          int k_stride, int ready_tick, int ticket, int32_t* dst_slots, void* stream) {
    int rc = check_layer(L, n_units, nb_stride, "schedule_recall");
    if (rc != SCOUT_OK || n_units == 0) return rc;
    if (!ids || !n_ids || !dst_slots || k_stride <= 0 || ready_tick < 0 || ticket < 0) {
        scout_host::set_error(SCOUT_ERR_INVALID_ARGUMENT, "schedule_recall: bad arguments");
        return SCOUT_ERR_INVALID_ARGUMENT;
    }
    tier_recall_kernel<<<n_units, TT, 0, static_cast<cudaStream_t>(stream)>>>(*L, nb_stride, n_tokens, ids, n_ids,
                                                                              k_stride, ready_tick, ticket, dst_slots);
    return scout_host::check_launch("scout_tier_schedule_recall");
}

extern "C" int scout_tier_plan(const scout_tier_layer* L, int n_units, int nb_stride, const int32_t* n_tokens,
                               int next_tick, int32_t* block_table, void* stream) {
    int rc = check_layer(L, n_units, nb_stride, "residency_set");
    if (rc != SCOUT_OK || n_units == 0) return rc;
    if (!block_table) {
        scout_host::set_error(SCOUT_ERR_INVALID_ARGUMENT, "residency_set: null block table");
        return SCOUT_ERR_INVALID_ARGUMENT;
    }
    tier_plan_kernel<<<n_units, TT, 0, static_cast<cudaStream_t>(stream)>>>(*L, nb_stride, n_tokens, next_tick,
                                                                            block_table);
    return scout_host::check_launch("scout_tier_plan");
}

extern "C" int scout_tier_place(const scout_tier_layer* L, int n_units, int nb_stride, const int32_t* n_tokens,
                                const int32_t* keep, const int32_t* n_keep, int k_stride, int32_t* fill_slots,
                                void* stream) {
    int rc = check_layer(L, n_units, nb_stride, "place_after_prefill");
    if (rc != SCOUT_OK || n_units == 0) return rc;
    if (!keep || !n_keep || k_stride <= 0) {
        scout_host::set_error(SCOUT_ERR_INVALID_ARGUMENT, "place_after_prefill: bad keep list");
        return SCOUT_ERR_INVALID_ARGUMENT;
    }
    tier_place_kernel<<<n_units, TT, 0, static_cast<cudaStream_t>(stream)>>>(*L, nb_stride, n_tokens, keep, n_keep,
                                                                             k_stride, fill_slots);
    return scout_host::check_launch("scout_tier_place");
}

extern "C" int scout_tier_prefill(const scout_tier_layer* L, int n_units, int nb_stride, const int32_t* n_tokens,
                                  int clock_step, const float* k_rows, const float* v_rows, int max_tokens,
                                  void* kv_pool, int kv_dtype, void* digests, void* host_tier, long long host_base,
                                  long long host_blocks, int32_t* blk_slot, void* stream) {
    int rc = check_layer(L, n_units, nb_stride, "prefill");
    if (rc != SCOUT_OK || n_units == 0) return rc;
    if (!n_tokens || !k_rows || !v_rows || !kv_pool || !digests || !blk_slot || max_tokens <= 0 ||
        (kv_dtype != SCOUT_BF16 && kv_dtype != SCOUT_F32)) {
        scout_host::set_error(SCOUT_ERR_INVALID_ARGUMENT, "prefill: bad arguments (bf16 / f32 KV, min/max digests)");
        return SCOUT_ERR_INVALID_ARGUMENT;
    }
    auto st = static_cast<cudaStream_t>(stream);
    tier_prefill_state_kernel<<<n_units, TT, 0, st>>>(*L, nb_stride, n_tokens, max_tokens, clock_step, blk_slot);
    if ((rc = scout_host::check_launch("scout_tier_prefill (state)")) != SCOUT_OK) return rc;
    uint8_t* hv = nullptr;
    if (host_tier) {
        void* d = nullptr;
        if (cudaHostGetDevicePointer(&d, host_tier, 0) == cudaSuccess && d) hv = static_cast<uint8_t*>(d);
        else {
            cudaGetLastError();
            hv = static_cast<uint8_t*>(host_tier);  // device memory
        }
    }
    const int max_blocks = (max_tokens + BS - 1) / BS;
    const dim3 grid(max_blocks < nb_stride ? max_blocks : nb_stride, n_units);
    if (kv_dtype == SCOUT_BF16) {
        tier_prefill_data_kernel<__nv_bfloat16><<<grid, TT, BF16_SLOT_BYTES, st>>>(
            n_tokens, k_rows, v_rows, max_tokens, blk_slot, nb_stride, static_cast<uint8_t*>(kv_pool), digests, hv,
            host_base, host_blocks);
    } else {
        scout_host::ensure_smem(reinterpret_cast<const void*>(tier_prefill_data_kernel<float>), F32_SLOT_BYTES);
        tier_prefill_data_kernel<float><<<grid, TT, F32_SLOT_BYTES, st>>>(
            n_tokens, k_rows, v_rows, max_tokens, blk_slot, nb_stride, static_cast<uint8_t*>(kv_pool), digests, hv,
            host_base, host_blocks);
    }
    return scout_host::check_launch("scout_tier_prefill (data)");
}

extern "C" int scout_tier_mark(const scout_tier_layer* L, int n_units, int nb_stride, const int32_t* ids,
                               const int32_t* n_ids, int k_stride, int step, void* stream) {
    int rc = check_layer(L, n_units, nb_stride, "mark_selected");
    if (rc != SCOUT_OK || n_units == 0) return rc;
    if (!ids || !n_ids || k_stride <= 0) {
        scout_host::set_error(SCOUT_ERR_INVALID_ARGUMENT, "mark_selected: bad id lists");
        return SCOUT_ERR_INVALID_ARGUMENT;
    }
    tier_mark_kernel<<<n_units, TT, 0, static_cast<cudaStream_t>(stream)>>>(*L, nb_stride, ids, n_ids, k_stride, step);
    return scout_host::check_launch("scout_tier_mark");
}

// ===========================================================================
// Engine-internal multi-layer launches (device tier mode, k5_batch.h): the
// per-layer bookkeeping of a whole decode step in two launches instead of
// ~4 per layer (tiny kernels cost ~10 us each behind the persistent K2).
#include "k5_batch.h"

namespace {

// residency_set of every layer (grid units x layers): next run of layer l at step = tick(step, l)
__global__ void __launch_bounds__(TT) tier_plan_layers_kernel(const scout_tier_layer* Ls, int nbs,
                                                              const int32_t* n_tokens, int step, int n_layers,
                                                              int32_t* tables) {
    const int u = blockIdx.x, l = blockIdx.y;
    const scout_tier_layer& L = Ls[l];
    const size_t o = static_cast<size_t>(u) * nbs;
    const int nb = min(n_blocks_of(n_tokens[u]), nbs);
    const int next_tick = step * n_layers + l;
    int32_t* out = tables + static_cast<size_t>(l) * gridDim.x * nbs + o;
    for (int b = threadIdx.x; b < nbs; b += TT) {
        int v = -1;
        if (b < nb) {
            const int r = L.ready[o + b];
            if (L.tier[o + b] || (r >= 0 && r <= next_tick)) v = L.table[o + b];
        }
        out[b] = v;
    }
}

__device__ void post_recall(const TierPostArgs& a, const scout_tier_layer& L, Unit& U, int u, int l, int pos,
                            TierSm& S);

__device__ int find_sorted(const int32_t* v, int n, int x) {
    int lo = 0, hi = n;
    while (lo < hi) {
        const int mid = (lo + hi) >> 1;
        if (v[mid] < x) lo = mid + 1;
        else hi = mid;
    }
    return lo < n && v[lo] == x;
}

// check_split (engine.hpp:317-329) on K1's split of this step: every
// predicted block on exactly one side, the two sides' sizes adding up, and
// the token accounting (resident + CPU rows = the predicted blocks' rows at
// selection time). A violation is the unit's sticky error SCOUT_TIER_ERR_SPLIT.
__device__ void check_split(const TierPostArgs& a, Unit& U, int u, int l, int pos, TierSm& S) {
    const size_t lu = static_cast<size_t>(l) * gridDim.x + u, row = lu * a.k;
    const int ns = a.n_sel[lu], nr = a.n_res[lu], nc = a.n_cpu[lu];
    const int nb = n_blocks_of(pos);
    int bad = 0, tok = 0;
    for (int i = threadIdx.x; i < ns; i += TT) {
        const int b = a.sel_ids[row + i];
        tok += b == nb - 1 ? pos - (nb - 1) * BS : BS;
        if (find_sorted(a.res_ids + row, nr, b) == find_sorted(a.cpu_ids + row, nc, b)) bad = 1;
    }
    bad = block_sum(bad, S);
    tok = block_sum(tok, S);
    if (threadIdx.x == 0 && (bad || nr + nc != ns || tok != a.res_tok[lu] + a.cpu_tok[lu])) set_err(U, SCOUT_TIER_ERR_SPLIT);
}

// After the step's attention, per (unit, layer): append the token (open /
// seal + enforce_capacity, row write, digest fold), write a sealed block
// through to the host tier, and when the layer is due, schedule the recall of
// K1's CPU-side ids (validation, slot assignment). n_tokens is read as the
// count before the append; the caller advances it afterwards.
__global__ void __launch_bounds__(TT) tier_post_layers_kernel(const TierPostArgs a) {
    __shared__ TierSm S;
    __shared__ int s_slot, s_sealed;
    const int u = blockIdx.x, l = a.layer0 + blockIdx.y, c = threadIdx.x;
    const scout_tier_layer& L = a.layers[l];
    Unit U = unit_of(L, u, a.nbs);
    const int pos = a.n_tokens[u];
    const int id = pos / BS, r = pos % BS;
    if (a.res_ids) check_split(a, U, u, l, pos, S);
    // ---- append bookkeeping (tier_append_kernel's logic)
    if (c == 0) {
        S.err = 0;
        if (id >= a.nbs) {
            set_err(U, SCOUT_ERR_INVALID_ARGUMENT);
            S.err = 1;
        } else if (r == 0) {
            const int slot = ring_pop(U);
            if (slot < 0) {
                set_err(U, SCOUT_ERR_LOGIC);
                S.err = 1;
            } else {
                U.table[id] = slot;
                U.tier[id] = 1;
                U.ready[id] = -1;
                U.last_sel[id] = a.step;
            }
        }
        s_slot = S.err ? -1 : U.table[id];
        s_sealed = (!S.err && (pos + 1) % BS == 0) ? id : -1;
    }
    __syncthreads();
    const int slot = s_slot, sealed_blk = s_sealed;
    const size_t sbytes = a.kv_f32 ? F32_SLOT_BYTES : BF16_SLOT_BYTES;
    if (slot >= 0 && a.kv_f32) {
        // ---- row write + digest fold (scout_kv_append, f32 KV: row-major slot, minmax)
        float* base = reinterpret_cast<float*>(a.pool + static_cast<size_t>(slot) * F32_SLOT_BYTES);
        const size_t row = (static_cast<size_t>(l) * gridDim.x + u) * D + c;
        const float v = a.k_new[row];
        base[r * D + c] = v;
        base[BS * D + r * D + c] = a.v_new[row];
        float* dig = static_cast<float*>(a.digests[l]) + static_cast<size_t>(u) * 2 * D * a.nbs;
        float& lo = dig[static_cast<size_t>(c) * a.nbs + id];
        float& hi = dig[static_cast<size_t>(D + c) * a.nbs + id];
        if (r == 0) {
            lo = v;
            hi = v;
        } else {  // std::min / std::max fold (digest.hpp:45-46)
            if (v < lo) lo = v;
            if (hi < v) hi = v;
        }
    } else if (slot >= 0) {
        // ---- row write + digest fold (scout_kv_append, bf16 KV, minmax)
        __nv_bfloat16* base = reinterpret_cast<__nv_bfloat16*>(a.pool + static_cast<size_t>(slot) * BF16_SLOT_BYTES);
        const int off = bf16_tile_offset(r, c);
        const size_t row = (static_cast<size_t>(l) * gridDim.x + u) * D + c;
        const __nv_bfloat16 kq = __float2bfloat16_rn(a.k_new[row]);
        base[off] = kq;
        base[BS * D + off] = __float2bfloat16_rn(a.v_new[row]);
        __nv_bfloat16* dig = static_cast<__nv_bfloat16*>(a.digests[l]) + static_cast<size_t>(u) * 2 * D * a.nbs;
        __nv_bfloat16& lo = dig[static_cast<size_t>(c) * a.nbs + id];
        __nv_bfloat16& hi = dig[static_cast<size_t>(D + c) * a.nbs + id];
        const float v = __bfloat162float(kq);
        if (r == 0) {
            lo = kq;
            hi = kq;
        } else {  // std::min / std::max fold (digest.hpp:45-46)
            const float lf = __bfloat162float(lo), hf = __bfloat162float(hi);
            if (v < lf) lo = kq;
            if (hf < v) hi = kq;
        }
    }
    if (sealed_blk >= 0) {
        // ---- seal: mark, write-through of the block image, enforce capacity
        __syncthreads();  // the row just written belongs to the image
        if (c == 0) U.last_sel[sealed_blk] = a.step;
        if (a.host_tier) {
            long long hi = (static_cast<long long>(l) * a.host_units + a.host_unit0 + u) * a.nbs + sealed_blk;
            if (a.host_blocks > 0) hi %= a.host_blocks;
            const int4* src = reinterpret_cast<const int4*>(a.pool + static_cast<size_t>(slot) * sbytes);
            int4* dst = reinterpret_cast<int4*>(a.host_tier + static_cast<size_t>(hi) * sbytes);
            for (int i = c; i < static_cast<int>(sbytes / 16); i += TT) dst[i] = __ldcg(src + i);
        }
        __syncthreads();
        enforce_capacity(L, U, id + 1, pos + 1, S);
    }
    // ---- periodic recall (engine.hpp:299-307): when the layer is due, the
    // predicted set minus the residency evaluated after this append
    // (maybe_schedule_recall, recall.hpp:114-126), then schedule_recall's
    // validation and slot assignment (tier_recall_kernel's logic)
    if (a.recall_due[l]) {
        __syncthreads();  // the seal's eviction first
        post_recall(a, L, U, u, l, pos, S);
    }
    // ---- the layer's planning view for the next step (tier_plan_layers_kernel's
    // logic): nothing touches this layer's state between here and that step's
    // plan, so the view is the same and the step need not wait for a plan launch
    if (a.plan_out) {
        __syncthreads();  // this CTA's append / seal / eviction / recall writes first
        const size_t o = static_cast<size_t>(u) * a.nbs;
        const int nbn = min(n_blocks_of(pos + 1), a.nbs);
        const int next_tick = a.plan_step * a.n_layers + l;
        int32_t* out = a.plan_out + static_cast<size_t>(l) * gridDim.x * a.nbs + o;
        for (int b = c; b < a.nbs; b += TT) {
            int v = -1;
            if (b < nbn) {
                const int rd = L.ready[o + b];
                if (L.tier[o + b] || (rd >= 0 && rd <= next_tick)) v = L.table[o + b];
            }
            out[b] = v;
        }
    }
}

__device__ void post_recall(const TierPostArgs& a, const scout_tier_layer& L, Unit& U, int u, int l, int pos,
                            TierSm& S) {
    const int c = threadIdx.x, lane = c & 31, w = c >> 5;
    const int ntok = pos + 1;  // after this step's append
    const int nb = min(n_blocks_of(ntok), a.nbs);
    const size_t row = (static_cast<size_t>(l) * gridDim.x + u) * a.k;
    const int32_t* pred = a.sel_ids + row;
    const int np = a.n_sel[static_cast<size_t>(l) * gridDim.x + u];
    int32_t* my = a.rc_ids + row;
    int32_t* dst = a.dst + row;
    // residency_set(l) at clock (step, l): fast blocks plus tickets ready by
    // next_run_of(l) = (step, l) (kv_store.hpp:156-170, 328-331)
    const int next_tick = a.step * a.n_layers + l;
    // set_difference(predicted, residency) in id order: a block-wide
    // order-preserving compaction of the predicted ids that are not resident
    int n = 0;
    for (int base = 0; base < np; base += TT) {
        const int i = base + c;
        int b = -1;
        bool take = false;
        if (i < np) {
            b = pred[i];
            const bool in_range = b >= 0 && b < a.nbs;
            const int rd = in_range ? U.ready[b] : -1;
            take = !in_range || !(U.tier[b] || (rd >= 0 && rd <= next_tick));
        }
        const unsigned bal = __ballot_sync(0xffffffffu, take);
        if (lane == 0) S.cnt[w] = __popc(bal);
        __syncthreads();
        int off = n;
        for (int j = 0; j < w; ++j) off += S.cnt[j];
        int tot = 0;
        for (int j = 0; j < TW; ++j) tot += S.cnt[j];
        if (take) my[off + __popc(bal & ((1u << lane) - 1u))] = b;
        n += tot;
        __syncthreads();
    }
    if (c == 0) a.rc_n[static_cast<size_t>(l) * gridDim.x + u] = n;
    __syncthreads();  // the compacted list
    if (n == 0) return;  // nothing to move (the trigger still resets the cadence, on the host)
    // schedule_recall (kv_store.hpp:175-197): sealed, slow, not in flight, a
    // sorted set; else the unit's whole ticket is rejected
    int bad = 0;
    for (int i = c; i < n; i += TT) {
        const int b = my[i];
        if (b < 0 || b >= nb || !sealed(b, ntok) || U.tier[b] || U.ready[b] >= 0 || (i > 0 && my[i - 1] >= b)) bad = 1;
    }
    bad = block_sum(bad, S);
    if (c == 0) {
        S.err = 0;
        if (bad) {
            set_err(U, SCOUT_ERR_INVALID_ARGUMENT);
            S.err = 1;
        } else if (*U.n_free < n) {
            set_err(U, SCOUT_ERR_LOGIC);
            S.err = 1;
        } else {
            const int hits = assign_recall_slots(U, my, n, dst);
            if (a.rc_stats) {  // warm hits (no bytes) / blocks to copy
                atomicAdd(a.rc_stats, static_cast<unsigned long long>(hits));
                atomicAdd(a.rc_stats + 1, static_cast<unsigned long long>(n - hits));
            }
        }
    }
    __syncthreads();
    for (int i = c; i < n; i += TT) {
        if (S.err) {
            dst[i] = -1;
            continue;
        }
        const int b = my[i];
        U.ready[b] = (a.step + 1) * a.n_layers + l;
        U.ticket[b] = a.ticket_base + l;
    }
}

__global__ void __launch_bounds__(TT) tier_apply_layers_kernel(const TierApplyArgs a) {
    __shared__ TierSm S;
    const int l = a.layer[blockIdx.y];
    apply_unit(a.layers[l], blockIdx.x, a.nbs, a.n_tokens, a.due_tick[blockIdx.y], nullptr, S);
}

// GpuSidePolicy::all_resident (engine.hpp:28-29, 253-256): the on-device
// side of layer l is its whole fast tier at attention time (after
// begin_layer's tickets), residency_set(l) in ascending id order, with each
// block's pool slot. Tier mode reads the K5 state (fast = tier flag; an
// in-flight block already holds its destination slot in `table` but is not
// fast yet); the static mode reads the layer's block table (slot >= 0).
__global__ void __launch_bounds__(TT) tier_resident_lists_kernel(const ResidentListArgs a) {
    __shared__ TierSm S;
    const int u = blockIdx.x, l = a.layer0 + blockIdx.y;
    const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
    const size_t o = static_cast<size_t>(u) * a.nbs;
    const int32_t* table = a.layers ? a.layers[l].table + o : a.tables[l] + o;
    const uint8_t* tier = a.layers ? a.layers[l].tier + o : nullptr;
    const int nb = min(n_blocks_of(a.n_tokens[u]), a.nbs);
    const size_t row = (static_cast<size_t>(l) * gridDim.x + u) * a.stride;
    int total = 0;
    for (int base = 0; base < nb; base += TT) {
        const int b = base + static_cast<int>(threadIdx.x);
        const int slot = b < nb ? table[b] : -1;
        const bool f = b < nb && (tier ? tier[b] != 0 : slot >= 0);
        const unsigned bal = __ballot_sync(0xffffffffu, f);
        if (lane == 0) S.cnt[w] = __popc(bal);
        __syncthreads();
        int off = total, tot = 0;
#pragma unroll
        for (int i = 0; i < TW; ++i) {
            off += i < w ? S.cnt[i] : 0;
            tot += S.cnt[i];
        }
        if (f) {
            const int pos = off + __popc(bal & ((1u << lane) - 1u));
            a.ids[row + pos] = b;
            a.slots[row + pos] = slot;
        }
        total += tot;
        __syncthreads();
    }
    if (threadIdx.x == 0) a.n[static_cast<size_t>(l) * gridDim.x + u] = total;
}

__global__ void advance_tokens_kernel(int32_t* n_tokens, int n) {
    const int i = blockIdx.x * blockDim.x + threadIdx.x;
    if (i < n) n_tokens[i] += 1;
}

}  // namespace

int scout_tier_plan_layers(const scout_tier_layer* layers_dev, int n_layers, int n_units, int nb_stride,
                           const int32_t* n_tokens, int step, int32_t* tables, cudaStream_t st) {
    tier_plan_layers_kernel<<<dim3(n_units, n_layers), TT, 0, st>>>(layers_dev, nb_stride, n_tokens, step, n_layers,
                                                                    tables);
    return scout_host::check_launch("tier plan (all layers)");
}

int scout_tier_post_layers(const TierPostArgs& a, int n_units, int n_layers_launch, cudaStream_t st) {
    tier_post_layers_kernel<<<dim3(n_units, n_layers_launch), TT, 0, st>>>(a);
    return scout_host::check_launch("tier post-attention");
}

int scout_tier_apply_layers(const TierApplyArgs& a, int n_units, cudaStream_t st) {
    if (a.n <= 0) return SCOUT_OK;
    tier_apply_layers_kernel<<<dim3(n_units, a.n), TT, 0, st>>>(a);
    return scout_host::check_launch("tier apply (due layers)");
}

int scout_tier_resident_lists(const ResidentListArgs& a, int n_units, int n_layers_launch, cudaStream_t st) {
    if (n_layers_launch <= 0 || n_units <= 0) return SCOUT_OK;
    tier_resident_lists_kernel<<<dim3(n_units, n_layers_launch), TT, 0, st>>>(a);
    return scout_host::check_launch("resident lists (all_resident)");
}

int scout_tier_advance(int32_t* n_tokens, int n_units, cudaStream_t st) {
    advance_tokens_kernel<<<(n_units + 255) / 256, 256, 0, st>>>(n_tokens, n_units);
    return scout_host::check_launch("advance n_tokens");
}
