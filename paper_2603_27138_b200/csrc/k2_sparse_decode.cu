// K2 (+K3 fused) — paged block-sparse flash-decode over GPU-resident blocks.
//
// Replaces the GPU side of one decode layer in the reference:
//   partial_attention  proj/include/scout/attention.hpp:73-95
//   accumulate_token   attention.hpp:38-50 (online softmax, unnormalised)
//   merge / finalize   attention.hpp:100-122, engine.hpp:271-273
// batched over every (request, KV head) unit of a layer, GQA-grouped: the G
// query heads of a KV head share one pass over its selected K/V blocks (the
// reference, single-head, re-reads K/V per head).
//
// bf16 path (the hot one): one persistent CTA per SM that walks a whole
// decode step's layers (the engine's launch) or one layer (the C ABI):
//   * per layer, work balance ("stream-K"): the concatenation of every unit's
//     resident block list is cut into equal ranges; a range covers pieces
//     ("segments") of one or more units. Segment (cta c, unit u) owns partial
//     slot c+u; the last CTA to finish a unit (atomic counter) LSE-merges the
//     unit's segment partials and the CPU co-attention partial;
//   * a planner/producer warp builds layer L+1's plan while layer L computes
//     (double-buffered) and streams each 32 KiB block with one 1-D bulk copy
//     (TMA engine) into an mbarrier ring that never drains between layers;
//     it waits on device flags for K1's lists (K1 runs concurrently on
//     another stream) and for recalls landed;
//   * six consumer warps (three pairs, one 32-token half each) run both GEMMs
//     on the tensor cores (mma.sync m16n8k16 bf16, fp32 accumulate) in a
//     transposed form that wastes no rows at G=8:
//        S^T[32 tok x 8 heads] = K[32 x 128] . Q^T      (q split hi+lo bf16)
//        O^T[128 x 8 heads]   += V^T[128 x 32] . P^T    (P^T via movmatrix)
//     with the online-softmax state per head in registers (log2 domain).
// f32 path (config 1, CUDA cores): split-K over blocks, 4 warps per CTA, then
// a small combine kernel (same merge rule).
#include "scout_common.cuh"

#include <cstddef>
#include <cstring>

#include <math_constants.h>

using namespace scout_dev;

namespace {

constexpr float LOG2E = 1.4426950408889634f;
constexpr float LN2 = 0.6931471805599453f;

// ------------------------------------------------------------ workspace --
constexpr int HEAD_STRIDE = D + 4;         // per head in a partial slot: o(128), m, l, pad (16B-aligned)
constexpr int PART_STRIDE = 8 * HEAD_STRIDE;  // floats per partial slot: [8 heads]
constexpr int SIMPLE_SPLIT = 8;
constexpr int GRID_CAP = 1024;

__host__ __device__ inline size_t ctr_bytes(int n_units) { return ((static_cast<size_t>(n_units) * 4 + 255) / 256) * 256; }
}  // namespace

#include "k2_step.h"

namespace {

// =========================================================== bf16 kernel ==
namespace tc {
// One stage = one whole 32 KiB block (K tile then V tile): a single bulk copy,
// the transfer size at which random gathers get the most out of HBM3e
// (tools/microbench/gather.cu: 2x8 KiB 5.1, 16 KiB 5.9, 32 KiB 6.7 TB/s).
// Consumer warps work in pairs: warp 2p+h takes 32-token half h of every
// block j (CTA-global stream index, continuing across layers) with
// j % NPAIR == p; pair p double-buffers its own stages p and p + NPAIR, so
// every stage is filled and drained in order by one pair.
constexpr int NPAIR = 3;
constexpr int NC = 2 * NPAIR;               // consumer warps
constexpr int NCT = NC * 32;                // consumer threads
constexpr int NCOMB = 2;                    // combiner warps (segments alternate between them)
constexpr int NTHREADS = NCT + 32 * (2 + NCOMB);  // + producer, planner and combiner warps
constexpr int NST = 2 * NPAIR;              // ring stages
constexpr int STAGE_BYTES = 32768;          // one block: K tile (16 KiB) + V tile (16 KiB)
#ifndef SCOUT_K2_NPLAN
#define SCOUT_K2_NPLAN 2
#endif
#ifndef SCOUT_K2_MAXSEG
#define SCOUT_K2_MAXSEG 64
#endif
#ifndef SCOUT_K2_MAXB
#define SCOUT_K2_MAXB 384
#endif
constexpr int NPLAN = SCOUT_K2_NPLAN;       // plan chunk buffers (the planner runs NPLAN - 1 chunks ahead)
constexpr int MAXSEG = SCOUT_K2_MAXSEG;     // segments per plan chunk
constexpr int MAXB = SCOUT_K2_MAXB;         // blocks per plan chunk
constexpr int CB_ROW = D;  // combine rows (no pad: the conflicted state stores are once per segment)
constexpr size_t SMEM_BYTES = static_cast<size_t>(NST) * STAGE_BYTES;

// A segment piece: blocks [j0, j1) of unit `unit`'s resident list. A CTA's
// segment of a unit that does not fit the rest of a plan chunk is split over
// consecutive chunks; the consumers carry its softmax state in registers from
// a piece marked SEG_CONT_NEXT to the next one (marked SEG_CONT_PREV).
constexpr int SEG_CONT_PREV = 1, SEG_CONT_NEXT = 2;
struct Seg {
    int unit, j0, j1, nseg, cfirst, f0;  // f0: first block of the piece in the chunk's block list
    int cont;
};

// One plan chunk: a piece of this CTA's share of one layer (at most MAXSEG
// segment pieces and MAXB blocks; a layer's share is one or more chunks, so a
// range of any length or unit count is planned whole). Built by the planner
// warp ahead of the consumers (double-buffered).
constexpr int ZMAX = 16;
constexpr int NR_REG = 16;  // resident counts the planner holds in registers per lane (512 units)  // units without a resident block this CTA finalizes, listed in the plan
constexpr int CH_FIRST = 1, CH_LAST = 2;  // first / last chunk of its layer
// A plan entry packs the pool slot (< 2^26: 2 TiB of 32 KiB slots, more than
// any device holds) with the block's valid rows - 1 (0..63).
constexpr int BLK_ROWS_SHIFT = 26;
constexpr uint32_t BLK_SLOT_MASK = (1u << BLK_ROWS_SHIFT) - 1u;
__device__ __forceinline__ size_t blk_slot(uint32_t e) { return e & BLK_SLOT_MASK; }
__device__ __forceinline__ int blk_rows(uint32_t e) { return static_cast<int>(e >> BLK_ROWS_SHIFT) + 1; }
struct Plan {
    Seg segs[MAXSEG];
    uint32_t blk[MAXB];      // resident blocks in stream order: pool slot | (valid rows - 1) << 26
    int zero_units[ZMAX];    // first chunk: units u == blockIdx.x (mod grid) with no resident block
    int nsegs, nblk, jbase, nzero;  // nzero > ZMAX: scan n_res instead
    int layer, flags;
};

struct Smem {
    uint64_t full[NST];
    uint64_t empty[NST];
    uint64_t plan_full[NPLAN];
    uint64_t plan_empty[NPLAN];
    uint64_t seg_full[NCOMB];  // the NC consumer warps left a segment's states (segment s: combiner s % NCOMB)
    uint64_t seg_empty;        // its combiner has read them
    int layer_fin[K2_MAX_LAYERS];  // combiners done with layer L (the last one counts the CTA in)
    Plan plan[NPLAN];
    int warp_area[NC];   // 1: the warp left a state in wstate, -1: no state
    // per-warp segment states (o^T rows, m, l), merged by the combiner warp
    // while the consumers go on with the next segment
    alignas(16) float wstate[NC][8 * CB_ROW + 16];
};

__device__ __forceinline__ int stage_of(int j) { return (j % NPAIR) + NPAIR * ((j / NPAIR) & 1); }

__device__ __forceinline__ unsigned ld_acquire(const unsigned* p) {
    unsigned v;
    asm volatile("ld.acquire.gpu.global.u32 %0, [%1];" : "=r"(v) : "l"(p) : "memory");
    return v;
}
// Spin until *p >= token (wrap-safe). A flag that never arrives (a producer
// that cannot be scheduled) traps after 10 s instead of hanging the device.
__device__ __forceinline__ void wait_flag(const unsigned* p, unsigned token) {
    if (p == nullptr) return;
    if (static_cast<int>(ld_acquire(p) - token) >= 0) return;
    const unsigned long long t0 = global_ns();
    while (static_cast<int>(ld_acquire(p) - token) < 0) {
        __nanosleep(256);
        if (global_ns() - t0 > 10000000000ull) __trap();
    }
}

// Merge n partial slots (+ the optional CPU partial) of unit u into the
// outputs (merge / finalize, attention.hpp:100-122; both empty -> zeros,
// engine.hpp:273). NT threads cover 8 heads x 32 lanes x 4 channels.
template <int G, int NT>
__device__ void finalize_unit(const float* cpu_o, const float* cpu_ml, float* out_o, float* out_ml, int u,
                              const float* parts, int first_slot, int nslots, int ctid) {
    for (int idx = ctid; idx < 8 * 32; idx += NT) {
        const int h = idx >> 5;
        const int d0 = (idx & 31) * 4;
        if (h >= G) continue;
        const size_t head = static_cast<size_t>(u) * G + h;
        float M = -CUDART_INF_F;
        for (int i = 0; i < nslots; ++i) {
            const float* p = parts + static_cast<size_t>(first_slot + i) * PART_STRIDE + h * HEAD_STRIDE;
            M = fmaxf(M, __ldcg(p + D));
        }
        float cm = -CUDART_INF_F, cl = 0.f;
        if (cpu_ml) {
            cm = cpu_ml[head * 2] * LOG2E;
            cl = cpu_ml[head * 2 + 1];
            if (cl > 0.f) M = fmaxf(M, cm);
        }
        float4 acc = make_float4(0.f, 0.f, 0.f, 0.f);
        float L = 0.f;
        if (M != -CUDART_INF_F) {
            for (int i = 0; i < nslots; ++i) {
                const float* p = parts + static_cast<size_t>(first_slot + i) * PART_STRIDE + h * HEAD_STRIDE;
                const float l = __ldcg(p + D + 1);
                if (!(l > 0.f)) continue;
                const float w = l * exp2f(__ldcg(p + D) - M);
                L += w;
                const float4 x = __ldcg(reinterpret_cast<const float4*>(p + d0));
                acc.x += w * x.x; acc.y += w * x.y; acc.z += w * x.z; acc.w += w * x.w;
            }
            if (cl > 0.f) {
                const float w = cl * exp2f(cm - M);
                L += w;
                const float4 co = *reinterpret_cast<const float4*>(cpu_o + head * D + d0);
                acc.x += w * co.x; acc.y += w * co.y; acc.z += w * co.z; acc.w += w * co.w;
            }
        }
        const float inv = L > 0.f ? 1.f / L : 0.f;
        *reinterpret_cast<float4*>(out_o + head * D + d0) = make_float4(acc.x * inv, acc.y * inv, acc.z * inv, acc.w * inv);
        if ((idx & 31) == 0) {
            out_ml[head * 2] = L > 0.f ? M * LN2 : -CUDART_INF_F;
            out_ml[head * 2 + 1] = L;
        }
    }
}

// four channels d0..d0+3 of a CPU-partial row, f32 or bf16
__device__ __forceinline__ float4 load_co(const void* cpu_o, size_t off, bool bf16) {
    if (bf16) {
        const uint2 w = *reinterpret_cast<const uint2*>(static_cast<const __nv_bfloat16*>(cpu_o) + off);
        return make_float4(__uint_as_float(w.x << 16), __uint_as_float(w.x & 0xFFFF0000u), __uint_as_float(w.y << 16),
                           __uint_as_float(w.y & 0xFFFF0000u));
    }
    return *reinterpret_cast<const float4*>(static_cast<const float*>(cpu_o) + off);
}

// finalize_unit for one warp (the combiner): lane owns channels 4*lane.. of
// every head, and each phase issues all of its loads before using them, so a
// unit costs ~2 L2 round trips per partial slot rather than one per head.
template <int G>
__device__ void finalize_unit_warp(const void* cpu_o, bool co_bf16, const float* cpu_ml, float* out_o, float* out_ml,
                                   int u, const float* parts, int first_slot, int nslots, int lane) {
    const int d0 = lane * 4;
    float M[G], cm[G], cl[G], L[G];
    float4 acc[G];
#pragma unroll
    for (int h = 0; h < G; ++h) {
        M[h] = -CUDART_INF_F; cm[h] = -CUDART_INF_F; cl[h] = 0.f; L[h] = 0.f;
        acc[h] = make_float4(0.f, 0.f, 0.f, 0.f);
    }
    if (cpu_ml) {
#pragma unroll
        for (int h = 0; h < G; ++h) {
            const size_t head = static_cast<size_t>(u) * G + h;
            cm[h] = cpu_ml[head * 2] * LOG2E;
            cl[h] = cpu_ml[head * 2 + 1];
        }
    }
    for (int i = 0; i < nslots; ++i) {
        const float* p = parts + static_cast<size_t>(first_slot + i) * PART_STRIDE;
#pragma unroll
        for (int h = 0; h < G; ++h) M[h] = fmaxf(M[h], __ldcg(p + h * HEAD_STRIDE + D));
    }
#pragma unroll
    for (int h = 0; h < G; ++h)
        if (cl[h] > 0.f) M[h] = fmaxf(M[h], cm[h]);
    for (int i = 0; i < nslots; ++i) {
        const float* p = parts + static_cast<size_t>(first_slot + i) * PART_STRIDE;
        float pm[G], pl[G];
        float4 px[G];
#pragma unroll
        for (int h = 0; h < G; ++h) {
            pm[h] = __ldcg(p + h * HEAD_STRIDE + D);
            pl[h] = __ldcg(p + h * HEAD_STRIDE + D + 1);
            px[h] = __ldcg(reinterpret_cast<const float4*>(p + h * HEAD_STRIDE + d0));
        }
#pragma unroll
        for (int h = 0; h < G; ++h) {
            if (M[h] == -CUDART_INF_F || !(pl[h] > 0.f)) continue;
            const float w = pl[h] * exp2f(pm[h] - M[h]);
            L[h] += w;
            acc[h].x += w * px[h].x; acc[h].y += w * px[h].y; acc[h].z += w * px[h].z; acc[h].w += w * px[h].w;
        }
    }
    if (cpu_ml) {
        float4 co[G];
#pragma unroll
        for (int h = 0; h < G; ++h)
            co[h] = load_co(cpu_o, (static_cast<size_t>(u) * G + h) * D + d0, co_bf16);
#pragma unroll
        for (int h = 0; h < G; ++h) {
            if (M[h] == -CUDART_INF_F || !(cl[h] > 0.f)) continue;
            const float w = cl[h] * exp2f(cm[h] - M[h]);
            L[h] += w;
            acc[h].x += w * co[h].x; acc[h].y += w * co[h].y; acc[h].z += w * co[h].z; acc[h].w += w * co[h].w;
        }
    }
#pragma unroll
    for (int h = 0; h < G; ++h) {
        const size_t head = static_cast<size_t>(u) * G + h;
        const float inv = L[h] > 0.f ? 1.f / L[h] : 0.f;
        *reinterpret_cast<float4*>(out_o + head * D + d0) =
            make_float4(acc[h].x * inv, acc[h].y * inv, acc[h].z * inv, acc[h].w * inv);
        if (lane == 0) {
            out_ml[head * 2] = L[h] > 0.f ? M[h] * LN2 : -CUDART_INF_F;
            out_ml[head * 2 + 1] = L[h];
        }
    }
}

// ---------------------------------------------------------------- planner
// The plan buffer of chunk c, once every role has released its previous use.
__device__ __forceinline__ Plan& plan_acquire(Smem& sm, int c, long long& waited, bool prof) {
    const long long t0 = prof ? clock64() : 0;
    if (c >= NPLAN) mbar_wait(&sm.plan_empty[c % NPLAN], ((c / NPLAN) - 1) & 1);
    if (prof) waited += clock64() - t0;
    return sm.plan[c % NPLAN];
}

// Finish chunk c (its segment pieces are written): pull the query rows of the
// segments starting here into L2, fill the block list (pool slot, valid rows)
// and publish it to the producer, consumers and combiners.
template <typename Args>
__device__ void plan_publish(const Args& a, const K2Layer& io, Smem& sm, int c, int nseg, int nblk, int jbase,
                             int layer, int flags, int lane) {
    Plan& P = sm.plan[c % NPLAN];
    __syncwarp();  // lane 0's segment records
    {
        const int qbytes = a.group * D * (a.q_bf16 ? 2 : 4);
        const int lines = (qbytes + 127) / 128;
        for (int i = lane; i < nseg * lines; i += 32) {
            const int si = i / lines, li = i % lines;
            if (P.segs[si].cont & SEG_CONT_PREV) continue;
            const uint8_t* qp = static_cast<const uint8_t*>(io.q) +
                                static_cast<size_t>(P.segs[si].unit) * qbytes + static_cast<size_t>(li) * 128;
            asm volatile("prefetch.global.L2 [%0];" ::"l"(qp));
        }
    }
    // four blocks per lane per round, their loads in flight together (the
    // producer waits for this list)
    constexpr int PB = 4;
    for (int f0 = 0; f0 < nblk; f0 += 32 * PB) {
        int unit[PB], slot[PB], rid[PB], nt[PB];
#pragma unroll
        for (int r = 0; r < PB; ++r) {
            const int f = f0 + 32 * r + lane;
            unit[r] = -1;
            if (f >= nblk) continue;
            int lo = 0, hi = nseg - 1;  // the last piece with f0 <= f (f0 ascending)
            while (lo < hi) {
                const int mid = (lo + hi + 1) >> 1;
                if (P.segs[mid].f0 <= f) lo = mid;
                else hi = mid - 1;
            }
            const Seg sg = P.segs[lo];
            const size_t idx = static_cast<size_t>(sg.unit) * a.k_stride + sg.j0 + (f - sg.f0);
            unit[r] = sg.unit;
            slot[r] = __ldcg(io.res_slots + idx);
            rid[r] = __ldcg(io.res_ids + idx);
            nt[r] = __ldcg(a.n_tokens + sg.unit);
        }
#pragma unroll
        for (int r = 0; r < PB; ++r) {
            if (unit[r] < 0) continue;
            const int nb = (nt[r] + BS - 1) / BS;
            const int rows = (rid[r] == nb - 1) ? nt[r] - (nb - 1) * BS : BS;  // the open block's fill
            P.blk[f0 + 32 * r + lane] = static_cast<uint32_t>(slot[r]) | (static_cast<uint32_t>(rows - 1) << BLK_ROWS_SHIFT);
        }
    }
    if (lane == 0) {
        P.nsegs = nseg;
        P.nblk = nblk;
        P.jbase = jbase;
        P.layer = layer;
        P.flags = flags;
    }
    __syncwarp();
    if (lane == 0) mbar_arrive(&sm.plan_full[c % NPLAN]);
}

// Planner (one warp): this CTA's share of layer `layer`'s resident blocks, as
// one or more plan chunks (c: chunk counter, j: CTA-global block stream index).
// Stream-K: the concatenation of every unit's resident block list is cut into
// geff = min(grid, T) equal ranges (every range non-empty, so a unit's segment
// count is the number of CTAs between the ones holding its first and last
// block); segment (cta c, unit u) owns partial slot c+u. A range may touch any
// number of units and hold any number of blocks: pieces go into chunks of at
// most MAXSEG pieces / MAXB blocks, a segment split at a chunk boundary.
template <typename Args>
__device__ void plan_layer(const Args& a, const K2Layer& io, Smem& sm, int layer, int& c, int& j, int lane,
                           long long& waited) {
    const int nunits = a.n_units;
    // the units' resident counts: up to 32 * NR_REG units are loaded once, all
    // loads in flight together (one dependent round trip per pass instead of
    // one per 32 units: a single-layer launch waits for its plan)
    int nr[NR_REG];
    const bool cached = nunits <= 32 * NR_REG;
    if (cached) {
#pragma unroll
        for (int i = 0; i < NR_REG; ++i) {
            const int u = 32 * i + lane;
            nr[i] = u < nunits ? __ldcg(io.n_res + u) : 0;
        }
    }
    auto n_res_of = [&](int base) -> int {
        if (cached) {
            int v = 0;
#pragma unroll
            for (int i = 0; i < NR_REG; ++i)
                if (32 * i == base) v = nr[i];
            return v;
        }
        const int u = base + lane;
        return u < nunits ? io.n_res[u] : 0;
    };
    Plan* P = &plan_acquire(sm, c, waited, a.prof != nullptr);
    long long T = 0;
    {
        int loc = 0, nz = 0;
        for (int base = 0; base < nunits; base += 32) {
            const int u = base + lane;
            const int n = n_res_of(base);
            loc += n;
            // units with no resident block that this CTA finalizes (CPU partial or zeros)
            const bool z = u < nunits && n == 0 && u % static_cast<int>(gridDim.x) == static_cast<int>(blockIdx.x);
            const unsigned bz = __ballot_sync(0xffffffffu, z);
            const int pos = nz + __popc(bz & ((1u << lane) - 1u));
            if (z && pos < ZMAX) P->zero_units[pos] = u;
            nz += __popc(bz);
        }
        if (lane == 0) P->nzero = nz;
#pragma unroll
        for (int o = 16; o; o >>= 1) loc += __shfl_xor_sync(0xffffffffu, loc, o);
        T = loc;
    }
    const long long grid = T < static_cast<long long>(gridDim.x) ? (T > 0 ? T : 1) : gridDim.x;
    const long long cta = blockIdx.x;
    const long long lo = cta < grid ? T * cta / grid : T, hi = cta < grid ? T * (cta + 1) / grid : T;
    long long run = 0;
    int nseg = 0, nblk = 0, jb = j, first = CH_FIRST;
    for (int base = 0; base < nunits && run < hi; base += 32) {
        const int n = n_res_of(base);
        int incl = n;
#pragma unroll
        for (int o = 1; o < 32; o <<= 1) {
            const int y = __shfl_up_sync(0xffffffffu, incl, o);
            if (lane >= o) incl += y;
        }
        const long long pre = run + incl - n;
        const long long s0 = max(pre, lo), s1 = min(pre + n, hi);
        const bool has = n > 0 && s0 < s1;
        int my_j0 = 0, my_j1 = 0, my_nseg = 0, my_cf = 0;
        if (has) {
            my_j0 = static_cast<int>(s0 - pre);
            my_j1 = static_cast<int>(s1 - pre);
            const long long cf = ((pre + 1) * grid - 1) / T;  // CTA holding position p: floor(((p+1)*grid-1)/T)
            const long long cl = ((pre + n) * grid - 1) / T;
            my_nseg = static_cast<int>(cl - cf + 1);
            my_cf = static_cast<int>(cf);
        }
        unsigned bal = __ballot_sync(0xffffffffu, has);
        while (bal) {  // this CTA's segments of the 32 units, in unit order
            const int src = __ffs(bal) - 1;
            bal &= bal - 1;
            int j0 = __shfl_sync(0xffffffffu, my_j0, src);
            const int j1 = __shfl_sync(0xffffffffu, my_j1, src);
            const int ns = __shfl_sync(0xffffffffu, my_nseg, src);
            const int cf = __shfl_sync(0xffffffffu, my_cf, src);
            int cont = 0;
            while (j0 < j1) {
                if (nseg == MAXSEG || nblk == MAXB) {  // chunk full: publish, continue in the next
                    plan_publish(a, io, sm, c, nseg, nblk, jb, layer, first, lane);
                    ++c;
                    first = 0;
                    jb += nblk;
                    nseg = nblk = 0;
                    P = &plan_acquire(sm, c, waited, a.prof != nullptr);
                    if (lane == 0) P->nzero = 0;
                }
                const int take = min(j1 - j0, MAXB - nblk);
                if (lane == 0)
                    P->segs[nseg] = Seg{base + src, j0, j0 + take, ns, cf, nblk, cont | (take < j1 - j0 ? SEG_CONT_NEXT : 0)};
                ++nseg;
                nblk += take;
                j0 += take;
                cont = SEG_CONT_PREV;
            }
        }
        run += __shfl_sync(0xffffffffu, incl, 31);
    }
    plan_publish(a, io, sm, c, nseg, nblk, jb, layer, first | CH_LAST, lane);
    ++c;
    j = jb + nblk;
}

// Register cap: a warp's registers come from its SM sub-partition's 16K file
// (warp w -> SMSP w % 4), and with nine or ten warps SMSP 0 hosts three. At
// the 168 registers ptxas picks by itself, SMSP 0 had 256 registers left and
// no 4-warp kernel (the tier bookkeeping that runs beside K2 on the post
// stream) could launch next to K2 until it exited: the recalls then landed a
// step late and K2 waited for them (tier mode 6.05 -> 7.1 ms per step). 144
// leaves room for two 32-register warps on SMSP 0 and does not spill.
template <int G, int NL>
__global__ void __maxnreg__(144) sparse_decode_tc_kernel(const K2StepArgsT<NL> a) {
    extern __shared__ __align__(1024) uint8_t dsmem[];
    __shared__ Smem sm;
    uint8_t* stages = dsmem;

    const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
    const int nunits = a.n_units;

    for (int i = tid; i < K2_MAX_LAYERS; i += NTHREADS) sm.layer_fin[i] = 0;
    if (tid == 0) {
        for (int i = 0; i < NST; ++i) {
            mbar_init(&sm.full[i], 1);
            mbar_init(&sm.empty[i], 2);  // both warps of the owning pair release
        }
        for (int i = 0; i < NPLAN; ++i) {
            mbar_init(&sm.plan_full[i], 1);
            mbar_init(&sm.plan_empty[i], NC + 1 + NCOMB);  // every consumer warp, the producer and the combiners
        }
        for (int i = 0; i < NCOMB; ++i) mbar_init(&sm.seg_full[i], NC);
        mbar_init(&sm.seg_empty, 1);
        fence_mbar_init();
    }
    // PDL (single-layer launches): inputs from the preceding kernel are
    // complete past this point
    griddep_wait();
    griddep_launch_dependents();
    __syncthreads();

    if (warp == NC + 1) {
        // ======================================== planner warp: layer L's plan
        // while the producer still streams layer L-1 (a plan costs a few
        // dependent global round trips: inline in the producer it left the
        // ring draining at every layer boundary, ~20% at config 2)
        int j = 0;  // CTA-global block stream index (continues across layers)
        int c = 0;  // plan chunk counter (continues across layers)
        long long w_empty = 0, w_plan = 0, tq = 0;  // SCOUT_K2_PROF: waiting for a free plan buffer, planning
        for (int L = 0; L < a.n_layers; ++L) {
            const K2Layer& io = a.layers[L];
            if (a.prof) tq = clock64();
            if (lane == 0) {
                // K1 published layer L's lists / the layer's inputs landed
                if (a.k1_flag) wait_flag(a.k1_flag + L, a.token);
                if (io.in_flag) wait_flag(io.in_flag, a.token);
            }
            __syncwarp();
            plan_layer(a, io, sm, L, c, j, lane, w_empty);
            if (a.prof) w_plan += clock64() - tq;
        }
        w_plan -= w_empty;
        if (a.prof && lane == 0) {
            unsigned long long* pr = a.prof + blockIdx.x * 16;
            atomicAdd(pr + 10, static_cast<unsigned long long>(w_empty));
            atomicAdd(pr + 11, static_cast<unsigned long long>(w_plan));
        }
        return;
    }
    if (warp == NC) {
        // ======================================== producer warp (lane 0)
        if (lane != 0) return;
        const uint64_t pol = policy_evict_first();
        const uint8_t* pool = static_cast<const uint8_t*>(a.kv_pool);
        int j = 0;
        long long t_plan = 0, t_empty = 0;  // SCOUT_K2_PROF: cycles blocked on a plan / a free stage
        const long long t_start = clock64();
        for (int c = 0;; ++c) {
            const int b = c % NPLAN;
            long long t0 = a.prof ? clock64() : 0;
            mbar_wait(&sm.plan_full[b], (c / NPLAN) & 1);
            const int L = sm.plan[b].layer, fl = sm.plan[b].flags;
            const K2Layer& io = a.layers[L];
            // blocks recalled for this layer one step ago must have landed
            if ((fl & CH_FIRST) && io.recall_token && a.recall_flag) wait_flag(a.recall_flag + L, io.recall_token);
            if (a.prof) t_plan += clock64() - t0;
            const int nblk = sm.plan[b].nblk;
            // L2 prefetch runs K2_PF blocks ahead of the ring: the ring's 6
            // stages alone keep ~4 us of this SM's share of HBM bandwidth in
            // flight, which the loaded latency eats (SCOUT_K2_PROF: producer on
            // a full ring while the consumers wait for data)
            const int pf = a.l2_prefetch;
            for (int f = 0; f < min(pf, nblk); ++f)
                bulk_prefetch_l2(pool + blk_slot(sm.plan[b].blk[f]) * BF16_SLOT_BYTES, STAGE_BYTES);
            for (int f = 0; f < nblk; ++f, ++j) {
                const int s = stage_of(j);
                if (f + pf < nblk)
                    bulk_prefetch_l2(pool + blk_slot(sm.plan[b].blk[f + pf]) * BF16_SLOT_BYTES,
                                     STAGE_BYTES);
                if (a.prof) t0 = clock64();
                if (j >= NST) mbar_wait(&sm.empty[s], ((j / NST) - 1) & 1);
                if (a.prof) t_empty += clock64() - t0;
                mbar_arrive_expect_tx(&sm.full[s], STAGE_BYTES);
                bulk_g2s_evict_first(stages + s * STAGE_BYTES,
                                     pool + blk_slot(sm.plan[b].blk[f]) * BF16_SLOT_BYTES,
                                     STAGE_BYTES, &sm.full[s], pol);
            }
            mbar_arrive(&sm.plan_empty[b]);  // the producer is done reading this plan
            if ((fl & CH_LAST) && L == a.n_layers - 1) break;
        }
        if (a.prof) {
            unsigned long long* pr = a.prof + blockIdx.x * 16;
            atomicAdd(pr + 0, static_cast<unsigned long long>(clock64() - t_start));
            atomicAdd(pr + 1, static_cast<unsigned long long>(t_plan));
            atomicAdd(pr + 2, static_cast<unsigned long long>(t_empty));
            atomicAdd(pr + 3, static_cast<unsigned long long>(j));
        }
        return;
    }

    if (warp >= NC + 2) {
        // ======================================== combiner warps: each merges
        // every NCOMB-th segment's NC warp states and writes the unit's output
        // (nseg == 1) or its partial (+ the cross-CTA finalize when last), off
        // the consumers' path; they share the units without a resident block,
        // and the last to finish a layer counts the CTA in. One combiner kept
        // up at config 3 but not where segments are short (config 2: busy 81%,
        // consumers waiting for it 19% of their time)
        const int cw = warp - (NC + 2);
        long long k_wait = 0, k_busy = 0, tq = 0;
        int segidx = 0;  // segments flushed by the consumers (pieces ending one)
        for (int c = 0;; ++c) {
            const int b = c % NPLAN;
            mbar_wait(&sm.plan_full[b], (c / NPLAN) & 1);
            const Plan& P = sm.plan[b];
            const int L = P.layer, fl = P.flags;
            const K2Layer& io = a.layers[L];
            int* ctr = reinterpret_cast<int*>(static_cast<uint8_t*>(a.workspace) + static_cast<size_t>(L) * a.ws_layer_bytes);
            float* parts = reinterpret_cast<float*>(reinterpret_cast<uint8_t*>(ctr) + ctr_bytes(nunits));
            for (int si = 0; si < P.nsegs; ++si) {
                if (P.segs[si].cont & SEG_CONT_NEXT) continue;  // the segment goes on in the next chunk
                if (segidx++ % NCOMB != cw) continue;
                const Seg sg = P.segs[si];
                const int u = sg.unit;
                if (a.prof) tq = clock64();
                mbar_wait(&sm.seg_full[cw], ((segidx - 1) / NCOMB) & 1);
                if (a.prof) { const long long t1 = clock64(); k_wait += t1 - tq; tq = t1; }
                // lane: channels 4*lane..4*lane+3 of every head
                const int d0 = lane * 4;
                float Ms[G], Ls[G];
                float4 accs[G];
#pragma unroll
                for (int hh = 0; hh < G; ++hh) {  // heads >= G carry nothing
                    float M = -CUDART_INF_F;
#pragma unroll
                    for (int w = 0; w < NC; ++w)
                        if (sm.warp_area[w] >= 0) M = fmaxf(M, sm.wstate[w][8 * CB_ROW + hh]);
                    float Lsum = 0.f;
                    float4 acc = make_float4(0.f, 0.f, 0.f, 0.f);
#pragma unroll
                    for (int w = 0; w < NC; ++w) {
                        if (sm.warp_area[w] < 0) continue;
                        const float* wb = sm.wstate[w];
                        const float l = wb[8 * CB_ROW + 8 + hh];
                        if (!(l > 0.f)) continue;
                        const float fct = exp2f(wb[8 * CB_ROW + hh] - M);
                        Lsum += l * fct;
                        const float4 x = *reinterpret_cast<const float4*>(wb + hh * CB_ROW + d0);
                        acc.x += fct * x.x; acc.y += fct * x.y; acc.z += fct * x.z; acc.w += fct * x.w;
                    }
                    Ms[hh] = M; Ls[hh] = Lsum; accs[hh] = acc;
                }
                __syncwarp();
                if (lane == 0) mbar_arrive(&sm.seg_empty);  // states read: the consumers may overwrite them
                // the unit's CPU partial, all heads' loads in flight at once (nseg == 1)
                float cms[G], cls[G];
                float4 cos_[G];
#pragma unroll
                for (int hh = 0; hh < G; ++hh) {
                    cms[hh] = -CUDART_INF_F; cls[hh] = 0.f; cos_[hh] = make_float4(0.f, 0.f, 0.f, 0.f);
                    if (sg.nseg == 1 && io.cpu_ml) {
                        const size_t head = static_cast<size_t>(u) * G + hh;
                        cms[hh] = io.cpu_ml[head * 2] * LOG2E;
                        cls[hh] = io.cpu_ml[head * 2 + 1];
                        cos_[hh] = load_co(io.cpu_o, head * D + d0, a.cpu_bf16 != 0);
                    }
                }
#pragma unroll
                for (int hh = 0; hh < G; ++hh) {
                    const float M = Ms[hh], Lsum = Ls[hh];
                    const float4 acc = accs[hh];
                    const float inv = Lsum > 0.f ? 1.f / Lsum : 0.f;
                    if (sg.nseg == 1) {
                        // the whole unit is here: merge with the CPU partial and write out
                        const size_t head = static_cast<size_t>(u) * G + hh;
                        const float cm = cms[hh], cl = cls[hh];
                        float Mt = M, wa = 1.f, wb = 0.f, Lt = Lsum;
                        if (cl > 0.f) {
                            Mt = fmaxf(M, cm);
                            wa = Lsum > 0.f ? exp2f(M - Mt) : 0.f;
                            wb = cl * exp2f(cm - Mt);
                            Lt = Lsum * wa + wb;
                        }
                        const float invt = Lt > 0.f ? 1.f / Lt : 0.f;
                        float4 res;
                        if (cl > 0.f) {
                            const float4 co = cos_[hh];
                            res = make_float4((acc.x * wa + wb * co.x) * invt, (acc.y * wa + wb * co.y) * invt,
                                              (acc.z * wa + wb * co.z) * invt, (acc.w * wa + wb * co.w) * invt);
                        } else {
                            res = make_float4(acc.x * inv, acc.y * inv, acc.z * inv, acc.w * inv);
                        }
                        *reinterpret_cast<float4*>(io.o + head * D + d0) = res;
                        if (lane == 0) {
                            io.ml[head * 2] = Lt > 0.f ? Mt * LN2 : -CUDART_INF_F;
                            io.ml[head * 2 + 1] = Lt;
                        }
                    } else {
                        // this segment's partial (o normalised, m2, l) -> slot c+u
                        float* p = parts + (static_cast<size_t>(blockIdx.x) + u) * PART_STRIDE + hh * HEAD_STRIDE;
                        *reinterpret_cast<float4*>(p + d0) =
                            make_float4(acc.x * inv, acc.y * inv, acc.z * inv, acc.w * inv);
                        if (lane == 0) { p[D] = M; p[D + 1] = Lsum; }
                    }
                }
                if (sg.nseg != 1) {
                    // publish the partial: __syncwarp orders the lanes' stores
                    // before lane 0's gpu-scope fence, which precedes the counter
                    __syncwarp();
                    int last = 0;
                    if (lane == 0) {
                        __threadfence();
                        const int old = atomicAdd(&ctr[u], 1);
                        last = old == sg.nseg - 1;
                        if (last) __threadfence();  // acquire: the other segments' partials are visible
                    }
                    last = __shfl_sync(0xffffffffu, last, 0);
                    if (last) {
                        // last CTA for unit u: its segments are CTAs cfirst..cfirst+nseg-1 at slots c+u
                        // (partials read with ld.global.cg: L2, never a stale L1 line)
                        finalize_unit_warp<G>(io.cpu_o, a.cpu_bf16 != 0, io.cpu_ml, io.o, io.ml, u, parts, sg.cfirst + u, sg.nseg, lane);
                        if (lane == 0) ctr[u] = 0;  // leave the counter zeroed for the next launch
                    }
                }
                if (a.prof) k_busy += clock64() - tq;
            }
            if (a.prof) tq = clock64();
            // ---- units with no resident block: output = CPU partial (or empty),
            // listed by the planner in the layer's first chunk (no n_res read on this path)
            if (!(fl & CH_FIRST)) {
            } else if (P.nzero <= ZMAX) {
                for (int i = cw; i < P.nzero; i += NCOMB)
                    finalize_unit_warp<G>(io.cpu_o, a.cpu_bf16 != 0, io.cpu_ml, io.o, io.ml, P.zero_units[i], parts, 0, 0, lane);
            } else {
                for (int u = blockIdx.x + cw * gridDim.x; u < nunits; u += NCOMB * gridDim.x) {
                    if (io.n_res[u] != 0) continue;
                    finalize_unit_warp<G>(io.cpu_o, a.cpu_bf16 != 0, io.cpu_ml, io.o, io.ml, u, parts, 0, 0, lane);
                }
            }
            // done with layer L: release the plan buffer; the last combiner counts
            // the CTA in. Each orders its lanes' outputs (__syncwarp) before its
            // gpu-scope fence, the fence before its shared-memory count, and the
            // last one's fence after that count precedes the layer counter.
            __syncwarp();
            if (lane == 0) {
                mbar_arrive(&sm.plan_empty[b]);
                if ((fl & CH_LAST) && a.layer_done) {
                    __threadfence();
                    if (atomicAdd(&sm.layer_fin[L], 1) == NCOMB - 1) {
                        __threadfence();
                        atomicAdd(a.layer_done + L, 1u + (blockIdx.x == 0 ? a.done_extra : 0u));
                    }
                }
            }
            if (a.prof) k_busy += clock64() - tq;
            if ((fl & CH_LAST) && L == a.n_layers - 1) break;
        }
        if (a.prof && lane == 0) {
            unsigned long long* pr = a.prof + blockIdx.x * 16;
            atomicAdd(pr + 8, static_cast<unsigned long long>(k_wait));
            atomicAdd(pr + 9, static_cast<unsigned long long>(k_busy));
        }
        return;
    }

    // ====================================================== consumer warps
    const int g = lane >> 2, t = lane & 3;
    const int pair = warp >> 1, hsel = warp & 1;
    const float sl2 = a.scale * LOG2E;
    // SCOUT_K2_PROF: cycles waiting for data, loading Q, in segment ends, on plans / layer ends
    long long c_full = 0, c_q = 0, c_end = 0, c_plan = 0, tp = 0;
    int segidx = 0;  // CTA-global count of flushed segments (the state buffer's phase)
    // one segment's state; a segment split over plan chunks keeps it across them
    uint32_t bh[8][2], bl[8][2];  // Q^T fragments (hi/lo split), heads >= G are zero
    float m2[2] = {-CUDART_INF_F, -CUDART_INF_F};
    float lp[2] = {0.f, 0.f};
    float oacc[8][4];
    int held = -1;  // stage of the pair's last block: handed back at the next block or the segment end
    bool any = false;
    for (int c = 0;; ++c) {
        const int b = c % NPLAN;
        if (a.prof) tp = clock64();
        mbar_wait(&sm.plan_full[b], (c / NPLAN) & 1);
        if (a.prof) c_plan += clock64() - tp;
        const Plan& P = sm.plan[b];
        const int nsegs = P.nsegs, jbase = P.jbase, L = P.layer, fl = P.flags;
        const K2Layer& io = a.layers[L];
        for (int si = 0; si < nsegs; ++si) {
            const Seg sg = P.segs[si];
            const int u = sg.unit;
            if (!(sg.cont & SEG_CONT_PREV)) {
                if (a.prof) tp = clock64();
                const bool live = g < G;
                const size_t qoff = (static_cast<size_t>(u) * G + (live ? g : 0)) * D;
                if (a.q_bf16) {  // the query is bf16 already: lo part zero
                    const uint32_t* qb = reinterpret_cast<const uint32_t*>(static_cast<const __nv_bfloat16*>(io.q) + qoff);
#pragma unroll
                    for (int kk = 0; kk < 8; ++kk)
#pragma unroll
                        for (int half = 0; half < 2; ++half) {
                            bh[kk][half] = live ? qb[(16 * kk + 8 * half + 2 * t) >> 1] : 0u;
                            bl[kk][half] = 0u;
                        }
                } else {
                    const float* qh = static_cast<const float*>(io.q) + qoff;
#pragma unroll
                    for (int kk = 0; kk < 8; ++kk) {
#pragma unroll
                        for (int half = 0; half < 2; ++half) {
                            float2 v = live ? *reinterpret_cast<const float2*>(qh + 16 * kk + 8 * half + 2 * t)
                                            : make_float2(0.f, 0.f);
                            const __nv_bfloat162 hv = __floats2bfloat162_rn(v.x, v.y);
                            const float2 hf = __bfloat1622float2(hv);
                            bh[kk][half] = *reinterpret_cast<const uint32_t*>(&hv);
                            bl[kk][half] = pack_bf16(v.x - hf.x, v.y - hf.y);
                        }
                    }
                }
                if (a.prof) { __syncwarp(); c_q += clock64() - tp; }
                m2[0] = m2[1] = -CUDART_INF_F;
                lp[0] = lp[1] = 0.f;
#pragma unroll
                for (int i = 0; i < 8; ++i) oacc[i][0] = oacc[i][1] = oacc[i][2] = oacc[i][3] = 0.f;
                held = -1;
                any = false;
            }

            const int f1 = sg.f0 + (sg.j1 - sg.j0);
            const int jf0 = jbase + sg.f0;
            for (int f = sg.f0 + ((pair - jf0) % NPAIR + NPAIR) % NPAIR; f < f1; f += NPAIR) {
                if (held >= 0) {  // the pair's previous block is done: hand its stage back
                    __syncwarp();
                    if (lane == 0) mbar_arrive(&sm.empty[held]);
                }
                const int jj = jbase + f;
                const int s = stage_of(jj);
                held = s;
                const int valid = min(HALF_ROWS, blk_rows(P.blk[f]) - hsel * HALF_ROWS);
                if (a.prof) tp = clock64();
                mbar_wait(&sm.full[s], (jj / NST) & 1);
                __syncwarp();  // lanes may leave the try_wait loop apart: reconverge before .aligned ops
                if (a.prof) c_full += clock64() - tp;
                if (valid <= 0) continue;  // open block with one half: the other warp idles
                any = true;
                const uint32_t kbase = smem_u32(stages + s * STAGE_BYTES) + hsel * HALF_BYTES_BF16;
                const uint32_t vbase = kbase + BF16_TILE_BYTES;
                if (valid < HALF_ROWS) {
                    // rows past the open block's fill hold stale bytes: P is 0
                    // there, but 0 * NaN would poison O, so zero those V rows.
                    for (int i = lane; i < (HALF_ROWS - valid) * 16; i += 32) {
                        const int row = valid + (i >> 4), chunk = i & 15;
                        const uint32_t addr = vbase + (chunk >> 3) * 4096 + row * 128 + ((chunk & 7) << 4);
                        asm volatile("st.shared.v4.u32 [%0], {%1, %1, %1, %1};" ::"r"(addr), "r"(0) : "memory");
                    }
                    __syncwarp();
                }
                // ---- S^T = K . Q^T (hi and lo halves of q accumulate separately)
                float sh[2][4] = {{0, 0, 0, 0}, {0, 0, 0, 0}}, slo[2][4] = {{0, 0, 0, 0}, {0, 0, 0, 0}};
#pragma unroll
                for (int kk = 0; kk < 8; ++kk) {
                    const int slab = kk >> 2, cb = (kk & 3) * 2;
#pragma unroll
                    for (int mt = 0; mt < 2; ++mt) {
                        const int row = 16 * mt + (lane & 7) + ((lane >> 3) & 1) * 8;
                        const int chunk = cb + (lane >> 4);
                        const uint32_t addr = kbase + slab * 4096 + row * 128 + ((chunk ^ (row & 7)) << 4);
                        uint32_t a0, a1, a2, a3;
                        ldsm_x4(addr, a0, a1, a2, a3);
                        mma_bf16(sh[mt], a0, a1, a2, a3, bh[kk][0], bh[kk][1]);
                        if (!a.q_bf16) mma_bf16(slo[mt], a0, a1, a2, a3, bl[kk][0], bl[kk][1]);
                    }
                }
                // ---- online softmax (columns = heads 2t, 2t+1; rows = tokens)
                float sv[2][4];
                float mx0 = -CUDART_INF_F, mx1 = -CUDART_INF_F;
#pragma unroll
                for (int mt = 0; mt < 2; ++mt) {
                    const int r0 = 16 * mt + g, r1 = r0 + 8;
                    sv[mt][0] = r0 < valid ? (sh[mt][0] + slo[mt][0]) * sl2 : -CUDART_INF_F;
                    sv[mt][1] = r0 < valid ? (sh[mt][1] + slo[mt][1]) * sl2 : -CUDART_INF_F;
                    sv[mt][2] = r1 < valid ? (sh[mt][2] + slo[mt][2]) * sl2 : -CUDART_INF_F;
                    sv[mt][3] = r1 < valid ? (sh[mt][3] + slo[mt][3]) * sl2 : -CUDART_INF_F;
                    mx0 = fmaxf(mx0, fmaxf(sv[mt][0], sv[mt][2]));
                    mx1 = fmaxf(mx1, fmaxf(sv[mt][1], sv[mt][3]));
                }
#pragma unroll
                for (int o = 4; o < 32; o <<= 1) {
                    mx0 = fmaxf(mx0, __shfl_xor_sync(0xffffffffu, mx0, o));
                    mx1 = fmaxf(mx1, __shfl_xor_sync(0xffffffffu, mx1, o));
                }
                const float mn0 = fmaxf(m2[0], mx0), mn1 = fmaxf(m2[1], mx1);
                const float al0 = fast_exp2(m2[0] - mn0), al1 = fast_exp2(m2[1] - mn1);
                m2[0] = mn0;
                m2[1] = mn1;
                float ps0 = 0.f, ps1 = 0.f;
                uint32_t pb[2][2];
#pragma unroll
                for (int mt = 0; mt < 2; ++mt) {
                    const float p0 = fast_exp2(sv[mt][0] - mn0), p1 = fast_exp2(sv[mt][1] - mn1);
                    const float p2 = fast_exp2(sv[mt][2] - mn0), p3 = fast_exp2(sv[mt][3] - mn1);
                    ps0 += p0 + p2;
                    ps1 += p1 + p3;
                    pb[mt][0] = movmatrix_t(pack_bf16(p0, p1));
                    pb[mt][1] = movmatrix_t(pack_bf16(p2, p3));
                }
                lp[0] = lp[0] * al0 + ps0;
                lp[1] = lp[1] * al1 + ps1;
#pragma unroll
                for (int md = 0; md < 8; ++md) {
                    oacc[md][0] *= al0; oacc[md][1] *= al1; oacc[md][2] *= al0; oacc[md][3] *= al1;
                }
                // ---- O^T += V^T . P^T
#pragma unroll
                for (int md = 0; md < 8; ++md) {
#pragma unroll
                    for (int kk = 0; kk < 2; ++kk) {
                        const int row = 16 * kk + (lane & 7) + ((lane >> 4) & 1) * 8;
                        const int cg = 2 * md + ((lane >> 3) & 1);
                        const uint32_t addr = vbase + (cg >> 3) * 4096 + row * 128 + (((cg & 7) ^ (row & 7)) << 4);
                        uint32_t a0, a1, a2, a3;
                        ldsm_x4_t(addr, a0, a1, a2, a3);
                        mma_bf16(oacc[md], a0, a1, a2, a3, pb[kk][0], pb[kk][1]);
                    }
                }
            }
            if (sg.cont & SEG_CONT_NEXT) continue;  // the segment goes on in the next chunk
            if (a.prof) tp = clock64();
            // ---- warp state -> the combiner; the stage goes back right away
#pragma unroll
            for (int o = 4; o < 32; o <<= 1) {
                lp[0] += __shfl_xor_sync(0xffffffffu, lp[0], o);
                lp[1] += __shfl_xor_sync(0xffffffffu, lp[1], o);
            }
            __syncwarp();
            const int area = (held >= 0 && any) ? 1 : -1;
            if (held >= 0 && lane == 0) mbar_arrive(&sm.empty[held]);  // all lanes are past their last ldmatrix
            held = -1;
            // the combiner has read the previous segment's states
            if (segidx > 0) mbar_wait(&sm.seg_empty, (segidx - 1) & 1);
            if (area >= 0) {
                float* cb = sm.wstate[warp];
#pragma unroll
                for (int md = 0; md < 8; ++md) {
                    cb[(2 * t) * CB_ROW + 16 * md + g] = oacc[md][0];
                    cb[(2 * t + 1) * CB_ROW + 16 * md + g] = oacc[md][1];
                    cb[(2 * t) * CB_ROW + 16 * md + g + 8] = oacc[md][2];
                    cb[(2 * t + 1) * CB_ROW + 16 * md + g + 8] = oacc[md][3];
                }
                if (g == 0) {
                    cb[8 * CB_ROW + 2 * t] = m2[0];
                    cb[8 * CB_ROW + 2 * t + 1] = m2[1];
                    cb[8 * CB_ROW + 8 + 2 * t] = lp[0];
                    cb[8 * CB_ROW + 8 + 2 * t + 1] = lp[1];
                }
            }
            if (lane == 0) sm.warp_area[warp] = area;
            __syncwarp();  // every lane's state stores before lane 0's (release) arrive
            if (lane == 0) mbar_arrive(&sm.seg_full[segidx % NCOMB]);
            ++segidx;
            if (a.prof) c_end += clock64() - tp;
        }
        // this warp is done with the chunk's plan
        __syncwarp();
        if (lane == 0) mbar_arrive(&sm.plan_empty[b]);
        if ((fl & CH_LAST) && L == a.n_layers - 1) break;
    }
    if (a.prof && lane == 0) {
        unsigned long long* pr = a.prof + blockIdx.x * 16;
        atomicAdd(pr + 4, static_cast<unsigned long long>(c_full));
        atomicAdd(pr + 5, static_cast<unsigned long long>(c_q));
        atomicAdd(pr + 6, static_cast<unsigned long long>(c_end));
        atomicAdd(pr + 7, static_cast<unsigned long long>(c_plan));
    }
}

}  // namespace tc

// ========================================================= f32 kernel ====
// CUDA-core split-K path (f32 KV, config 1). CTA (unit, split) handles blocks
// j = split, split+SIMPLE_SPLIT, ...; warp w handles tokens r = w, w+4, ...;
// lane owns channels 4*lane .. 4*lane+3.
namespace simple {
constexpr int NW = 4;

template <int G>
__global__ void __launch_bounds__(NW * 32) decode_f32_kernel(const scout_decode_args a) {
    __shared__ float sm_o[NW][G][D];
    __shared__ float sm_ml[NW][G][2];
    const int u = blockIdx.x, split = blockIdx.y;
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    const int ks = a.k_stride;
    const int nres = a.n_res[u];
    const int nt = a.n_tokens[u];
    const int nb = (nt + BS - 1) / BS, tail = nt - (nb - 1) * BS;
    const float sl2 = a.scale * LOG2E;
    float qv[G][4];
#pragma unroll
    for (int g = 0; g < G; ++g) {
        const float4 x = *reinterpret_cast<const float4*>(static_cast<const float*>(a.q) + (static_cast<size_t>(u) * G + g) * D + 4 * lane);
        qv[g][0] = x.x; qv[g][1] = x.y; qv[g][2] = x.z; qv[g][3] = x.w;
    }
    float m2[G], l[G], o[G][4];
#pragma unroll
    for (int g = 0; g < G; ++g) {
        m2[g] = -CUDART_INF_F; l[g] = 0.f;
        o[g][0] = o[g][1] = o[g][2] = o[g][3] = 0.f;
    }
    const uint8_t* pool = static_cast<const uint8_t*>(a.kv_pool);
    for (int j = split; j < nres; j += SIMPLE_SPLIT) {
        const size_t slot = static_cast<size_t>(a.res_slots[static_cast<size_t>(u) * ks + j]);
        const int id = a.res_ids[static_cast<size_t>(u) * ks + j];
        const int rows = (id == nb - 1) ? tail : BS;
        const float* kt = reinterpret_cast<const float*>(pool + slot * F32_SLOT_BYTES);
        const float* vt = kt + BS * D;
        for (int r = warp; r < rows; r += NW) {
            const float4 k4 = *reinterpret_cast<const float4*>(kt + r * D + 4 * lane);
            const float4 v4 = *reinterpret_cast<const float4*>(vt + r * D + 4 * lane);
#pragma unroll
            for (int g = 0; g < G; ++g) {
                float s = qv[g][0] * k4.x + qv[g][1] * k4.y + qv[g][2] * k4.z + qv[g][3] * k4.w;
#pragma unroll
                for (int off = 16; off; off >>= 1) s += __shfl_xor_sync(0xffffffffu, s, off);
                s *= sl2;
                const float mn = fmaxf(m2[g], s);
                const float al = exp2f(m2[g] - mn), p = exp2f(s - mn);
                m2[g] = mn;
                l[g] = l[g] * al + p;
                o[g][0] = o[g][0] * al + p * v4.x;
                o[g][1] = o[g][1] * al + p * v4.y;
                o[g][2] = o[g][2] * al + p * v4.z;
                o[g][3] = o[g][3] * al + p * v4.w;
            }
        }
    }
#pragma unroll
    for (int g = 0; g < G; ++g) {
        *reinterpret_cast<float4*>(&sm_o[warp][g][4 * lane]) = make_float4(o[g][0], o[g][1], o[g][2], o[g][3]);
        if (lane == 0) { sm_ml[warp][g][0] = m2[g]; sm_ml[warp][g][1] = l[g]; }
    }
    __syncthreads();
    // combine the NW warps -> partial (o normalised, m2, l) for (unit, split)
    float* parts = reinterpret_cast<float*>(static_cast<uint8_t*>(a.workspace) + ctr_bytes(a.n_units));
    float* p = parts + (static_cast<size_t>(u) * SIMPLE_SPLIT + split) * PART_STRIDE;
    for (int i = threadIdx.x; i < G * D; i += NW * 32) {
        const int g = i / D, d = i % D;
        float M = -CUDART_INF_F;
        for (int w = 0; w < NW; ++w) M = fmaxf(M, sm_ml[w][g][0]);
        float L = 0.f, acc = 0.f;
        for (int w = 0; w < NW; ++w) {
            if (!(sm_ml[w][g][1] > 0.f)) continue;
            const float f = exp2f(sm_ml[w][g][0] - M);
            L += sm_ml[w][g][1] * f;
            acc += sm_o[w][g][d] * f;
        }
        p[g * HEAD_STRIDE + d] = L > 0.f ? acc / L : 0.f;
        if (d == 0) { p[g * HEAD_STRIDE + D] = M; p[g * HEAD_STRIDE + D + 1] = L; }
    }
}

template <int G>
__global__ void combine_kernel(const scout_decode_args a) {
    const int u = blockIdx.x;
    const float* parts = reinterpret_cast<const float*>(static_cast<const uint8_t*>(a.workspace) + ctr_bytes(a.n_units));
    tc::finalize_unit<G, 128>(a.cpu_o, a.cpu_ml, a.o, a.ml, u, parts, u * SIMPLE_SPLIT, SIMPLE_SPLIT, threadIdx.x);
}
}  // namespace simple

int num_sms() {
    static int n = 0;
    if (n == 0) {
        int dev = 0;
        cudaGetDevice(&dev);
        cudaDeviceGetAttribute(&n, cudaDevAttrMultiProcessorCount, dev);
        if (n <= 0) n = 148;
    }
    return n;
}

int tc_grid(int max_ctas) {
    int g = max_ctas > 0 ? max_ctas : num_sms();
    return g > GRID_CAP ? GRID_CAP : g;
}

}  // namespace

int scout_k2_grid(int n_units, int k_stride, int max_ctas) {
    // persistent: at most one CTA per SM (a CTA's range of any size is planned
    // in chunks, so neither the unit count nor the list length raises the grid)
    (void)n_units;
    (void)k_stride;
    return tc_grid(max_ctas);
}

size_t scout_k2_ws_layer_bytes(int n_units, int grid) {
    const size_t slots = static_cast<size_t>(grid) + static_cast<size_t>(n_units);
    return ((ctr_bytes(n_units) + slots * PART_STRIDE * sizeof(float)) + 255) / 256 * 256;
}

int scout_k2_launch(const K2StepArgs& a, cudaStream_t st, bool pdl) {
    using namespace scout_host;
    if (a.n_layers < 1 || a.n_layers > K2_MAX_LAYERS) {
        set_error(SCOUT_ERR_INVALID_ARGUMENT, "K2: n_layers %d out of range (max %d)", a.n_layers, K2_MAX_LAYERS);
        return SCOUT_ERR_INVALID_ARGUMENT;
    }
    const int grid = scout_k2_grid(a.n_units, a.k_stride, a.max_ctas);
    if (a.group != 1 && a.group != 2 && a.group != 4 && a.group != 8) {
        set_error(SCOUT_ERR_INVALID_ARGUMENT, "K2: group %d not in {1,2,4,8}", a.group);
        return SCOUT_ERR_INVALID_ARGUMENT;
    }
    auto go = [&](auto kern, const auto& args) {
        ensure_smem(reinterpret_cast<const void*>(kern), tc::SMEM_BYTES);
        launch(kern, dim3(grid), dim3(tc::NTHREADS), tc::SMEM_BYTES, st, pdl, args);
    };
    if (a.n_layers == 1) {  // the 1-slot parameter block
        static thread_local K2StepArgsT<1> a1;
        std::memcpy(&a1, &a, offsetof(K2StepArgs, layers));
        a1.layers[0] = a.layers[0];
        switch (a.group) {
            case 1: go(tc::sparse_decode_tc_kernel<1, 1>, a1); break;
            case 2: go(tc::sparse_decode_tc_kernel<2, 1>, a1); break;
            case 4: go(tc::sparse_decode_tc_kernel<4, 1>, a1); break;
            default: go(tc::sparse_decode_tc_kernel<8, 1>, a1); break;
        }
    } else {
        switch (a.group) {
            case 1: go(tc::sparse_decode_tc_kernel<1, K2_MAX_LAYERS>, a); break;
            case 2: go(tc::sparse_decode_tc_kernel<2, K2_MAX_LAYERS>, a); break;
            case 4: go(tc::sparse_decode_tc_kernel<4, K2_MAX_LAYERS>, a); break;
            default: go(tc::sparse_decode_tc_kernel<8, K2_MAX_LAYERS>, a); break;
        }
    }
    return check_launch("scout_sparse_decode");
}

extern "C" int scout_sparse_decode_grid(int n_units, int k_stride, int max_ctas) {
    return scout_k2_grid(n_units, k_stride, max_ctas);
}

extern "C" size_t scout_sparse_decode_workspace_bytes(int n_units, int group, int max_ctas) {
    (void)group;
    (void)max_ctas;
    if (n_units < 0) return 0;
    const size_t g = GRID_CAP;  // covers any grid scout_k2_grid can pick
    const size_t slots_tc = g + static_cast<size_t>(n_units);
    const size_t slots_simple = static_cast<size_t>(n_units) * SIMPLE_SPLIT;
    const size_t slots = slots_tc > slots_simple ? slots_tc : slots_simple;
    return ctr_bytes(n_units) + slots * PART_STRIDE * sizeof(float);
}

extern "C" int scout_sparse_decode(const scout_decode_args* args, void* stream) {
    using namespace scout_host;
    if (!args) {
        set_error(SCOUT_ERR_INVALID_ARGUMENT, "scout_sparse_decode: null args");
        return SCOUT_ERR_INVALID_ARGUMENT;
    }
    const scout_decode_args& a = *args;
    if (a.n_units < 0 || a.k_stride <= 0) {
        set_error(SCOUT_ERR_INVALID_ARGUMENT, "scout_sparse_decode: bad n_units %d / k_stride %d", a.n_units,
                  a.k_stride);
        return SCOUT_ERR_INVALID_ARGUMENT;
    }
    if (!(a.scale > 0.f)) {
        set_error(SCOUT_ERR_INVALID_ARGUMENT, "partial_attention: scale must be > 0");
        return SCOUT_ERR_INVALID_ARGUMENT;
    }
    if (a.group != 1 && a.group != 2 && a.group != 4 && a.group != 8) {
        set_error(SCOUT_ERR_INVALID_ARGUMENT, "scout_sparse_decode: group %d not in {1,2,4,8}", a.group);
        return SCOUT_ERR_INVALID_ARGUMENT;
    }
    if (a.q_dtype != SCOUT_F32 && !(a.q_dtype == SCOUT_BF16 && a.kv_dtype == SCOUT_BF16)) {
        set_error(SCOUT_ERR_INVALID_ARGUMENT, "scout_sparse_decode: q dtype %d unsupported with kv dtype %d",
                  a.q_dtype, a.kv_dtype);
        return SCOUT_ERR_INVALID_ARGUMENT;
    }
    if (a.n_units == 0) return SCOUT_OK;
    if (!a.q || !a.kv_pool || !a.res_slots || !a.res_ids || !a.n_res || !a.n_tokens || !a.o || !a.ml ||
        !a.workspace || ((a.cpu_o == nullptr) != (a.cpu_ml == nullptr))) {
        set_error(SCOUT_ERR_INVALID_ARGUMENT, "scout_sparse_decode: null buffer");
        return SCOUT_ERR_INVALID_ARGUMENT;
    }
    if (a.workspace_bytes < scout_sparse_decode_workspace_bytes(a.n_units, a.group, a.max_ctas)) {
        set_error(SCOUT_ERR_INVALID_ARGUMENT, "scout_sparse_decode: workspace too small (%zu < %zu)",
                  a.workspace_bytes, scout_sparse_decode_workspace_bytes(a.n_units, a.group, a.max_ctas));
        return SCOUT_ERR_INVALID_ARGUMENT;
    }
    auto st = static_cast<cudaStream_t>(stream);
    if (a.kv_dtype == SCOUT_BF16) {
        K2StepArgs k{};
        k.n_units = a.n_units;
        k.group = a.group;
        k.k_stride = a.k_stride;
        k.n_layers = 1;
        k.scale = a.scale;
        k.kv_pool = a.kv_pool;
        k.n_tokens = a.n_tokens;
        k.workspace = a.workspace;
        k.ws_layer_bytes = a.workspace_bytes;
        k.max_ctas = a.max_ctas;
        k.q_bf16 = a.q_dtype == SCOUT_BF16;
        k.layers[0] = K2Layer{a.q, a.res_slots, a.res_ids, a.n_res, a.cpu_o, a.cpu_ml, a.o, a.ml, nullptr, 0u, 0u};
        return scout_k2_launch(k, st, (a.flags & SCOUT_LAUNCH_PDL) != 0);
    } else if (a.kv_dtype == SCOUT_F32) {
        const dim3 grid(a.n_units, SIMPLE_SPLIT);
        switch (a.group) {
            case 1: simple::decode_f32_kernel<1><<<grid, simple::NW * 32, 0, st>>>(a);
                    simple::combine_kernel<1><<<a.n_units, 128, 0, st>>>(a); break;
            case 2: simple::decode_f32_kernel<2><<<grid, simple::NW * 32, 0, st>>>(a);
                    simple::combine_kernel<2><<<a.n_units, 128, 0, st>>>(a); break;
            case 4: simple::decode_f32_kernel<4><<<grid, simple::NW * 32, 0, st>>>(a);
                    simple::combine_kernel<4><<<a.n_units, 128, 0, st>>>(a); break;
            default: simple::decode_f32_kernel<8><<<grid, simple::NW * 32, 0, st>>>(a);
                     simple::combine_kernel<8><<<a.n_units, 128, 0, st>>>(a); break;
        }
    } else {
        set_error(SCOUT_ERR_UNSUPPORTED, "scout_sparse_decode: kv dtype %d unsupported", a.kv_dtype);
        return SCOUT_ERR_UNSUPPORTED;
    }
    return check_launch("scout_sparse_decode");
}

