// K1 — block scoring + deterministic top-k + resident/CPU split.
//
// Replaces, per (request, KV-head) unit of one layer:
//   digest_score   reference proj/include/scout/digest.hpp:62-72
//   select_topk    digest.hpp:101-118 (score desc, then id asc; ids ascending;
//                  k == 0 rejected at :103)
//   the split      engine.hpp:238-242 = set_intersection / set_difference
//                  (digest.hpp:77-87) against residency_set (kv_store.hpp:156)
//   mark_selected  kv_store.hpp:222-228
//
// Bit-exactness. The reference sums in double, sequentially,
// from +0.0. For f32 queries against f32/bf16 digests every product q*lo / q*hi
// is exact in double (24+24 < 53 significand bits), so
//   s += max(q*lo, q*hi)  ==  s = fma(q, q >= 0 ? hi : lo, s)
// bit for bit; one thread owns one block's whole sum, in the reference's
// (stacked, channel-major) order. The generic f64 path (arbitrary doubles,
// the C++ drop-in wrapper) uses explicit __dmul_rn / __dadd_rn so nothing is
// contracted. Selection is a radix select over an order-preserving 64-bit
// image of the score (-0.0 folded onto +0.0, as the reference's != / >
// comparisons do), with equal scores ranked by block id through a block scan.
#include "scout_common.cuh"

#include <cstdlib>
#include <type_traits>

using namespace scout_dev;

namespace {

// 128 threads, ~30 KB of shared memory, 72 registers: 7 CTAs per SM. Many
// small CTAs hide the latency-bound selection phases best; a deeper digest ring
// costs more (fewer CTAs) than it buys (64-layer batch, tools/gpu/k1_sweep.sh:
// 2 x 8 KiB 0.78 ms, 1 x 16 KiB 0.78, 3 x 8 KiB 0.86, 2 x 32 KiB 1.16)
#ifndef SCOUT_K1_THREADS
#define SCOUT_K1_THREADS 128
#endif
#ifndef SCOUT_K1_MINB
#define SCOUT_K1_MINB 4
#endif
constexpr int K1_THREADS = SCOUT_K1_THREADS;
static_assert(K1_THREADS >= 128, "one thread per channel when staging the query sums");
constexpr int K1_MAXBUF = 4;                    // digest chunk buffers (bulk-copy ring), runtime depth <= this
constexpr int K1_CHUNK_BYTES = 8192;            // lo + hi rows of one chunk (default; SCOUT_K1_CHUNK)
constexpr int K1_REG_BLOCKS = 16 * K1_THREADS;  // nb_stride up to this: running scores live in registers
                                                // (up to 4 block quads per thread)

// qs [D*G] f64 | pn [D] float2 | keys [nbs] u64 | cls [nbs] u8 | (nbs > K1_REG_BLOCKS:
// s_acc [nbs] f64 | a_acc [nbs] f32) | digest chunk ring (MODE 0)
__host__ __device__ inline size_t k1_stage_offset(int G, int nbs) {
    size_t head = static_cast<size_t>(D) * G * 8 + static_cast<size_t>(D) * 8 + static_cast<size_t>(nbs) * 9;
    head = (head + 15) / 16 * 16;
    if (nbs > K1_REG_BLOCKS) head += static_cast<size_t>(nbs) * 12;
    return (head + 127) / 128 * 128;
}
__host__ __device__ inline size_t k1_chunk_bytes(int nbs, int esz, int chunk) {
    // the chunk is at least one channel of lo + hi rows
    const size_t one = static_cast<size_t>(nbs) * 2 * esz;
    return one > static_cast<size_t>(chunk) ? one : chunk;
}
__host__ __device__ inline size_t k1_smem_bytes(int G, int nbs, int esz, int nbuf, int chunk) {
    return k1_stage_offset(G, nbs) + nbuf * k1_chunk_bytes(nbs, esz, chunk);
}

}  // namespace

#include "k1_batch.h"

namespace {
constexpr int K1_WARPS = K1_THREADS / 32;

__device__ __forceinline__ uint64_t score_key(double s) {
    if (s == 0.0) s = 0.0;  // fold -0.0 onto +0.0
    const uint64_t u = static_cast<uint64_t>(__double_as_longlong(s));
    return (u >> 63) ? ~u : (u | 0x8000000000000000ull);
}

__device__ __forceinline__ double ref_max(double a, double b) { return (a < b) ? b : a; }  // std::max

template <typename T>
__device__ __forceinline__ double widen(T x);
template <>
__device__ __forceinline__ double widen<__nv_bfloat16>(__nv_bfloat16 x) {
    return static_cast<double>(__bfloat162float(x));
}
template <>
__device__ __forceinline__ double widen<float>(float x) {
    return static_cast<double>(x);
}

// Block-wide exclusive scan of one int per thread; returns the prefix and
// writes the total to *total. All threads must call.
__device__ int block_exclusive_scan(int v, int* warp_tot, int* total) {
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    int x = v;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
        const int y = __shfl_up_sync(0xffffffffu, x, o);
        if (lane >= o) x += y;
    }
    if (lane == 31) warp_tot[warp] = x;
    __syncthreads();
    if (warp == 0) {
        int t = lane < K1_WARPS ? warp_tot[lane] : 0;
#pragma unroll
        for (int o = 1; o < 32; o <<= 1) {
            const int y = __shfl_up_sync(0xffffffffu, t, o);
            if (lane >= o) t += y;
        }
        if (lane < K1_WARPS) warp_tot[lane] = t;  // inclusive
    }
    __syncthreads();
    const int before = (warp == 0 ? 0 : warp_tot[warp - 1]) + x - v;
    *total = warp_tot[K1_WARPS - 1];
    __syncthreads();
    return before;
}

// ------------------------------------------------------------- scoring --
// Exact reference-order score of one block (MODE 0): fma chain over the
// stacked vector, channel-major (digest.hpp:62-72 on q_s[c*G+g]).
template <typename DigT, int G>
__device__ __forceinline__ double exact_score_minmax(const DigT* lo, const DigT* hi, size_t ns, int b,
                                                     const double* qs) {
    // the chain is sequential, its operands are not: each chunk's 2 x XC
    // digest words are loaded together, so the chain waits on memory once
    // per chunk instead of once per channel (the rare exact path of a near
    // tie was ~30 us per block, the straggler of a single-layer launch)
    constexpr int XC = 8;
    double acc = 0.0;
#pragma unroll 1
    for (int c0 = 0; c0 < D; c0 += XC) {
        DigT L[XC], H[XC];
#pragma unroll
        for (int i = 0; i < XC; ++i) {
            L[i] = lo[(c0 + i) * ns + b];
            H[i] = hi[(c0 + i) * ns + b];
        }
#pragma unroll
        for (int i = 0; i < XC; ++i) {
            const double l = widen(L[i]), h = widen(H[i]);
#pragma unroll
            for (int g = 0; g < G; ++g) {
                const double qv = qs[(c0 + i) * G + g];
                acc = fma(qv, qv >= 0.0 ? h : l, acc);
            }
        }
    }
    return acc;
}

// Generic f64 paths (the drop-in wrapper): exact, no contraction.
template <int G, int MODE>
__device__ __forceinline__ double exact_score_f64(const double* dig, size_t ns, int b, const double* qs) {
    double acc = 0.0;
    if constexpr (MODE == 1) {
        const double* lo = dig;
        const double* hi = dig + D * ns;
        for (int c = 0; c < D; ++c) {
            const double l = lo[c * ns + b], h = hi[c * ns + b];
#pragma unroll
            for (int g = 0; g < G; ++g) {
                const double qv = qs[c * G + g];
                acc = __dadd_rn(acc, ref_max(__dmul_rn(qv, l), __dmul_rn(qv, h)));
            }
        }
    } else {
        for (int c = 0; c < D; ++c) {
            const double m = dig[c * ns + b];
#pragma unroll
            for (int g = 0; g < G; ++g) acc = __dadd_rn(acc, __dmul_rn(qs[c * G + g], m));
        }
    }
    return acc;
}

__device__ __forceinline__ double key_to_double(uint64_t k) {
    const uint64_t u = (k >> 63) ? (k & 0x7FFFFFFFFFFFFFFFull) : ~k;
    return __longlong_as_double(static_cast<long long>(u));
}

struct SelScratch {
    uint32_t hist[256];
    uint64_t cand[32];
    uint64_t wmax[K1_WARPS], wmin[K1_WARPS];
    uint64_t prefix;
    int krem;
    int count;
    int n;
};

// k-th largest key among the candidates: radix select with 8-bit digits, MSB
// first, starting at the highest bit in which the candidates differ (a
// max / min reduction skips the common prefix, so the first histogram already
// spreads the keys instead of piling them into one bin); once <= 32
// candidates share the prefix one warp finishes by rank. Returns thr and
// need_eq = how many candidates equal to thr belong to the top k (the lowest
// ids among them, digest.hpp:108-111). k <= #candidates.
template <class KeyF, class CandF>
__device__ void radix_kth(int nb, int k, KeyF keyf, CandF candf, SelScratch& S, uint64_t& thr, int& need_eq) {
    const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
    uint64_t kmax = 0, kmin = ~0ull;
    for (int b = tid; b < nb; b += K1_THREADS) {
        if (!candf(b)) continue;
        const uint64_t key = keyf(b);
        kmax = key > kmax ? key : kmax;
        kmin = key < kmin ? key : kmin;
    }
#pragma unroll
    for (int o = 16; o; o >>= 1) {
        const uint64_t x = __shfl_xor_sync(0xffffffffu, kmax, o), y = __shfl_xor_sync(0xffffffffu, kmin, o);
        kmax = x > kmax ? x : kmax;
        kmin = y < kmin ? y : kmin;
    }
    if (lane == 0) { S.wmax[warp] = kmax; S.wmin[warp] = kmin; }
    __syncthreads();
#pragma unroll
    for (int w = 0; w < K1_WARPS; ++w) {
        kmax = S.wmax[w] > kmax ? S.wmax[w] : kmax;
        kmin = S.wmin[w] < kmin ? S.wmin[w] : kmin;
    }
    if (kmax == kmin) {  // every candidate equal (k <= #candidates)
        thr = kmax;
        need_eq = k;
        __syncthreads();
        return;
    }
    int hi = 63 - __clzll(static_cast<long long>(kmax ^ kmin));  // highest differing bit
    uint64_t mask = hi == 63 ? 0ull : ~((2ull << hi) - 1ull);      // bits above hi: shared by all
    uint64_t prefix = kmax & mask;
    int krem = k;
    while (hi >= 0) {
        const int w = hi + 1 < 8 ? hi + 1 : 8;
        const int shift = hi - w + 1;
        const uint32_t nbin = 1u << w;
        for (int i = tid; i < 256; i += K1_THREADS) S.hist[i] = 0;
        __syncthreads();
        for (int b = tid; b < nb; b += K1_THREADS) {
            if (!candf(b)) continue;
            const uint64_t key = keyf(b);
            if ((key & mask) == prefix) atomicAdd(&S.hist[(key >> shift) & (nbin - 1u)], 1u);
        }
        __syncthreads();
        if (tid < 32) {
            // lane l scans bins 255-8l .. 248-8l (bins >= nbin are empty)
            uint32_t cnt[8];
            uint32_t local = 0;
#pragma unroll
            for (int i = 0; i < 8; ++i) {
                cnt[i] = S.hist[255 - 8 * tid - i];
                local += cnt[i];
            }
            uint32_t incl = local;
#pragma unroll
            for (int o = 1; o < 32; o <<= 1) {
                const uint32_t y = __shfl_up_sync(0xffffffffu, incl, o);
                if (tid >= o) incl += y;
            }
            const uint32_t excl = incl - local;
            if (excl < static_cast<uint32_t>(krem) && incl >= static_cast<uint32_t>(krem)) {
                uint32_t cum = excl;
#pragma unroll
                for (int i = 0; i < 8; ++i) {
                    if (cum + cnt[i] >= static_cast<uint32_t>(krem)) {
                        S.prefix = prefix | (static_cast<uint64_t>(255 - 8 * tid - i) << shift);
                        S.krem = krem - static_cast<int>(cum);
                        S.count = static_cast<int>(cnt[i]);
                        break;
                    }
                    cum += cnt[i];
                }
            }
        }
        __syncthreads();
        prefix = S.prefix;
        krem = S.krem;
        mask |= static_cast<uint64_t>(nbin - 1u) << shift;
        hi = shift - 1;
        if (hi >= 0 && S.count <= 32) {
            // few candidates left: gather them and rank inside one warp
            if (tid == 0) S.n = 0;
            __syncthreads();
            for (int b = tid; b < nb; b += K1_THREADS) {
                if (!candf(b)) continue;
                const uint64_t key = keyf(b);
                if ((key & mask) == prefix) S.cand[atomicAdd(&S.n, 1)] = key;
            }
            __syncthreads();
            if (tid < 32) {
                const int n = S.n;
                const uint64_t mine = tid < n ? S.cand[tid] : 0;
                int gt = 0, eq = 0;
                for (int j = 0; j < n; ++j) {
                    const uint64_t o = S.cand[j];
                    gt += o > mine;
                    eq += o == mine;
                }
                __syncwarp();
                if (tid < n && gt < krem && krem <= gt + eq) {
                    S.prefix = mine;
                    S.krem = krem - gt;
                }
            }
            __syncthreads();
            thr = S.prefix;
            need_eq = S.krem;
            __syncthreads();
            return;
        }
    }
    thr = prefix;
    need_eq = krem;
    __syncthreads();
}

enum : uint8_t { CLS_OUT = 0, CLS_IN = 1, CLS_Z = 2 };

// Fast score of one 4-block quad over one chunk of channels (MODE 0): products
// and the running sum in fp32, flushed to the f64 accumulators every 8
// channels (<= 16 terms per fp32 chain); a_acc gathers sum |terms| for the band.
template <typename DigT>
__device__ __forceinline__ void fast_quad(const DigT* blo, const DigT* bhi, int ns, int b0, int nch, const float2* pn,
                                          int ch0, double (&s)[4], float (&a)[4]) {
    for (int c0 = 0; c0 < nch; c0 += 8) {
        const int c1 = min(nch, c0 + 8);
        float t[4] = {0.f, 0.f, 0.f, 0.f};
#pragma unroll 4
        for (int cl = c0; cl < c1; ++cl) {
            float l[4], h[4];
            if constexpr (sizeof(DigT) == 2) {
                const uint2 lv = *reinterpret_cast<const uint2*>(blo + cl * ns + b0);
                const uint2 hv = *reinterpret_cast<const uint2*>(bhi + cl * ns + b0);
                l[0] = __uint_as_float(lv.x << 16); l[1] = __uint_as_float(lv.x & 0xFFFF0000u);
                l[2] = __uint_as_float(lv.y << 16); l[3] = __uint_as_float(lv.y & 0xFFFF0000u);
                h[0] = __uint_as_float(hv.x << 16); h[1] = __uint_as_float(hv.x & 0xFFFF0000u);
                h[2] = __uint_as_float(hv.y << 16); h[3] = __uint_as_float(hv.y & 0xFFFF0000u);
            } else {
                const float4 lv = *reinterpret_cast<const float4*>(blo + cl * ns + b0);
                const float4 hv = *reinterpret_cast<const float4*>(bhi + cl * ns + b0);
                l[0] = lv.x; l[1] = lv.y; l[2] = lv.z; l[3] = lv.w;
                h[0] = hv.x; h[1] = hv.y; h[2] = hv.z; h[3] = hv.w;
            }
            const float2 pv = pn[ch0 + cl];  // (P_c, N_c): sums of the non-negative / negative q_g[c]
#pragma unroll
            for (int e = 0; e < 4; ++e) {
                t[e] = fmaf(h[e], pv.x, fmaf(l[e], pv.y, t[e]));
                a[e] = fmaf(fabsf(h[e]), pv.x, fmaf(fabsf(l[e]), -pv.y, a[e]));
            }
        }
#pragma unroll
        for (int e = 0; e < 4; ++e) s[e] += static_cast<double>(t[e]);
    }
}

// fast_quad over all 128 channels straight from global memory (bf16 digests):
// each thread streams its quad's lo / hi words of 4 channels per batch with
// evict-first loads, the next batch in flight while this one is summed; no
// shared-memory ring, no per-chunk barrier. Chains of 8 channels, as above.
#ifndef SCOUT_K1_DCB
#define SCOUT_K1_DCB 4  // channels per direct-load batch (two batches in flight)
#endif
#ifndef SCOUT_K1_DMINB
#define SCOUT_K1_DMINB 6   // CTAs per SM the direct QPT=2 variant is compiled for (80 registers)
#endif
#ifndef SCOUT_K1_DMINB1
#define SCOUT_K1_DMINB1 8  // ... and the QPT=1 variant (64 registers)
#endif
constexpr int DCB = SCOUT_K1_DCB;
// single-layer launches (few CTAs beside a running K2, each unit's digests
// latency-bound): batches of 8 channels, twice the loads in flight
#ifndef SCOUT_K1_DCB_SINGLE
#define SCOUT_K1_DCB_SINGLE 8
#endif
#ifndef SCOUT_K1_SMINB
#define SCOUT_K1_SMINB 4  // CTAs per SM the single-layer variants are compiled for
#endif
constexpr int DCB_SINGLE = SCOUT_K1_DCB_SINGLE;
template <int B>
__device__ __forceinline__ void ld_quad4(const __nv_bfloat16* lo, const __nv_bfloat16* hi, size_t ns, int b0, int c0,
                                         uint2 (&L)[B], uint2 (&H)[B]) {
#pragma unroll
    for (int i = 0; i < B; ++i) {
        L[i] = __ldcs(reinterpret_cast<const uint2*>(lo + static_cast<size_t>(c0 + i) * ns + b0));
        H[i] = __ldcs(reinterpret_cast<const uint2*>(hi + static_cast<size_t>(c0 + i) * ns + b0));
    }
}
template <int B>
__device__ __forceinline__ void sum_quad4(const uint2 (&L)[B], const uint2 (&H)[B], const float2* pn, int c0,
                                          float (&t)[4], float (&a)[4]) {
#pragma unroll
    for (int i = 0; i < B; ++i) {
        float l[4], h[4];
        l[0] = __uint_as_float(L[i].x << 16); l[1] = __uint_as_float(L[i].x & 0xFFFF0000u);
        l[2] = __uint_as_float(L[i].y << 16); l[3] = __uint_as_float(L[i].y & 0xFFFF0000u);
        h[0] = __uint_as_float(H[i].x << 16); h[1] = __uint_as_float(H[i].x & 0xFFFF0000u);
        h[2] = __uint_as_float(H[i].y << 16); h[3] = __uint_as_float(H[i].y & 0xFFFF0000u);
        const float2 pv = pn[c0 + i];
#pragma unroll
        for (int e = 0; e < 4; ++e) {
            t[e] = fmaf(h[e], pv.x, fmaf(l[e], pv.y, t[e]));
            a[e] = fmaf(fabsf(h[e]), pv.x, fmaf(fabsf(l[e]), -pv.y, a[e]));
        }
    }
}
// channels [cb, ce) (multiples of 2 * B)
template <int B>
__device__ __forceinline__ void fast_quad_direct(const __nv_bfloat16* lo, const __nv_bfloat16* hi, size_t ns, int b0,
                                                 const float2* pn, double (&s)[4], float (&a)[4], int cb = 0,
                                                 int ce = D) {
    static_assert(B == 4 || B == 8, "8-channel fp32 chains: batches of 4 (two per chain) or 8");
    uint2 L0[B], H0[B], L1[B], H1[B];
    ld_quad4<B>(lo, hi, ns, b0, cb, L0, H0);
#pragma unroll 1
    for (int c0 = cb; c0 < ce; c0 += 2 * B) {
        float t[4] = {0.f, 0.f, 0.f, 0.f};
        ld_quad4<B>(lo, hi, ns, b0, c0 + B, L1, H1);
        sum_quad4<B>(L0, H0, pn, c0, t, a);
        if (B == 8) {  // one chain per batch
#pragma unroll
            for (int e = 0; e < 4; ++e) { s[e] += static_cast<double>(t[e]); t[e] = 0.f; }
        }
        if (c0 + 2 * B < ce) ld_quad4<B>(lo, hi, ns, b0, c0 + 2 * B, L0, H0);
        sum_quad4<B>(L1, H1, pn, c0 + B, t, a);
#pragma unroll
        for (int e = 0; e < 4; ++e) s[e] += static_cast<double>(t[e]);
    }
}

// QPT: block quads per thread whose running scores live in registers (1: up
// to 512 blocks, 2: up to 1024, 4: up to 2048); 0: shared-memory accumulators.
template <typename DigT, int G, int MODE, int QPT, bool DIRECT = false, int NA = K1_MAX_LAYERS>
__global__ void __launch_bounds__(K1_THREADS, DIRECT ? (NA == 1 ? SCOUT_K1_SMINB : (QPT == 1 ? SCOUT_K1_DMINB1 : (QPT == 2 ? SCOUT_K1_DMINB : 4)))
                                                      : ((QPT == 1 || QPT == 2) ? 7 : SCOUT_K1_MINB))
    score_topk_kernel(const K1BatchT<NA> batch) {
    constexpr int KB = NA == 1 ? DCB_SINGLE : DCB;  // channels per direct-load batch
    // Work items are (layer, unit) pairs, flattened layer-major. Classic grid
    // (units x layers): one item per CTA. Persistent grid (batch.persist): CTA
    // c takes items c, c + grid, ... and the digest ring keeps streaming across
    // item boundaries, so one item's latency-bound selection phase overlaps
    // the next item's first digest chunks.
    const int n_units = batch.a[0].n_units;
    const long long total_items = static_cast<long long>(n_units) * batch.n;
    const long long first = batch.persist ? blockIdx.x : static_cast<long long>(blockIdx.y) * n_units + blockIdx.x;
    const long long stride = batch.persist ? gridDim.x : total_items;
    const int n_my = first < total_items ? static_cast<int>((total_items - first + stride - 1) / stride) : 0;
    extern __shared__ __align__(16) uint8_t k1_smem[];
    const size_t ns = static_cast<size_t>(batch.a[0].nb_stride);
    double* qs = reinterpret_cast<double*>(k1_smem);             // [D][G] stacked order
    float2* pn = reinterpret_cast<float2*>(qs + D * G);          // [D] (sum q>=0, sum q<0) rounded to f32
    uint64_t* keys = reinterpret_cast<uint64_t*>(pn + D);        // [nb_stride]
    uint8_t* cls = reinterpret_cast<uint8_t*>(keys + ns);        // [nb_stride]
    uint8_t* big = k1_smem + (static_cast<size_t>(D) * G * 8 + D * 8 + ns * 9 + 15) / 16 * 16;
    double* s_acc = reinterpret_cast<double*>(big);              // [nb_stride] (nb_stride > K1_REG_BLOCKS)
    float* a_acc = reinterpret_cast<float*>(s_acc + ns);         // [nb_stride]
    uint8_t* stagebuf = k1_smem + k1_stage_offset(G, static_cast<int>(ns));  // nbuf x chunk (MODE 0)
    __shared__ uint64_t s_full[K1_MAXBUF];
    __shared__ SelScratch S;
    __shared__ int warp_tot[K1_WARPS];
    __shared__ int s_tok[2];
    __shared__ int s_cnt[2];
    __shared__ int s_cnt2[2];
    __shared__ float s_amax;

    const int tid = threadIdx.x;
    const int nbuf = batch.nbuf;
    // digest chunk ring: chunks of `cpc` channels (lo rows + hi rows) stream
    // through shared memory with 1-D bulk copies (TMA engine); global chunk
    // numbers run across this CTA's items. The first copies go out before
    // anything else so the query staging hides under them.
    constexpr int esz = static_cast<int>(sizeof(DigT));
    const int cpc = max(1, min(D, batch.chunk / (2 * static_cast<int>(ns) * esz)));
    const int nchunks = (D + cpc - 1) / cpc;
    const uint32_t lo_bytes = static_cast<uint32_t>(cpc * ns * esz);  // one half of a chunk buffer
    const long long total_chunks = static_cast<long long>(n_my) * nchunks;
    // issuer state (thread 0): next global chunk and the item it belongs to
    long long g_iss = 0;
    int iss_item = 0, iss_chunk = 0;
    const DigT* iss_lo = nullptr;
    auto item_digests = [&](int local) {
        const long long it = first + static_cast<long long>(local) * stride;
        const scout_topk_args& ai = batch.a[it / n_units];
        return static_cast<const DigT*>(ai.digests) + static_cast<size_t>(it % n_units) * 2 * D * ns;
    };
    auto issue_next = [&]() {
        if (iss_chunk == 0) iss_lo = item_digests(iss_item);
        const int ch0 = iss_chunk * cpc, nch = min(cpc, D - ch0);
        const uint32_t bytes = static_cast<uint32_t>(nch * ns * esz);
        const int slot = static_cast<int>(g_iss % nbuf);
        uint8_t* buf = stagebuf + static_cast<size_t>(slot) * 2 * lo_bytes;
        mbar_arrive_expect_tx(&s_full[slot], 2 * bytes);
        bulk_g2s(buf, iss_lo + ch0 * ns, bytes, &s_full[slot]);
        bulk_g2s(buf + lo_bytes, iss_lo + (D + ch0) * ns, bytes, &s_full[slot]);
        ++g_iss;
        if (++iss_chunk == nchunks) {
            iss_chunk = 0;
            ++iss_item;
        }
    };
    constexpr bool can_direct = DIRECT && MODE == 0 && QPT > 0 && sizeof(DigT) == 2;
    constexpr bool direct = can_direct;
    if constexpr (MODE == 0) {
        if (tid == 0 && !direct) {
            for (int i = 0; i < nbuf; ++i) mbar_init(&s_full[i], 1);
            fence_mbar_init();
            while (g_iss < nbuf && g_iss < total_chunks) issue_next();
        }
    }
    // PDL: the next kernel may launch now; this one only reads inputs until it
    // publishes its lists (griddep_wait below orders those writes).
    griddep_launch_dependents();
    long long g_cons = 0;  // chunks consumed (uniform across threads)
    for (int item = 0; item < n_my; ++item) {
    const long long it = first + static_cast<long long>(item) * stride;
    const scout_topk_args& a = batch.a[it / n_units];
    const int u = static_cast<int>(it % n_units);
    const DigT* lo = static_cast<const DigT*>(a.digests) + static_cast<size_t>(u) * 2 * D * ns;
    const DigT* hi = lo + D * ns;
    if (a.scores_out) griddep_wait();
    int ntok = a.n_tokens[u];
    ntok = max(0, min(ntok, a.nb_stride * BS));
    const int nb = (ntok + BS - 1) / BS;
    const int tail = ntok - (nb - 1) * BS;

    for (int i = tid; i < D * G; i += K1_THREADS) {
        const int g = i / D, c = i % D;
        double v;
        const size_t qi = (static_cast<size_t>(u) * G + g) * D + c;
        if constexpr (MODE == 0)
            v = a.q_dtype == SCOUT_BF16 ? static_cast<double>(__bfloat162float(static_cast<const __nv_bfloat16*>(a.q)[qi]))
                                        : static_cast<const float*>(a.q)[qi];
        else v = static_cast<const double*>(a.q)[qi];
        qs[c * G + g] = v;
    }
    if (tid < 2) { s_tok[tid] = 0; s_cnt[tid] = 0; }
    if (tid == 0) s_amax = 0.f;
    __syncthreads();

    const int k = a.k;
    const bool take_all = nb <= k;

    if constexpr (MODE == 0) {
        // ---- fast score s~_b = sum_c hi_c * P_c + lo_c * N_c in fp32 chains of <= 16
        // terms summed in f64 (P_c / N_c: sums of the non-negative / negative q_g[c],
        // rounded to f32). Error vs the reference's sequential double sum:
        //   |s~ - s_ref| <= (16 + 1) u32 A_b + 2^-43 A_b + underflow < A_b 2^-19 + 2^-126
        // with A_b = sum |terms| (fp32, rounded up by 1.0001). Blocks within the
        // band of the k-th score are decided exactly below.
        if (tid < D) {
            double P = 0.0, N = 0.0;
#pragma unroll
            for (int g = 0; g < G; ++g) {
                const double qv = qs[tid * G + g];
                if (qv >= 0.0) P += qv;
                else N += qv;
            }
            pn[tid] = make_float2(static_cast<float>(P), static_cast<float>(N));
            // f32-subnormal sums lose the relative bound: decide the unit exactly
            if ((P != 0.0 && P < 0x1p-126) || (N != 0.0 && N > -0x1p-126))
                atomicMax(reinterpret_cast<int*>(&s_amax), 0x7f800000);
        }
        const int nq = (nb + 3) >> 2;
        constexpr bool regs = QPT > 0;
        if (!regs)
            for (int i = tid; i < nq * 4; i += K1_THREADS) { s_acc[i] = 0.0; a_acc[i] = 0.f; }
        __syncthreads();
        constexpr int RQ = QPT > 0 ? QPT : 1;
        double rs[RQ][4];
        float ra[RQ][4];
#pragma unroll
        for (int q = 0; q < RQ; ++q)
#pragma unroll
            for (int e = 0; e < 4; ++e) { rs[q][e] = 0.0; ra[q][e] = 0.f; }
        if constexpr (can_direct) {
            const __nv_bfloat16* dlo = reinterpret_cast<const __nv_bfloat16*>(lo);
            const __nv_bfloat16* dhi = reinterpret_cast<const __nv_bfloat16*>(hi);
            const int ntail = nq - K1_THREADS;  // quads past the first pass
            if (QPT == 2 && ntail > 0 && ntail <= 32) {
                // a stride just above 4 * K1_THREADS blocks (tier mode: room for
                // appended blocks): the few tail quads would leave one thread each
                // streaming all 128 channels while the CTA waits. Instead every
                // warp takes a quarter of the channels of every tail quad, and
                // warp 0 adds the four partials (f64 sums of the same <= 8-channel
                // fp32 chains: the error bound is unchanged).
                if (tid < nq) fast_quad_direct<KB>(dlo, dhi, ns, 4 * tid, pn, rs[0], ra[0]);
                double* ps = reinterpret_cast<double*>(stagebuf);        // [K1_WARPS][32][4]
                float* pa = reinterpret_cast<float*>(ps + K1_WARPS * 128);  // [K1_WARPS][32][4]
                const int w = tid >> 5, l = tid & 31;
                if (l < ntail) {
                    double s4[4] = {0.0, 0.0, 0.0, 0.0};
                    float a4[4] = {0.f, 0.f, 0.f, 0.f};
                    const int cq = D / K1_WARPS;
                    fast_quad_direct<KB>(dlo, dhi, ns, 4 * (K1_THREADS + l), pn, s4, a4, w * cq, (w + 1) * cq);
#pragma unroll
                    for (int e = 0; e < 4; ++e) { ps[(w * 32 + l) * 4 + e] = s4[e]; pa[(w * 32 + l) * 4 + e] = a4[e]; }
                }
                __syncthreads();
                if (tid < ntail)
                    for (int ww = 0; ww < K1_WARPS; ++ww)
#pragma unroll
                        for (int e = 0; e < 4; ++e) {
                            rs[RQ - 1][e] += ps[(ww * 32 + tid) * 4 + e];
                            ra[RQ - 1][e] += pa[(ww * 32 + tid) * 4 + e];
                        }
            } else if (direct) {
#pragma unroll
                for (int q = 0; q < RQ; ++q) {
                    const int j = tid + q * K1_THREADS;
                    if (j < nq) fast_quad_direct<KB>(dlo, dhi, ns, 4 * j, pn, rs[q], ra[q]);
                }
            }
        }
        for (int c = 0; c < (direct ? 0 : nchunks); ++c, ++g_cons) {
            const int slot = static_cast<int>(g_cons % nbuf);
            mbar_wait(&s_full[slot], static_cast<uint32_t>((g_cons / nbuf) & 1));
            const int ch0 = c * cpc, nch = min(cpc, D - ch0);
            const DigT* blo = reinterpret_cast<const DigT*>(stagebuf + static_cast<size_t>(slot) * 2 * lo_bytes);
            const DigT* bhi = reinterpret_cast<const DigT*>(reinterpret_cast<const uint8_t*>(blo) + lo_bytes);
            if constexpr (regs) {
#pragma unroll
                for (int q = 0; q < QPT; ++q) {
                    const int j = tid + q * K1_THREADS;
                    if (j < nq) fast_quad<DigT>(blo, bhi, static_cast<int>(ns), 4 * j, nch, pn, ch0, rs[q], ra[q]);
                }
            } else {
                for (int j = tid; j < nq; j += K1_THREADS) {
                    double s4[4];
                    float a4[4];
#pragma unroll
                    for (int e = 0; e < 4; ++e) { s4[e] = s_acc[e * nq + j]; a4[e] = a_acc[e * nq + j]; }
                    fast_quad<DigT>(blo, bhi, static_cast<int>(ns), 4 * j, nch, pn, ch0, s4, a4);
#pragma unroll
                    for (int e = 0; e < 4; ++e) { s_acc[e * nq + j] = s4[e]; a_acc[e * nq + j] = a4[e]; }
                }
            }
            __syncthreads();  // buffer drained by every thread: refill it (possibly with the next item's chunks)
            if (tid == 0 && g_iss < total_chunks) issue_next();
        }
        float amax = 0.f;
        if constexpr (regs) {
#pragma unroll
            for (int q = 0; q < QPT; ++q) {
                const int j = tid + q * K1_THREADS;
#pragma unroll
                for (int e = 0; e < 4; ++e)
                    if (4 * j + e < nb) {
                        keys[4 * j + e] = score_key(rs[q][e]);
                        amax = fmaxf(amax, ra[q][e] * 1.0001f);
                    }
            }
        } else {
            for (int b = tid; b < nb; b += K1_THREADS) {
                keys[b] = score_key(s_acc[(b & 3) * nq + (b >> 2)]);
                amax = fmaxf(amax, a_acc[(b & 3) * nq + (b >> 2)] * 1.0001f);
            }
        }
        // NaN / inf (fp32 overflow) -> an infinite band: every block is decided exactly
        if (!(amax <= 3.0e38f)) amax = __int_as_float(0x7f800000);
#pragma unroll
        for (int o = 16; o; o >>= 1) amax = fmaxf(amax, __shfl_xor_sync(0xffffffffu, amax, o));
        if ((tid & 31) == 0) atomicMax(reinterpret_cast<int*>(&s_amax), __float_as_int(amax));
        if (a.scores_out)  // exact reference-order scores (tests / diagnostics only)
            for (int b = tid; b < nb; b += K1_THREADS)
                a.scores_out[u * ns + b] = exact_score_minmax<DigT, G>(lo, hi, ns, b, qs);
    } else {
        for (int b = tid; b < nb; b += K1_THREADS) {
            const double sc = exact_score_f64<G, MODE>(static_cast<const double*>(a.digests) +
                                                            static_cast<size_t>(u) * (MODE == 1 ? 2 : 1) * D * ns,
                                                        ns, b, qs);
            keys[b] = score_key(sc);
            if (a.scores_out) a.scores_out[u * ns + b] = sc;
        }
    }
    __syncthreads();

    // ---- classify every block: IN (certainly top-k), OUT, or Z (decide exactly)
    uint64_t thr = 0;
    int need_eq = 0;
    bool z_exact = false;  // Z members carry exact keys and a radix select among them
    if (take_all) {
        for (int b = tid; b < nb; b += K1_THREADS) cls[b] = CLS_IN;
    } else if constexpr (MODE != 0) {
        // keys are exact already: plain top-k
        radix_kth(nb, k, [&](int b) { return keys[b]; }, [](int) { return true; }, S, thr, need_eq);
        for (int b = tid; b < nb; b += K1_THREADS) cls[b] = CLS_Z;
        z_exact = true;
    } else {
        uint64_t tkey;
        int dummy;
        radix_kth(nb, k, [&](int b) { return keys[b]; }, [](int) { return true; }, S, tkey, dummy);
        const double T = key_to_double(tkey);
        const double band = 2.0 * (static_cast<double>(s_amax) * 0x1p-19 + 0x1p-126);
        int nin = 0, nz = 0;
        for (int b = tid; b < nb; b += K1_THREADS) {
            const double v = key_to_double(keys[b]);
            const uint8_t c = v > T + band ? CLS_IN : (v < T - band ? CLS_OUT : CLS_Z);
            cls[b] = c;
            nin += c == CLS_IN;
            nz += c == CLS_Z;
        }
        if (nin) atomicAdd(&s_cnt[0], nin);
        if (nz) atomicAdd(&s_cnt[1], nz);
        __syncthreads();
        int need = k - s_cnt[0];
        if (s_cnt[1] > need) {
            // stage 2: f64 scores of the Z blocks, one warp per block (lane
            // partial sums of 32 exact products + a 5-level butterfly): within
            // 37 u A < 2^-47 A of the exact sum, so within 2^-42 A of the
            // reference's sequential sum (1023 u A). The fp32 band's near-ties
            // mostly resolve here; only blocks inside the 2^-40 A band go on
            // to the sequential exact chain.
            {
                const int lane = tid & 31, warp = tid >> 5;
                int zi = 0;  // Z blocks in id order, dealt round-robin to the warps
                for (int base = 0; base < nb; base += 32) {
                    const int b = base + lane;
                    unsigned m = __ballot_sync(0xffffffffu, b < nb && cls[b] == CLS_Z);
                    while (m) {
                        const int j = base + __ffs(m) - 1;
                        m &= m - 1;
                        if (zi++ % K1_WARPS != warp) continue;
                        double acc = 0.0;
#pragma unroll
                        for (int i = 0; i < D / 32; ++i) {
                            const int c = lane + 32 * i;
                            const double l = widen(lo[c * ns + j]), h = widen(hi[c * ns + j]);
#pragma unroll
                            for (int g = 0; g < G; ++g) {
                                const double qv = qs[c * G + g];
                                acc = fma(qv, qv >= 0.0 ? h : l, acc);
                            }
                        }
#pragma unroll
                        for (int o = 16; o; o >>= 1) acc += __shfl_xor_sync(0xffffffffu, acc, o);
                        if (lane == 0) keys[j] = score_key(acc);
                    }
                }
            }
            if (tid < 2) s_cnt2[tid] = 0;
            __syncthreads();
            uint64_t tkey2;
            int dummy2;
            radix_kth(nb, need, [&](int b) { return keys[b]; }, [&](int b) { return cls[b] == CLS_Z; }, S, tkey2,
                      dummy2);
            const double T2 = key_to_double(tkey2);
            const double band2 = static_cast<double>(s_amax) * 0x1p-40;
            int nin2 = 0, nz2 = 0;
            for (int b = tid; b < nb; b += K1_THREADS) {
                if (cls[b] != CLS_Z) continue;
                const double v = key_to_double(keys[b]);
                const uint8_t c = v > T2 + band2 ? CLS_IN : (v < T2 - band2 ? CLS_OUT : CLS_Z);
                cls[b] = c;
                nin2 += c == CLS_IN;
                nz2 += c == CLS_Z;
            }
            if (nin2) atomicAdd(&s_cnt2[0], nin2);
            if (nz2) atomicAdd(&s_cnt2[1], nz2);
            __syncthreads();
            need -= s_cnt2[0];
            if (s_cnt2[1] > need) {
                // genuinely ambiguous boundary: exact reference-order scores for Z
                for (int b = tid; b < nb; b += K1_THREADS)
                    if (cls[b] == CLS_Z) keys[b] = score_key(exact_score_minmax<DigT, G>(lo, hi, ns, b, qs));
                __syncthreads();
                radix_kth(nb, need, [&](int b) { return keys[b]; }, [&](int b) { return cls[b] == CLS_Z; }, S, thr,
                          need_eq);
                z_exact = true;
            }
        }
    }
    __syncthreads();

    if (!batch.nowait) griddep_wait();  // everything before this launch is complete: safe to publish
    // ---- selection flags in id order: contiguous chunks per thread
    const int chunk = (nb + K1_THREADS - 1) / K1_THREADS;
    const int b_begin = min(nb, tid * chunk), b_end = min(nb, b_begin + chunk);
    int total;
    int eq_rank = 0;
    if (z_exact) {
        int eq_local = 0;
        for (int b = b_begin; b < b_end; ++b) eq_local += (cls[b] == CLS_Z && keys[b] == thr);
        eq_rank = block_exclusive_scan(eq_local, warp_tot, &total);
    }
    auto selected = [&](int b, int& er) {
        const uint8_t c = cls[b];
        if (c == CLS_IN) return true;
        if (c != CLS_Z) return false;
        if (!z_exact) return true;
        const uint64_t key = keys[b];
        if (key > thr) return true;
        if (key == thr) return er++ < need_eq;
        return false;
    };
    const int32_t* table = a.block_table ? a.block_table + static_cast<size_t>(u) * a.nb_stride : nullptr;
    int sel_local = 0, res_local = 0;
    {
        int er = eq_rank;
        for (int b = b_begin; b < b_end; ++b)
            if (selected(b, er)) {
                ++sel_local;
                if (table && table[b] >= 0) ++res_local;
            }
    }
    const int packed = block_exclusive_scan(sel_local | (res_local << 16), warp_tot, &total);
    int sel_pos = packed & 0xFFFF, res_pos = packed >> 16;
    int tok_res = 0, tok_cpu = 0;
    {
        int er = eq_rank;
        const size_t row = static_cast<size_t>(u) * a.k_stride;
        for (int b = b_begin; b < b_end; ++b) {
            if (!selected(b, er)) continue;
            const int rows = (b == nb - 1) ? tail : BS;
            if (a.sel_ids) a.sel_ids[row + sel_pos] = b;
            if (a.last_selected) a.last_selected[static_cast<size_t>(u) * a.nb_stride + b] = a.step;
            if (table) {
                const int slot = table[b];
                if (slot >= 0) {
                    if (a.res_slots) a.res_slots[row + res_pos] = slot;
                    if (a.res_ids) a.res_ids[row + res_pos] = b;
                    ++res_pos;
                    tok_res += rows;
                } else {
                    if (a.cpu_ids) a.cpu_ids[row + (sel_pos - res_pos)] = b;
                    tok_cpu += rows;
                }
            }
            ++sel_pos;
        }
    }
    if (tok_res) atomicAdd(&s_tok[0], tok_res);
    if (tok_cpu) atomicAdd(&s_tok[1], tok_cpu);
    __syncthreads();
    if (tid == 0) {
        const int nsel = total & 0xFFFF, nres = total >> 16;
        if (a.n_sel) a.n_sel[u] = nsel;
        if (table) {
            if (a.n_res) a.n_res[u] = nres;
            if (a.n_cpu) a.n_cpu[u] = nsel - nres;
            if (a.res_tokens) a.res_tokens[u] = s_tok[0];
            if (a.cpu_tokens) a.cpu_tokens[u] = s_tok[1];
        }
        if (a.done_flag) {
            // layer-wide completion: the last item of the layer publishes the
            // flag a concurrently running K2 polls (ld.acquire) before reading
            __threadfence();
            const unsigned old = atomicAdd(a.done_ctr, 1u);
            if (old == static_cast<unsigned>(n_units) - 1u) {
                *a.done_ctr = 0u;
                __threadfence();
                asm volatile("st.release.gpu.global.u32 [%0], %1;" ::"l"(a.done_flag), "r"(a.done_token) : "memory");
                if (batch.all_flag && atomicAdd(batch.all_ctr, 1u) == static_cast<unsigned>(batch.n) - 1u) {
                    *batch.all_ctr = 0u;  // every layer published: the launch's lists are complete
                    __threadfence();
                    asm volatile("st.release.gpu.global.u32 [%0], %1;" ::"l"(batch.all_flag), "r"(batch.all_token)
                                 : "memory");
                }
            }
        }
    }
    __syncthreads();  // shared state is reused by the next item
    }
}

template <typename DigT, int MODE, int NA>
int launch_g(K1BatchT<NA>& b, cudaStream_t st) {
    const scout_topk_args& a = b.a[0];
    // digest ring depth (tuning knob SCOUT_K1_NBUF, 1..K1_MAXBUF)
    // and chunk bytes (SCOUT_K1_CHUNK, 4096..65536)
    static const int nbuf_env = [] {
        const char* e = getenv("SCOUT_K1_NBUF");
        const int v = e ? atoi(e) : 2;
        return v < 1 ? 1 : (v > K1_MAXBUF ? K1_MAXBUF : v);
    }();
    static const int chunk_env = [] {
        const char* e = getenv("SCOUT_K1_CHUNK");
        const int v = e ? atoi(e) : K1_CHUNK_BYTES;
        return v < 4096 ? 4096 : (v > 65536 ? 65536 : v);
    }();
    b.nbuf = nbuf_env;
    b.chunk = chunk_env;
    // many blocks per unit: at least 4 channels per chunk (fewer ring round trips)
    if (MODE == 0 && a.nb_stride > 512) {
        const int four = 4 * a.nb_stride * 2 * static_cast<int>(sizeof(DigT));
        const int want = four < 32768 ? four : 32768;
        if (b.chunk < want) b.chunk = want;
    }
    static const bool direct_env = [] {
        const char* e = getenv("SCOUT_K1_DIRECT");
        return e ? atoi(e) != 0 : true;
    }();
    b.direct = MODE == 0 && sizeof(DigT) == 2 && direct_env && a.nb_stride <= K1_REG_BLOCKS;  // QPT 1 / 2 / 4
    // direct loads: no ring; the 2-quad variant keeps a tail-quad scratch there (K1_WARPS x 32 x 4 x (8 + 4) B)
    const size_t smem = MODE == 0 ? (b.direct ? k1_stage_offset(a.group, a.nb_stride) + K1_WARPS * 32 * 4 * 12
                                              : k1_smem_bytes(a.group, a.nb_stride, static_cast<int>(sizeof(DigT)),
                                                              b.nbuf, b.chunk))
                                  : k1_stage_offset(a.group, a.nb_stride);
    // persistent grid (SCOUT_K1_PERSIST=1): measured slower than the classic
    // one-item-per-CTA grid at config 3 (0.93 vs 0.86 ms per 64 layers), whose
    // freshly started CTAs overlap their prologue with other CTAs' selection
    // phases as well as a continuous ring does; kept opt-in and tested
    static const bool persist_env = [] {
        const char* e = getenv("SCOUT_K1_PERSIST");
        return e ? atoi(e) != 0 : false;
    }();
    auto go = [&](auto kern) {
        if (smem > 48 * 1024) scout_host::ensure_smem(reinterpret_cast<const void*>(kern), smem);
        // persistent grid: resident CTAs x SMs, when the items outnumber them
        const long long items = static_cast<long long>(a.n_units) * b.n;
        long long slots = 0;
        if (b.slots > 0) {
            slots = b.slots;
        } else if (b.slots < 0) {  // resident CTAs on -slots SMs
            int per_sm = 0;
            cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, kern, K1_THREADS, smem);
            slots = static_cast<long long>(per_sm > 0 ? per_sm : 1) * -b.slots;
        } else if (MODE == 0 && persist_env) {  // (occupancy queried only for the opt-in persistent grid)
            int per_sm = 0;
            cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, kern, K1_THREADS, smem);
            int dev = 0, sms = 148;
            cudaGetDevice(&dev);
            cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
            slots = static_cast<long long>(per_sm > 0 ? per_sm : 1) * sms;
        }
        b.persist = b.slots != 0 || (MODE == 0 && persist_env && items > slots);
        const dim3 grid = b.persist ? dim3(static_cast<unsigned>(slots)) : dim3(a.n_units, b.n);
        scout_host::launch(kern, grid, dim3(K1_THREADS), smem, st, (a.flags & SCOUT_LAUNCH_PDL) != 0, b);
    };
    const int ns = a.nb_stride;
    const int qpt = MODE != 0 ? 1 : (ns <= 4 * K1_THREADS ? 1 : (ns <= 8 * K1_THREADS ? 2 : (ns <= K1_REG_BLOCKS ? 4 : 0)));
    auto pick = [&](auto g) {
        constexpr int Gv = decltype(g)::value;
        if constexpr (MODE == 0 && sizeof(DigT) == 2) {
            if (b.direct) {
                if (qpt == 1) go(score_topk_kernel<DigT, Gv, MODE, 1, true, NA>);
                else if (qpt == 2) go(score_topk_kernel<DigT, Gv, MODE, 2, true, NA>);
                else go(score_topk_kernel<DigT, Gv, MODE, 4, true, NA>);
                return;
            }
        }
        if (qpt == 1) go(score_topk_kernel<DigT, Gv, MODE, 1, false, NA>);
        else if constexpr (MODE == 0) {
            if (qpt == 2) go(score_topk_kernel<DigT, Gv, MODE, 2, false, NA>);
            else if (qpt == 4) go(score_topk_kernel<DigT, Gv, MODE, 4, false, NA>);
            else go(score_topk_kernel<DigT, Gv, MODE, 0, false, NA>);
        }
    };
    switch (a.group) {
        case 1: pick(std::integral_constant<int, 1>{}); break;
        case 2: pick(std::integral_constant<int, 2>{}); break;
        case 4: pick(std::integral_constant<int, 4>{}); break;
        case 8: pick(std::integral_constant<int, 8>{}); break;
        default: return -1;
    }
    return 0;
}

int validate(const scout_topk_args& a) {
    using namespace scout_host;
    if (a.k == 0) {
        set_error(SCOUT_ERR_INVALID_ARGUMENT, "select_topk: k must be >= 1");
        return SCOUT_ERR_INVALID_ARGUMENT;
    }
    if (a.k < 0 || a.k > SCOUT_MAX_K || a.k_stride < a.k) {
        set_error(SCOUT_ERR_INVALID_ARGUMENT, "scout_score_topk_split: k=%d out of range (k_stride %d, max %d)", a.k,
                  a.k_stride, SCOUT_MAX_K);
        return SCOUT_ERR_INVALID_ARGUMENT;
    }
    if (a.n_units < 0 || a.nb_stride <= 0 || a.nb_stride % 8 != 0 || a.nb_stride > SCOUT_MAX_BLOCKS) {
        set_error(SCOUT_ERR_INVALID_ARGUMENT, "scout_score_topk_split: bad n_units %d / nb_stride %d", a.n_units,
                  a.nb_stride);
        return SCOUT_ERR_INVALID_ARGUMENT;
    }
    if (a.group != 1 && a.group != 2 && a.group != 4 && a.group != 8) {
        set_error(SCOUT_ERR_INVALID_ARGUMENT, "scout_score_topk_split: group %d not in {1,2,4,8}", a.group);
        return SCOUT_ERR_INVALID_ARGUMENT;
    }
    if (a.q_dtype != SCOUT_F32 && !(a.q_dtype == SCOUT_BF16 && a.digest_dtype != SCOUT_F64)) {
        set_error(SCOUT_ERR_INVALID_ARGUMENT, "scout_score_topk_split: q dtype %d unsupported with digest dtype %d",
                  a.q_dtype, a.digest_dtype);
        return SCOUT_ERR_INVALID_ARGUMENT;
    }
    if (a.n_units > 0 && (!a.q || !a.digests || !a.n_tokens)) {
        set_error(SCOUT_ERR_INVALID_ARGUMENT, "scout_score_topk_split: null q/digests/n_tokens");
        return SCOUT_ERR_INVALID_ARGUMENT;
    }
    return SCOUT_OK;
}

int launch_batch(K1Batch& b, cudaStream_t st) {
    using namespace scout_host;
    const scout_topk_args& a = b.a[0];
    int rc = -1;
    if (a.method == SCOUT_DIGEST_MINMAX && a.digest_dtype != SCOUT_F64 && b.n == 1) {
        // single layer: the 1-slot parameter block
        static thread_local K1Batch1 b1;
        b1.n = 1;
        b1.nowait = b.nowait;
        b1.slots = b.slots;
        b1.all_ctr = b.all_ctr;
        b1.all_flag = b.all_flag;
        b1.all_token = b.all_token;
        b1.a[0] = a;
        if (a.digest_dtype == SCOUT_BF16) rc = launch_g<__nv_bfloat16, 0>(b1, st);
        else if (a.digest_dtype == SCOUT_F32) rc = launch_g<float, 0>(b1, st);
    } else if (a.method == SCOUT_DIGEST_MINMAX) {
        if (a.digest_dtype == SCOUT_BF16) rc = launch_g<__nv_bfloat16, 0>(b, st);
        else if (a.digest_dtype == SCOUT_F32) rc = launch_g<float, 0>(b, st);
        else if (a.digest_dtype == SCOUT_F64) rc = launch_g<double, 1>(b, st);
    } else if (a.method == SCOUT_DIGEST_MEAN) {
        if (a.digest_dtype == SCOUT_F64) rc = launch_g<double, 2>(b, st);
    }
    if (rc != 0) {
        set_error(SCOUT_ERR_UNSUPPORTED, "scout_score_topk_split: method %d with digest dtype %d unsupported",
                  a.method, a.digest_dtype);
        return SCOUT_ERR_UNSUPPORTED;
    }
    return check_launch("scout_score_topk_split");
}

}  // namespace

extern "C" int scout_score_topk_split(const scout_topk_args* args, void* stream) {
    using namespace scout_host;
    if (!args) {
        set_error(SCOUT_ERR_INVALID_ARGUMENT, "scout_score_topk_split: null args");
        return SCOUT_ERR_INVALID_ARGUMENT;
    }
    const int rc = validate(*args);
    if (rc != SCOUT_OK) return rc;
    if (args->n_units == 0) return SCOUT_OK;
    static thread_local K1Batch b;  // kernel parameters (copied at launch)
    b.n = 1;
    b.nowait = 0;
    b.slots = 0;
    b.all_ctr = b.all_flag = nullptr;
    b.a[0] = *args;
    return launch_batch(b, static_cast<cudaStream_t>(stream));
}

static int k1_launch_batch(const scout_topk_args* layers, int n, cudaStream_t st, int slots, int nowait,
                           unsigned* all_ctr, unsigned* all_flag, unsigned all_token);

int scout_k1_launch_batch(const scout_topk_args* layers, int n, cudaStream_t st) {
    return k1_launch_batch(layers, n, st, 0, 0, nullptr, nullptr, 0);
}

int scout_k1_launch_batch_beside(const scout_topk_args* layers, int n, int sms, cudaStream_t st, unsigned* all_ctr,
                                 unsigned* all_flag, unsigned all_token) {
    if (sms <= 0 || (all_flag && !all_ctr)) {
        scout_host::set_error(SCOUT_ERR_INVALID_ARGUMENT, "K1 beside K2: %d SMs", sms);
        return SCOUT_ERR_INVALID_ARGUMENT;
    }
    for (int i = 0; i < n; ++i)
        if (!layers[i].done_flag || !layers[i].done_ctr) {
            scout_host::set_error(SCOUT_ERR_INVALID_ARGUMENT, "K1 beside K2: every layer publishes a flag");
            return SCOUT_ERR_INVALID_ARGUMENT;
        }
    return k1_launch_batch(layers, n, st, -sms, 1, all_ctr, all_flag, all_token);
}

static int k1_launch_batch(const scout_topk_args* layers, int n, cudaStream_t st, int slots, int nowait,
                           unsigned* all_ctr, unsigned* all_flag, unsigned all_token) {
    using namespace scout_host;
    if (n < 1 || n > K1_MAX_LAYERS) {
        set_error(SCOUT_ERR_INVALID_ARGUMENT, "K1 batch: %d layers (max %d)", n, K1_MAX_LAYERS);
        return SCOUT_ERR_INVALID_ARGUMENT;
    }
    for (int i = 0; i < n; ++i) {
        const int rc = validate(layers[i]);
        if (rc != SCOUT_OK) return rc;
        if (layers[i].n_units != layers[0].n_units || layers[i].group != layers[0].group ||
            layers[i].nb_stride != layers[0].nb_stride || layers[i].digest_dtype != layers[0].digest_dtype ||
            layers[i].method != layers[0].method) {
            set_error(SCOUT_ERR_INVALID_ARGUMENT, "K1 batch: layers must share shape / dtype / method");
            return SCOUT_ERR_INVALID_ARGUMENT;
        }
    }
    if (layers[0].n_units == 0) return SCOUT_OK;
    static thread_local K1Batch b;
    b.n = n;
    b.nowait = nowait;
    b.slots = slots;
    b.all_ctr = all_ctr;
    b.all_flag = all_flag;
    b.all_token = all_token;
    for (int i = 0; i < n; ++i) b.a[i] = layers[i];
    if (nowait) b.a[0].flags |= SCOUT_LAUNCH_PDL;
    return launch_batch(b, st);
}

extern "C" int scout_score_topk_split_batch(const scout_topk_args* args, int n, void* stream) {
    if (!args) {
        scout_host::set_error(SCOUT_ERR_INVALID_ARGUMENT, "scout_score_topk_split_batch: null args");
        return SCOUT_ERR_INVALID_ARGUMENT;
    }
    return scout_k1_launch_batch(args, n, static_cast<cudaStream_t>(stream));
}
