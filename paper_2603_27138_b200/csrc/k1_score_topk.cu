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

using namespace scout_dev;

namespace {

constexpr int K1_THREADS = 256;
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

// Scores for one unit. MODE 0: exact minmax (f32 q x f32/bf16 digests, fma),
// MODE 1: generic f64 minmax, MODE 2: generic f64 mean.
template <typename DigT, int G, int MODE>
__device__ __forceinline__ void score_unit(const scout_topk_args& a, int u, int nb, const double* qs,
                                           uint64_t* keys) {
    const size_t ns = static_cast<size_t>(a.nb_stride);
    if constexpr (MODE == 0) {
        const DigT* lo = static_cast<const DigT*>(a.digests) + static_cast<size_t>(u) * 2 * D * ns;
        const DigT* hi = lo + D * ns;
        const int npairs = (nb + 1) >> 1;
        for (int p = threadIdx.x; p < npairs; p += K1_THREADS) {
            const int b0 = 2 * p;
            double acc0 = 0.0, acc1 = 0.0;
#pragma unroll 4
            for (int c = 0; c < D; ++c) {
                double l0, l1, h0, h1;
                if constexpr (sizeof(DigT) == 2) {
                    const __nv_bfloat162 lv = *reinterpret_cast<const __nv_bfloat162*>(lo + c * ns + b0);
                    const __nv_bfloat162 hv = *reinterpret_cast<const __nv_bfloat162*>(hi + c * ns + b0);
                    l0 = widen(lv.x); l1 = widen(lv.y); h0 = widen(hv.x); h1 = widen(hv.y);
                } else {
                    const float2 lv = *reinterpret_cast<const float2*>(lo + c * ns + b0);
                    const float2 hv = *reinterpret_cast<const float2*>(hi + c * ns + b0);
                    l0 = lv.x; l1 = lv.y; h0 = hv.x; h1 = hv.y;
                }
#pragma unroll
                for (int g = 0; g < G; ++g) {
                    const double qv = qs[c * G + g];
                    const bool pos = qv >= 0.0;
                    acc0 = fma(qv, pos ? h0 : l0, acc0);
                    acc1 = fma(qv, pos ? h1 : l1, acc1);
                }
            }
            keys[b0] = score_key(acc0);
            if (a.scores_out) a.scores_out[u * ns + b0] = acc0;
            if (b0 + 1 < nb) {
                keys[b0 + 1] = score_key(acc1);
                if (a.scores_out) a.scores_out[u * ns + b0 + 1] = acc1;
            }
        }
    } else if constexpr (MODE == 1) {
        const double* lo = static_cast<const double*>(a.digests) + static_cast<size_t>(u) * 2 * D * ns;
        const double* hi = lo + D * ns;
        for (int b = threadIdx.x; b < nb; b += K1_THREADS) {
            double acc = 0.0;
            for (int c = 0; c < D; ++c) {
                const double l = lo[c * ns + b], h = hi[c * ns + b];
#pragma unroll
                for (int g = 0; g < G; ++g) {
                    const double qv = qs[c * G + g];
                    acc = __dadd_rn(acc, ref_max(__dmul_rn(qv, l), __dmul_rn(qv, h)));
                }
            }
            keys[b] = score_key(acc);
            if (a.scores_out) a.scores_out[u * ns + b] = acc;
        }
    } else {
        const double* mean = static_cast<const double*>(a.digests) + static_cast<size_t>(u) * D * ns;
        for (int b = threadIdx.x; b < nb; b += K1_THREADS) {
            double acc = 0.0;
            for (int c = 0; c < D; ++c) {
                const double m = mean[c * ns + b];
#pragma unroll
                for (int g = 0; g < G; ++g) acc = __dadd_rn(acc, __dmul_rn(qs[c * G + g], m));
            }
            keys[b] = score_key(acc);
            if (a.scores_out) a.scores_out[u * ns + b] = acc;
        }
    }
}

template <typename DigT, int G, int MODE>
__global__ void __launch_bounds__(K1_THREADS) score_topk_kernel(const scout_topk_args a) {
    extern __shared__ __align__(16) uint8_t k1_smem[];
    double* qs = reinterpret_cast<double*>(k1_smem);              // [D][G] stacked order
    uint64_t* keys = reinterpret_cast<uint64_t*>(qs + D * G);     // [nb_stride]
    __shared__ uint32_t hist[256];
    __shared__ int warp_tot[K1_WARPS];
    __shared__ uint64_t s_prefix;
    __shared__ int s_krem;
    __shared__ int s_tok[2];

    const int u = blockIdx.x;
    const int tid = threadIdx.x;
    int ntok = a.n_tokens[u];
    ntok = max(0, min(ntok, a.nb_stride * BS));
    const int nb = (ntok + BS - 1) / BS;
    const int tail = ntok - (nb - 1) * BS;

    // stage the G queries in stacked channel-major order q_s[c*G+g] (double)
    for (int i = tid; i < D * G; i += K1_THREADS) {
        const int g = i / D, c = i % D;
        double v;
        if constexpr (MODE == 0) v = static_cast<const float*>(a.q)[(static_cast<size_t>(u) * G + g) * D + c];
        else v = static_cast<const double*>(a.q)[(static_cast<size_t>(u) * G + g) * D + c];
        qs[c * G + g] = v;
    }
    if (tid < 2) s_tok[tid] = 0;
    __syncthreads();

    score_unit<DigT, G, MODE>(a, u, nb, qs, keys);
    __syncthreads();

    const int k = a.k;
    // ---- radix select of the k-th largest key (skipped when everything is selected)
    uint64_t thr = 0;
    int need_eq = 0;  // how many key == thr blocks (lowest ids) to take
    const bool take_all = nb <= k;
    if (!take_all) {
        uint64_t prefix = 0, mask = 0;
        int krem = k;
        for (int pass = 0; pass < 8; ++pass) {
            const int shift = 56 - 8 * pass;
            hist[tid] = 0;  // K1_THREADS == 256 bins
            __syncthreads();
            for (int b = tid; b < nb; b += K1_THREADS) {
                const uint64_t key = keys[b];
                if ((key & mask) == prefix) atomicAdd(&hist[(key >> shift) & 255u], 1u);
            }
            __syncthreads();
            if (tid < 32) {
                // lane l owns bins 255-8l ... 248-8l (descending)
                uint32_t cnt[8];
                uint32_t local = 0;
#pragma unroll
                for (int i = 0; i < 8; ++i) {
                    cnt[i] = hist[255 - 8 * tid - i];
                    local += cnt[i];
                }
                uint32_t incl = local;
#pragma unroll
                for (int o = 1; o < 32; o <<= 1) {
                    const uint32_t y = __shfl_up_sync(0xffffffffu, incl, o);
                    if (tid >= o) incl += y;
                }
                const uint32_t excl = incl - local;
                const bool hit = excl < static_cast<uint32_t>(krem) && incl >= static_cast<uint32_t>(krem);
                if (hit) {
                    uint32_t cum = excl;
                    int digit = 0;
                    uint32_t above = 0;
#pragma unroll
                    for (int i = 0; i < 8; ++i) {
                        if (cum + cnt[i] >= static_cast<uint32_t>(krem)) {
                            digit = 255 - 8 * tid - i;
                            above = cum;
                            break;
                        }
                        cum += cnt[i];
                    }
                    s_prefix = prefix | (static_cast<uint64_t>(digit) << shift);
                    s_krem = krem - static_cast<int>(above);
                }
            }
            __syncthreads();
            prefix = s_prefix;
            krem = s_krem;
            mask |= 0xFFull << shift;
        }
        thr = prefix;
        need_eq = krem;
    }

    // ---- selection flags in id order: contiguous chunks per thread
    const int chunk = (nb + K1_THREADS - 1) / K1_THREADS;
    const int b_begin = min(nb, tid * chunk), b_end = min(nb, b_begin + chunk);
    int total;
    int eq_rank = 0;
    if (!take_all) {
        int eq_local = 0;
        for (int b = b_begin; b < b_end; ++b) eq_local += keys[b] == thr;
        eq_rank = block_exclusive_scan(eq_local, warp_tot, &total);
    }
    // selected count and resident count per chunk
    const int32_t* table = a.block_table ? a.block_table + static_cast<size_t>(u) * a.nb_stride : nullptr;
    int sel_local = 0, res_local = 0;
    {
        int er = eq_rank;
        for (int b = b_begin; b < b_end; ++b) {
            bool sel = take_all;
            if (!take_all) {
                const uint64_t key = keys[b];
                if (key > thr) sel = true;
                else if (key == thr) { sel = er < need_eq; ++er; }
            }
            if (sel) {
                ++sel_local;
                if (table && table[b] >= 0) ++res_local;
            }
        }
    }
    const int packed = block_exclusive_scan(sel_local | (res_local << 16), warp_tot, &total);
    int sel_pos = packed & 0xFFFF, res_pos = packed >> 16;
    int tok_res = 0, tok_cpu = 0;
    {
        int er = eq_rank;
        const size_t row = static_cast<size_t>(u) * a.k_stride;
        for (int b = b_begin; b < b_end; ++b) {
            bool sel = take_all;
            if (!take_all) {
                const uint64_t key = keys[b];
                if (key > thr) sel = true;
                else if (key == thr) { sel = er < need_eq; ++er; }
            }
            if (!sel) continue;
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
    }
}

template <typename DigT, int MODE>
int launch_g(const scout_topk_args& a, cudaStream_t st) {
    const size_t smem = static_cast<size_t>(D) * a.group * 8 + static_cast<size_t>(a.nb_stride) * 8;
    auto go = [&](auto kern) {
        static size_t configured = 0;  // per instantiation; the attribute call is not free
        if (smem > 48 * 1024 && smem > configured) {
            cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, static_cast<int>(smem));
            configured = smem;
        }
        kern<<<a.n_units, K1_THREADS, smem, st>>>(a);
    };
    switch (a.group) {
        case 1: go(score_topk_kernel<DigT, 1, MODE>); break;
        case 2: go(score_topk_kernel<DigT, 2, MODE>); break;
        case 4: go(score_topk_kernel<DigT, 4, MODE>); break;
        case 8: go(score_topk_kernel<DigT, 8, MODE>); break;
        default: return -1;
    }
    return 0;
}

}  // namespace

extern "C" int scout_score_topk_split(const scout_topk_args* args, void* stream) {
    using namespace scout_host;
    if (!args) {
        set_error(SCOUT_ERR_INVALID_ARGUMENT, "scout_score_topk_split: null args");
        return SCOUT_ERR_INVALID_ARGUMENT;
    }
    const scout_topk_args& a = *args;
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
    if (a.n_units == 0) return SCOUT_OK;
    if (!a.q || !a.digests || !a.n_tokens) {
        set_error(SCOUT_ERR_INVALID_ARGUMENT, "scout_score_topk_split: null q/digests/n_tokens");
        return SCOUT_ERR_INVALID_ARGUMENT;
    }
    auto st = static_cast<cudaStream_t>(stream);
    int rc = -1;
    if (a.method == SCOUT_DIGEST_MINMAX) {
        if (a.digest_dtype == SCOUT_BF16) rc = launch_g<__nv_bfloat16, 0>(a, st);
        else if (a.digest_dtype == SCOUT_F32) rc = launch_g<float, 0>(a, st);
        else if (a.digest_dtype == SCOUT_F64) rc = launch_g<double, 1>(a, st);
    } else if (a.method == SCOUT_DIGEST_MEAN) {
        if (a.digest_dtype == SCOUT_F64) rc = launch_g<double, 2>(a, st);
    }
    if (rc != 0) {
        set_error(SCOUT_ERR_UNSUPPORTED, "scout_score_topk_split: method %d with digest dtype %d unsupported",
                  a.method, a.digest_dtype);
        return SCOUT_ERR_UNSUPPORTED;
    }
    return check_launch("scout_score_topk_split");
}
