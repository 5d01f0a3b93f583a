// K6 — layer-ahead query prediction on the 5th-gen tensor cores.
//
// Replaces, for a batch of requests,
//   normed = rms_normalize(x)                 reference numerics.hpp:99-108
//   q_pred = predict_next_query(normed, W_Q)  model.hpp:215-217 (= vec_mat, numerics.hpp:111-123)
// as called at engine.hpp:224 / :237 for layer i+1 from layer i's input.
//
// Shapes (Qwen3-32B): x [batch][hidden=5120], W_Q^{i+1} [hidden][Hq*d = 8192]
// (the reference's hidden x out layout). The GEMM has M = 8192 output
// features, N = batch (<= 256) and K = hidden: with a small batch it streams
// the weights once and is HBM-bound (84 MB per layer at bf16).
//
// Layouts (both operands K-major, UMMA "SWIZZLE_NONE" canonical form): core
// matrices of 8 rows x 8 bf16 (128 contiguous bytes, row stride 16 B); a
// [rows x 128] K-chunk of an operand is [row group g][k core c (16)][8 rows][8]
// (2 KiB per 8-row group), so LBO (next K core) = 128 B, SBO (next 8-row
// group) = 2 KiB, and the K=16 MMA step s starts 256 B further.
//   * weights are packed ONCE (scout_qpred_pack_weights, model load) into
//     [m_tile (128 features)][k chunk (128)][32 KiB core-matrix tile];
//   * the normalised batch is packed per call (K6a, rms_normalize fused) into
//     [k chunk][N/8 groups x 1 KiB].
// K6b: stream-K over (m_tile, k chunk). Warp 0 lane 0 streams A (32 KiB) + B
// (N*128 B) chunks with 1-D bulk copies (TMA engine) into an mbarrier ring;
// warp 1 lane 0 issues tcgen05.mma.cta_group::1.kind::f16 (M=128, N, K=16)
// into a TMEM accumulator and tcgen05.commit frees each stage; after the last
// chunk all four warps drain TMEM (tcgen05.ld 32x32b: warp w owns lanes
// 32w..32w+31 = features) into an fp32 partial. The last CTA of an m_tile
// sums the k-split partials in split order (deterministic) and writes q_pred
// [batch][features] in f32 and/or bf16 (K1's query input).
#include "scout_common.cuh"

#include <cstdlib>

using namespace scout_dev;

namespace {

constexpr int QP_M = 128;                 // features per tile (UMMA M)
constexpr int QP_KC = 128;                // K per chunk / stage (bigger transfers: fewer round trips)
constexpr int QP_A_BYTES = QP_M * QP_KC * 2;  // 32 KiB
constexpr int QP_GROUP = 8 * QP_KC;           // elements of one 8-row group of a chunk
constexpr uint32_t QP_SBO = QP_GROUP * 2;     // bytes between 8-row groups
constexpr int QP_THREADS = 128;
constexpr int QP_MAXN = 256;

__device__ __forceinline__ uint64_t umma_desc(uint32_t saddr, uint32_t lbo, uint32_t sbo) {
    // SM100 shared-memory matrix descriptor: start >> 4 [0,14), LBO >> 4 [16,30),
    // SBO >> 4 [32,46), version 1 [46,48), base offset 0, SWIZZLE_NONE (0) [61,64)
    return static_cast<uint64_t>((saddr >> 4) & 0x3FFFu) | (static_cast<uint64_t>((lbo >> 4) & 0x3FFFu) << 16) |
           (static_cast<uint64_t>((sbo >> 4) & 0x3FFFu) << 32) | (1ull << 46);
}
// kind::f16 instruction descriptor: D f32, A/B bf16, both K-major, N >> 3, M >> 4
__host__ __device__ constexpr uint32_t umma_idesc_bf16(int M, int N) {
    return (1u << 4) | (1u << 7) | (1u << 10) | (static_cast<uint32_t>(N >> 3) << 17) |
           (static_cast<uint32_t>(M >> 4) << 24);
}

__device__ __forceinline__ void tc_fence_after() { asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory"); }
__device__ __forceinline__ void tc_fence_before() { asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory"); }

__device__ __forceinline__ void umma_bf16(uint32_t tmem_d, uint64_t adesc, uint64_t bdesc, uint32_t idesc,
                                          uint32_t accumulate) {
    asm volatile(
        "{\n.reg .pred p;\nsetp.ne.b32 p, %4, 0;\n"
        "tcgen05.mma.cta_group::1.kind::f16 [%0], %1, %2, %3, p;\n}\n" ::"r"(tmem_d),
        "l"(adesc), "l"(bdesc), "r"(idesc), "r"(accumulate)
        : "memory");
}
__device__ __forceinline__ void umma_commit(uint64_t* bar) {
    asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];" ::"r"(smem_u32(bar))
                 : "memory");
}

// rms_normalize (numerics.hpp:99-108: ms = sum x^2 in double, rms = sqrt(ms/n),
// rms == 0 -> x unchanged) fused with the pack of x^ into the B-operand
// layout, bf16. One CTA per request; padded rows [batch, N) are zero. A thread
// owns 8 consecutive k (one 16-byte core-matrix row): two float4 loads, one
// 16-byte store. hidden % 128 == 0.
__global__ void __launch_bounds__(256) qpred_pack_x_kernel(const float* __restrict__ x, int hidden, int batch, int n_pad,
                                                          __nv_bfloat16* __restrict__ xb) {
    __shared__ double red[8];
    const int b = blockIdx.x, tid = threadIdx.x;
    griddep_launch_dependents();  // the GEMM may start streaming weights now
    const int n8 = hidden / 8;
    const float4* xr = reinterpret_cast<const float4*>(x + static_cast<size_t>(b) * hidden);
    double inv = 1.0;
    if (b < batch) {
        double s = 0.0;
        for (int i = tid; i < n8; i += 256) {
            const float4 u = xr[2 * i], v = xr[2 * i + 1];
            s += static_cast<double>(u.x) * u.x + static_cast<double>(u.y) * u.y + static_cast<double>(u.z) * u.z +
                 static_cast<double>(u.w) * u.w + static_cast<double>(v.x) * v.x + static_cast<double>(v.y) * v.y +
                 static_cast<double>(v.z) * v.z + static_cast<double>(v.w) * v.w;
        }
#pragma unroll
        for (int o = 16; o; o >>= 1) s += __shfl_xor_sync(0xffffffffu, s, o);
        if ((tid & 31) == 0) red[tid >> 5] = s;
        __syncthreads();
        double t = 0.0;
        for (int w = 0; w < 8; ++w) t += red[w];  // fixed order: deterministic
        const double rms = sqrt(t / hidden);
        inv = rms == 0.0 ? 1.0 : 1.0 / rms;
    }
    const int g = b >> 3, r = b & 7;
    for (int i = tid; i < n8; i += 256) {
        const int k = 8 * i, kc = k / QP_KC, c = (k % QP_KC) >> 3;
        uint4 pk = make_uint4(0u, 0u, 0u, 0u);
        if (b < batch) {
            const float4 u = xr[2 * i], v = xr[2 * i + 1];
            pk.x = pack_bf16(static_cast<float>(u.x * inv), static_cast<float>(u.y * inv));
            pk.y = pack_bf16(static_cast<float>(u.z * inv), static_cast<float>(u.w * inv));
            pk.z = pack_bf16(static_cast<float>(v.x * inv), static_cast<float>(v.y * inv));
            pk.w = pack_bf16(static_cast<float>(v.z * inv), static_cast<float>(v.w * inv));
        }
        *reinterpret_cast<uint4*>(xb + static_cast<size_t>(kc) * n_pad * QP_KC + static_cast<size_t>(g) * QP_GROUP + c * 64 +
                                  r * 8) = pk;
    }
}

// W [hidden][n_out] bf16 (the reference's layout) -> [m_tile][k chunk][16 KiB tile]
__global__ void qpred_pack_w_kernel(const __nv_bfloat16* __restrict__ w, int hidden, int n_out,
                                    __nv_bfloat16* __restrict__ wp) {
    const size_t total = static_cast<size_t>(hidden) * n_out;
    const int nkc = hidden / QP_KC;
    for (size_t i = blockIdx.x * static_cast<size_t>(blockDim.x) + threadIdx.x; i < total;
         i += static_cast<size_t>(gridDim.x) * blockDim.x) {
        const int k = static_cast<int>(i / n_out), n = static_cast<int>(i % n_out);  // coalesced reads
        const int mt = n / QP_M, m = n % QP_M, kc = k / QP_KC, kk = k % QP_KC;
        const size_t off = (static_cast<size_t>(mt) * nkc + kc) * (QP_M * QP_KC) + (m >> 3) * QP_GROUP + (kk >> 3) * 64 +
                           (m & 7) * 8 + (kk & 7);
        wp[off] = w[i];
    }
}

struct QpArgs {
    const __nv_bfloat16* wp;  // packed weights [tile][chunk][16 KiB] = units in stream order
    const __nv_bfloat16* xb;  // packed normalised batch [chunk][n_pad rows]
    float* out_f32;           // [batch][n_out] (optional)
    __nv_bfloat16* out_bf16;  // [batch][n_out] (optional)
    float* partial;           // [grid][2][128][n_pad]: a CTA's partial of its first / second tile
    int* counters;            // [n_out / 128], zero; left zeroed
    int hidden, n_out, batch, n_pad, nst;
    int pair;                 // 1: cluster pairs, CTA 2t+r holds K half r of tile t; halves meet in shared memory
};

// CTA holding unit u when T units are cut into `grid` equal ranges
__device__ __forceinline__ int cta_of(long long u, long long T, int grid) {
    return static_cast<int>(((u + 1) * grid - 1) / T);
}

// Stream-K over (feature tile, K chunk) units on every SM: CTA c takes units
// [T*c/grid, T*(c+1)/grid) of the flattened [tile][chunk] order, i.e. one
// contiguous run of the packed weights covering at most two tiles (grid >=
// tiles). Each tile gets its own TMEM accumulator (n_pad columns); the MMA
// issuer commits a tile's accumulator as soon as its last chunk is issued, so
// the epilogue of the first tile overlaps the streaming of the second. A
// tile held whole by one CTA goes straight to q_pred; a shared tile is
// parked as a partial and its last-arriving CTA sums the holders' partials in
// CTA order (deterministic).
__global__ void __launch_bounds__(QP_THREADS, 1) qpred_gemm_kernel(const QpArgs a) {
    extern __shared__ __align__(1024) uint8_t qsm[];
    __shared__ uint64_t full[8], empty[8], tfull[2];
    __shared__ uint32_t tmem_base;
    __shared__ int last;
    const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
    const int grid = gridDim.x, c = blockIdx.x;
    const int nkc = a.hidden / QP_KC;
    const long long T = static_cast<long long>(a.n_out / QP_M) * nkc;
    const long long u0 = T * c / grid, u1 = T * (c + 1) / grid;
    const int mt0 = static_cast<int>(u0 / nkc);
    const int nseg = (u1 - 1) / nkc > mt0 ? 2 : 1;
    const int nst = a.nst;
    const uint32_t b_bytes = static_cast<uint32_t>(a.n_pad) * QP_KC * 2;
    const uint32_t stage_bytes = QP_A_BYTES + b_bytes;
    const uint32_t need = 2u * static_cast<uint32_t>(a.n_pad);
    const uint32_t tcols = need <= 32 ? 32 : (need <= 64 ? 64 : (need <= 128 ? 128 : (need <= 256 ? 256 : 512)));

    if (tid == 0) {
        for (int i = 0; i < nst; ++i) {
            mbar_init(&full[i], 1);
            mbar_init(&empty[i], 1);
        }
        mbar_init(&tfull[0], 1);
        mbar_init(&tfull[1], 1);
        fence_mbar_init();
    }
    if (warp == 2) {  // TMEM: two accumulators of n_pad fp32 columns x 128 lanes
        asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(smem_u32(&tmem_base)),
                     "r"(tcols)
                     : "memory");
        asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;" ::: "memory");
    }
    tc_fence_before();
    __syncthreads();
    tc_fence_after();
    const uint32_t tmem = tmem_base;
    const int nunit = static_cast<int>(u1 - u0);

    if (warp == 0 && lane == 0) {
        // ---- producer: the CTA's run of packed weights + the matching batch chunks
        const uint64_t pol = policy_evict_first();
        const uint8_t* wsrc = reinterpret_cast<const uint8_t*>(a.wp) + static_cast<size_t>(u0) * QP_A_BYTES;
        const uint8_t* xsrc = reinterpret_cast<const uint8_t*>(a.xb);
        // the first ring's weights go out before the batch is packed (PDL)
        const int npre = min(nst, nunit);
        for (int i = 0; i < npre; ++i) {
            mbar_arrive_expect_tx(&full[i], stage_bytes);
            bulk_g2s_evict_first(qsm + static_cast<size_t>(i) * stage_bytes, wsrc + static_cast<size_t>(i) * QP_A_BYTES,
                                 QP_A_BYTES, &full[i], pol);
        }
        griddep_wait();
        // chunk index within the tile, advanced incrementally (no divisions in the loop)
        int kc = static_cast<int>(u0 % nkc);
        for (int i = 0; i < npre; ++i) {
            bulk_g2s(qsm + static_cast<size_t>(i) * stage_bytes + QP_A_BYTES, xsrc + static_cast<size_t>(kc) * b_bytes,
                     b_bytes, &full[i]);
            if (++kc == nkc) kc = 0;
        }
        for (int i = npre, s = npre % nst, ph = (npre / nst) & 1; i < nunit; ++i) {
            mbar_wait(&empty[s], ph ^ 1);
            uint8_t* st = qsm + static_cast<size_t>(s) * stage_bytes;
            mbar_arrive_expect_tx(&full[s], stage_bytes);
            bulk_g2s_evict_first(st, wsrc + static_cast<size_t>(i) * QP_A_BYTES, QP_A_BYTES, &full[s], pol);
            bulk_g2s(st + QP_A_BYTES, xsrc + static_cast<size_t>(kc) * b_bytes, b_bytes, &full[s]);
            if (++kc == nkc) kc = 0;
            if (++s == nst) { s = 0; ph ^= 1; }
        }
    } else if (warp == 1 && lane == 0) {
        // ---- MMA issuer: 4 x (M=128, N=n_pad, K=16) per chunk, accumulator per tile.
        // The issuing thread is the pipeline's serial path: no divisions in the loop.
        const uint32_t idesc = umma_idesc_bf16(QP_M, a.n_pad);
        int kc = static_cast<int>(u0 % nkc), seg = 0, s = 0, ph = 0;
        for (int i = 0; i < nunit; ++i) {
            const bool first = i == 0 || kc == 0;
            mbar_wait(&full[s], ph);
            tc_fence_after();
            const uint32_t sa = smem_u32(qsm + static_cast<size_t>(s) * stage_bytes);
            const uint32_t sb = sa + QP_A_BYTES;
            const uint32_t dcol = tmem + static_cast<uint32_t>(seg * a.n_pad);
#pragma unroll
            for (int k = 0; k < QP_KC / 16; ++k)
                umma_bf16(dcol, umma_desc(sa + 256 * k, 128, QP_SBO), umma_desc(sb + 256 * k, 128, QP_SBO), idesc,
                          (!first || k > 0) ? 1u : 0u);
            umma_commit(&empty[s]);  // the stage is free once these MMAs have read it
            if (i == nunit - 1 || kc == nkc - 1) umma_commit(&tfull[seg]);  // the tile's accumulator is done
            if (++kc == nkc) { kc = 0; ++seg; }
            if (++s == nst) { s = 0; ph ^= 1; }
        }
    }
    __syncwarp();
    // ---- epilogue, per tile held (thread = feature row, 32 batch columns per tcgen05.ld)
    auto tmem_load = [&](uint32_t col, float (&f)[32]) {
        uint32_t v[32];
        const uint32_t taddr = tmem + (static_cast<uint32_t>(warp * 32) << 16) + col;
        asm volatile(
            "tcgen05.ld.sync.aligned.32x32b.x32.b32 {%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15,"
            "%16,%17,%18,%19,%20,%21,%22,%23,%24,%25,%26,%27,%28,%29,%30,%31}, [%32];"
            : "=r"(v[0]), "=r"(v[1]), "=r"(v[2]), "=r"(v[3]), "=r"(v[4]), "=r"(v[5]), "=r"(v[6]), "=r"(v[7]),
              "=r"(v[8]), "=r"(v[9]), "=r"(v[10]), "=r"(v[11]), "=r"(v[12]), "=r"(v[13]), "=r"(v[14]), "=r"(v[15]),
              "=r"(v[16]), "=r"(v[17]), "=r"(v[18]), "=r"(v[19]), "=r"(v[20]), "=r"(v[21]), "=r"(v[22]),
              "=r"(v[23]), "=r"(v[24]), "=r"(v[25]), "=r"(v[26]), "=r"(v[27]), "=r"(v[28]), "=r"(v[29]),
              "=r"(v[30]), "=r"(v[31])
            : "r"(taddr));
        asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory");
#pragma unroll
        for (int j = 0; j < 32; ++j) f[j] = __uint_as_float(v[j]);
    };
    const int ngrp = (a.n_pad + 31) / 32;
    if (a.pair) {
        // ---- cluster pair: rank 1 drops its accumulator into rank 0's shared
        // memory (past the ring), a cluster barrier publishes it, rank 0 adds
        // its own and writes the tile. Replaces the partials' round trip through
        // L2 (store, fence, counter, reload) for the default 2-CTAs-per-tile grid.
        uint32_t rank;
        asm volatile("mov.u32 %0, %%cluster_ctarank;" : "=r"(rank));
        float* recv = reinterpret_cast<float*>(qsm + static_cast<size_t>(nst) * stage_bytes);  // [128][n_pad]
        const int row = warp * 32 + lane;
        mbar_wait(&tfull[0], 0);
        __syncwarp();
        tc_fence_after();
        if (rank == 1) {
            uint32_t remote;
            asm volatile("mapa.shared::cluster.u32 %0, %1, 0;" : "=r"(remote) : "r"(smem_u32(recv + row * a.n_pad)));
            for (int grp = 0; grp < ngrp; ++grp) {
                float f[32];
                tmem_load(static_cast<uint32_t>(grp * 32), f);
                const int ncol = min(32, a.n_pad - grp * 32);
#pragma unroll
                for (int j = 0; j < 32; j += 4)
                    if (j < ncol)
                        asm volatile("st.shared::cluster.v4.f32 [%0], {%1, %2, %3, %4};" ::"r"(remote + 4u * (grp * 32 + j)),
                                     "f"(f[j]), "f"(f[j + 1]), "f"(f[j + 2]), "f"(f[j + 3])
                                     : "memory");
            }
        }
        asm volatile("barrier.cluster.arrive.release.aligned;\n\tbarrier.cluster.wait.acquire.aligned;" ::: "memory");
        if (rank == 0) {
            const int feat = mt0 * QP_M + row;
            for (int grp = 0; grp < ngrp; ++grp) {
                float f[32];
                tmem_load(static_cast<uint32_t>(grp * 32), f);
                const float* rp = recv + row * a.n_pad + grp * 32;
#pragma unroll
                for (int j = 0; j < 32; ++j) {
                    const int bcol = grp * 32 + j;
                    if (bcol < a.batch) {
                        const float v = f[j] + rp[j];  // K half 0 + K half 1: the same order for every call
                        if (a.out_f32) a.out_f32[static_cast<size_t>(bcol) * a.n_out + feat] = v;
                        if (a.out_bf16) a.out_bf16[static_cast<size_t>(bcol) * a.n_out + feat] = __float2bfloat16_rn(v);
                    }
                }
            }
        }
    }
    for (int seg = 0; seg < (a.pair ? 0 : nseg); ++seg) {
        const int mt = mt0 + seg;
        const int feat = mt * QP_M + warp * 32 + lane;
        const long long t0 = static_cast<long long>(mt) * nkc, t1 = t0 + nkc;  // the tile's units
        const bool whole = u0 <= t0 && u1 >= t1;
        mbar_wait(&tfull[seg], 0);
        __syncwarp();  // tcgen05.ld is .sync.aligned: reconverge after the spin
        tc_fence_after();
        for (int grp = 0; grp < ngrp; ++grp) {
            float f[32];
            tmem_load(static_cast<uint32_t>(seg * a.n_pad + grp * 32), f);
            if (whole) {
#pragma unroll
                for (int j = 0; j < 32; ++j) {
                    const int bcol = grp * 32 + j;
                    if (bcol < a.batch) {
                        if (a.out_f32) a.out_f32[static_cast<size_t>(bcol) * a.n_out + feat] = f[j];
                        if (a.out_bf16) a.out_bf16[static_cast<size_t>(bcol) * a.n_out + feat] = __float2bfloat16_rn(f[j]);
                    }
                }
            } else {
                float* part = a.partial + ((static_cast<size_t>(c) * 2 + seg) * QP_M + warp * 32 + lane) * a.n_pad + grp * 32;
                const int ncol = min(32, a.n_pad - grp * 32);  // n_pad is a multiple of 16
#pragma unroll
                for (int j = 0; j < 32; j += 4)
                    if (j < ncol) *reinterpret_cast<float4*>(part + j) = make_float4(f[j], f[j + 1], f[j + 2], f[j + 3]);
            }
        }
        if (whole) continue;
        __threadfence();
        __syncthreads();
        const int cf = cta_of(t0, T, grid), cl = cta_of(t1 - 1, T, grid);
        if (tid == 0) last = atomicAdd(&a.counters[mt], 1) == cl - cf;
        __syncthreads();
        if (!last) continue;
        __threadfence();
        for (int grp = 0; grp < ngrp; ++grp) {
            const int ncol = min(32, a.n_pad - grp * 32);
            float acc[32];
            for (int h = cf; h <= cl; ++h) {
                // holder h parked this tile as its first (seg 0) or second (seg 1) tile
                const int hseg = static_cast<int>((T * h / grid) / nkc) == mt ? 0 : 1;
                const float* src = a.partial + ((static_cast<size_t>(h) * 2 + hseg) * QP_M + warp * 32 + lane) * a.n_pad + grp * 32;
                float p[32];
#pragma unroll
                for (int j = 0; j < 32; j += 4) {
                    const float4 t = j < ncol ? __ldcg(reinterpret_cast<const float4*>(src + j)) : make_float4(0.f, 0.f, 0.f, 0.f);
                    p[j] = t.x; p[j + 1] = t.y; p[j + 2] = t.z; p[j + 3] = t.w;
                }
#pragma unroll
                for (int j = 0; j < 32; ++j) acc[j] = h == cf ? p[j] : acc[j] + p[j];
            }
#pragma unroll
            for (int j = 0; j < 32; ++j) {
                const int bcol = grp * 32 + j;
                if (bcol < a.batch) {
                    if (a.out_f32) a.out_f32[static_cast<size_t>(bcol) * a.n_out + feat] = acc[j];
                    if (a.out_bf16) a.out_bf16[static_cast<size_t>(bcol) * a.n_out + feat] = __float2bfloat16_rn(acc[j]);
                }
            }
        }
        if (tid == 0) a.counters[mt] = 0;
    }
    tc_fence_before();
    __syncthreads();
    if (warp == 2)
        asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(tmem), "r"(tcols) : "memory");
}

int num_sms_k6() {
    static int n = 0;
    if (n == 0) {
        int dev = 0;
        cudaGetDevice(&dev);
        cudaDeviceGetAttribute(&n, cudaDevAttrMultiProcessorCount, dev);
        if (n <= 0) n = 148;
    }
    return n;
}

}  // namespace

// workspace: packed batch | tile counters | partials [grid][2][128][n_pad]
extern "C" size_t scout_qpred_workspace_bytes(int hidden, int n_out, int batch, int max_ctas) {
    if (hidden <= 0 || n_out <= 0 || batch <= 0) return 0;
    size_t grid = static_cast<size_t>(max_ctas > 0 ? max_ctas : 1024);  // covers any grid a call picks
    if (grid < static_cast<size_t>(n_out / QP_M)) grid = static_cast<size_t>(n_out / QP_M);
    const size_t n_pad = (static_cast<size_t>(batch) + 15) / 16 * 16;
    const size_t xb = static_cast<size_t>(hidden) * n_pad * 2;
    const size_t ctr = (static_cast<size_t>(n_out) / QP_M) * 4;
    const size_t part = grid * 2 * QP_M * n_pad * 4;
    return ((xb + 255) / 256 + (ctr + 255) / 256 + (part + 255) / 256) * 256;
}

extern "C" int scout_qpred_pack_weights(const void* w, int hidden, int n_out, void* w_packed, void* stream) {
    using namespace scout_host;
    if (!w || !w_packed || hidden <= 0 || n_out <= 0 || hidden % QP_KC || n_out % QP_M) {
        set_error(SCOUT_ERR_INVALID_ARGUMENT, "scout_qpred_pack_weights: hidden %% 128 and n_out %% 128 must be 0");
        return SCOUT_ERR_INVALID_ARGUMENT;
    }
    qpred_pack_w_kernel<<<1184, 256, 0, static_cast<cudaStream_t>(stream)>>>(
        static_cast<const __nv_bfloat16*>(w), hidden, n_out, static_cast<__nv_bfloat16*>(w_packed));
    return check_launch("scout_qpred_pack_weights");
}

extern "C" int scout_predict_query(const float* x, int batch, int hidden, const void* w_packed, int n_out,
                                   float* out_f32, void* out_bf16, void* workspace, size_t workspace_bytes,
                                   int max_ctas, void* stream) {
    using namespace scout_host;
    if (!x || !w_packed || !workspace || batch <= 0 || batch > QP_MAXN || hidden <= 0 || hidden % QP_KC ||
        n_out <= 0 || n_out % QP_M || (!out_f32 && !out_bf16)) {
        set_error(SCOUT_ERR_INVALID_ARGUMENT,
                  "predict_next_query: bad arguments (batch 1..256, hidden %% 128, n_out %% 128, an output)");
        return SCOUT_ERR_INVALID_ARGUMENT;
    }
    const int tiles = n_out / QP_M, nkc = hidden / QP_KC;
    const long long T = static_cast<long long>(tiles) * nkc;
    // default: a whole number of CTAs per tile (64 tiles on 148 SMs -> 128 CTAs,
    // half a tile each): every tile has the same holders and one reduction,
    // which beats spreading over all SMs with two partial tiles per CTA
    // (tools/debug/time_qpred.py: 21.8 vs 25.8 us per Qwen3-32B layer)
    int grid = max_ctas > 0 ? max_ctas : (tiles <= num_sms_k6() ? tiles * (num_sms_k6() / tiles) : num_sms_k6());
    if (grid > 1024) grid = 1024;
    if (grid < tiles) grid = tiles;  // a CTA's run must not span more than two tiles
    if (grid > T) grid = static_cast<int>(T);
    if (workspace_bytes < scout_qpred_workspace_bytes(hidden, n_out, batch, grid)) {
        set_error(SCOUT_ERR_INVALID_ARGUMENT, "predict_next_query: workspace too small");
        return SCOUT_ERR_INVALID_ARGUMENT;
    }
    const int n_pad = (batch + 15) / 16 * 16;
    auto st = static_cast<cudaStream_t>(stream);
    uint8_t* ws = static_cast<uint8_t*>(workspace);
    const size_t xb_bytes = (static_cast<size_t>(hidden) * n_pad * 2 + 255) / 256 * 256;
    const size_t ctr_bytes = (static_cast<size_t>(tiles) * 4 + 255) / 256 * 256;
    auto* xb = reinterpret_cast<__nv_bfloat16*>(ws);
    auto* ctr = reinterpret_cast<int*>(ws + xb_bytes);
    auto* part = reinterpret_cast<float*>(ws + xb_bytes + ctr_bytes);
    qpred_pack_x_kernel<<<n_pad, 256, 0, st>>>(x, hidden, batch, n_pad, xb);
    QpArgs a{static_cast<const __nv_bfloat16*>(w_packed), xb, out_f32, static_cast<__nv_bfloat16*>(out_bf16), part, ctr,
             hidden, n_out, batch, n_pad, 0, 0};
    // cluster pairs when every tile is exactly two K halves (the default grid)
    static const bool pair_env = [] {
        const char* e = getenv("SCOUT_QP_PAIR");
        return e ? atoi(e) != 0 : true;
    }();
    a.pair = pair_env && grid == 2 * tiles && nkc % 2 == 0 && n_pad <= 64;
    const uint32_t stage = QP_A_BYTES + static_cast<uint32_t>(n_pad) * QP_KC * 2;
    const uint32_t recv = a.pair ? static_cast<uint32_t>(QP_M) * n_pad * 4 : 0u;
    int nst = static_cast<int>((200u * 1024u) / stage);
    if (const char* e = getenv("SCOUT_QP_NST")) nst = atoi(e);  // tuning
    if (nst > 8) nst = 8;
    while (nst > 2 && static_cast<size_t>(nst) * stage + recv > 224u * 1024u) --nst;
    if (nst < 2) nst = 2;
    a.nst = nst;
    const size_t smem = static_cast<size_t>(nst) * stage + recv;
    ensure_smem(reinterpret_cast<const void*>(qpred_gemm_kernel), smem);
    launch(qpred_gemm_kernel, dim3(grid), dim3(QP_THREADS), smem, st, true, a, a.pair ? 2 : 1);
    return check_launch("scout_predict_query");
}
