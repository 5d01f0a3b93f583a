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
// [rows x 64] K-chunk of an operand is [row group g][k core c (8)][8 rows][8]
// (1 KiB per 8-row group), so LBO (next K core) = 128 B, SBO (next 8-row
// group) = 1 KiB, and the K=16 MMA step s starts 256 B further.
//   * weights are packed ONCE (scout_qpred_pack_weights, model load) into
//     [m_tile (128 features)][k chunk (64)][16 KiB core-matrix tile];
//   * the normalised batch is packed per call (K6a, rms_normalize fused) into
//     [k chunk][N/8 groups x 1 KiB].
// K6b: one CTA per (m_tile, k split). Warp 0 lane 0 streams A (16 KiB) + B
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
constexpr int QP_KC = 64;                 // K per chunk / stage
constexpr int QP_A_BYTES = QP_M * QP_KC * 2;  // 16 KiB
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
// 16-byte store. hidden % 64 == 0.
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
        *reinterpret_cast<uint4*>(xb + static_cast<size_t>(kc) * n_pad * QP_KC + static_cast<size_t>(g) * 512 + c * 64 +
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
        const size_t off = (static_cast<size_t>(mt) * nkc + kc) * (QP_M * QP_KC) + (m >> 3) * 512 + (kk >> 3) * 64 +
                           (m & 7) * 8 + (kk & 7);
        wp[off] = w[i];
    }
}

struct QpArgs {
    const __nv_bfloat16* wp;  // packed weights
    const __nv_bfloat16* xb;  // packed normalised batch
    float* out_f32;           // [batch][n_out] (optional)
    __nv_bfloat16* out_bf16;  // [batch][n_out] (optional)
    float* partial;           // [ksplit][n_out][n_pad]
    int* counters;            // [n_out / 128], zero; left zeroed
    int hidden, n_out, batch, n_pad, ksplit, nst;
};

__global__ void __launch_bounds__(QP_THREADS, 1) qpred_gemm_kernel(const QpArgs a) {
    extern __shared__ __align__(1024) uint8_t qsm[];
    __shared__ uint64_t full[8], empty[8], done;
    __shared__ uint32_t tmem_base;
    __shared__ int last;
    const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
    const int mt = blockIdx.x, ks = blockIdx.y;
    const int nkc = a.hidden / QP_KC;
    const int kc0 = static_cast<int>(static_cast<long long>(nkc) * ks / a.ksplit);
    const int kc1 = static_cast<int>(static_cast<long long>(nkc) * (ks + 1) / a.ksplit);
    const int nst = a.nst;
    const uint32_t b_bytes = static_cast<uint32_t>(a.n_pad) * QP_KC * 2;
    const uint32_t stage_bytes = QP_A_BYTES + b_bytes;
    const uint32_t tcols = a.n_pad <= 32 ? 32 : (a.n_pad <= 64 ? 64 : (a.n_pad <= 128 ? 128 : 256));

    if (tid == 0) {
        for (int i = 0; i < nst; ++i) {
            mbar_init(&full[i], 1);
            mbar_init(&empty[i], 1);
        }
        mbar_init(&done, 1);
        fence_mbar_init();
    }
    if (warp == 2) {  // TMEM accumulator: n_pad fp32 columns x 128 lanes
        asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(smem_u32(&tmem_base)),
                     "r"(tcols)
                     : "memory");
        asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;" ::: "memory");
    }
    tc_fence_before();
    __syncthreads();
    tc_fence_after();
    const uint32_t tmem = tmem_base;

    if (warp == 0 && lane == 0) {
        // ---- producer: A (weights) + B (batch) chunks, one bulk copy each
        const uint64_t pol = policy_evict_first();
        const uint8_t* wsrc = reinterpret_cast<const uint8_t*>(a.wp) + static_cast<size_t>(mt) * nkc * QP_A_BYTES;
        const uint8_t* xsrc = reinterpret_cast<const uint8_t*>(a.xb);
        // the first ring's weights go out before the batch is packed (PDL:
        // the pack kernel runs concurrently; its output is only read after
        // griddepcontrol.wait)
        const int npre = min(nst, kc1 - kc0);
        for (int i = 0; i < npre; ++i) {
            mbar_arrive_expect_tx(&full[i], stage_bytes);
            bulk_g2s_evict_first(qsm + static_cast<size_t>(i) * stage_bytes,
                                 wsrc + static_cast<size_t>(kc0 + i) * QP_A_BYTES, QP_A_BYTES, &full[i], pol);
        }
        griddep_wait();
        for (int i = 0; i < npre; ++i)
            bulk_g2s(qsm + static_cast<size_t>(i) * stage_bytes + QP_A_BYTES,
                     xsrc + static_cast<size_t>(kc0 + i) * b_bytes, b_bytes, &full[i]);
        for (int kc = kc0 + npre, i = npre; kc < kc1; ++kc, ++i) {
            const int s = i % nst;
            mbar_wait(&empty[s], ((i / nst) - 1) & 1);
            uint8_t* st = qsm + static_cast<size_t>(s) * stage_bytes;
            mbar_arrive_expect_tx(&full[s], stage_bytes);
            bulk_g2s_evict_first(st, wsrc + static_cast<size_t>(kc) * QP_A_BYTES, QP_A_BYTES, &full[s], pol);
            bulk_g2s(st + QP_A_BYTES, xsrc + static_cast<size_t>(kc) * b_bytes, b_bytes, &full[s]);
        }
    } else if (warp == 1 && lane == 0) {
        // ---- MMA issuer: 4 x (M=128, N=n_pad, K=16) per chunk into TMEM
        const uint32_t idesc = umma_idesc_bf16(QP_M, a.n_pad);
        for (int kc = kc0, i = 0; kc < kc1; ++kc, ++i) {
            const int s = i % nst;
            mbar_wait(&full[s], (i / nst) & 1);
            tc_fence_after();
            const uint32_t sa = smem_u32(qsm + static_cast<size_t>(s) * stage_bytes);
            const uint32_t sb = sa + QP_A_BYTES;
#pragma unroll
            for (int k = 0; k < QP_KC / 16; ++k)
                umma_bf16(tmem, umma_desc(sa + 256 * k, 128, 1024), umma_desc(sb + 256 * k, 128, 1024), idesc,
                          (i > 0 || k > 0) ? 1u : 0u);
            umma_commit(&empty[s]);  // the stage is free once these MMAs have read it
        }
        umma_commit(&done);  // accumulator complete
    }
    __syncwarp();
    // ---- epilogue: TMEM -> registers (thread = feature row, 32 batch columns
    // per tcgen05.ld). One split: straight to q_pred. Several: every CTA parks
    // its partial; the last one of the m_tile adds them in split order
    // (its own from registers), so the sum does not depend on arrival order.
    mbar_wait(&done, 0);
    __syncwarp();  // tcgen05.ld is .sync.aligned: reconverge after the spin
    tc_fence_after();
    const int feat = mt * QP_M + warp * 32 + lane;
    const int ngrp = (a.n_pad + 31) / 32;
    auto tmem_load = [&](int grp, float (&f)[32]) {
        uint32_t v[32];
        const uint32_t taddr = tmem + (static_cast<uint32_t>(warp * 32) << 16) + static_cast<uint32_t>(grp * 32);
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
    auto store_out = [&](int grp, const float (&f)[32]) {
#pragma unroll
        for (int j = 0; j < 32; ++j) {
            const int bcol = grp * 32 + j;
            if (bcol < a.batch) {
                if (a.out_f32) a.out_f32[static_cast<size_t>(bcol) * a.n_out + feat] = f[j];
                if (a.out_bf16) a.out_bf16[static_cast<size_t>(bcol) * a.n_out + feat] = __float2bfloat16_rn(f[j]);
            }
        }
    };
    if (a.ksplit == 1) {
        for (int grp = 0; grp < ngrp; ++grp) {
            float f[32];
            tmem_load(grp, f);
            store_out(grp, f);
        }
    } else {
        float* part = a.partial + (static_cast<size_t>(ks) * a.n_out + feat) * a.n_pad;
        for (int grp = 0; grp < ngrp; ++grp) {
            float f[32];
            tmem_load(grp, f);
            const int ncol = min(32, a.n_pad - grp * 32);  // n_pad is a multiple of 16
#pragma unroll
            for (int j = 0; j < 32; j += 4)
                if (j < ncol) *reinterpret_cast<float4*>(part + grp * 32 + j) = make_float4(f[j], f[j + 1], f[j + 2], f[j + 3]);
        }
        __threadfence();
        __syncthreads();
        if (tid == 0) last = atomicAdd(&a.counters[mt], 1) == a.ksplit - 1;
        __syncthreads();
        if (last) {
            __threadfence();
            for (int grp = 0; grp < ngrp; ++grp) {
                float own[32], acc[32];
                tmem_load(grp, own);
                const int ncol = min(32, a.n_pad - grp * 32);
                // splits two at a time: both loads in flight before the adds
                for (int s2 = 0; s2 < a.ksplit; s2 += 2) {
                    float p[2][32];
#pragma unroll
                    for (int h = 0; h < 2; ++h) {
                        const int sp = s2 + h;
                        if (sp >= a.ksplit) continue;
                        if (sp == ks) {
#pragma unroll
                            for (int j = 0; j < 32; ++j) p[h][j] = own[j];
                        } else {
                            const float* src = a.partial + (static_cast<size_t>(sp) * a.n_out + feat) * a.n_pad + grp * 32;
#pragma unroll
                            for (int j = 0; j < 32; j += 4) {
                                const float4 t = j < ncol ? __ldcg(reinterpret_cast<const float4*>(src + j))
                                                          : make_float4(0.f, 0.f, 0.f, 0.f);
                                p[h][j] = t.x; p[h][j + 1] = t.y; p[h][j + 2] = t.z; p[h][j + 3] = t.w;
                            }
                        }
                    }
#pragma unroll
                    for (int h = 0; h < 2; ++h)
                        if (s2 + h < a.ksplit)
#pragma unroll
                            for (int j = 0; j < 32; ++j) acc[j] = (s2 + h) == 0 ? p[h][j] : acc[j] + p[h][j];
                }
                store_out(grp, acc);
            }
            if (tid == 0) a.counters[mt] = 0;
        }
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

extern "C" size_t scout_qpred_workspace_bytes(int hidden, int n_out, int batch, int ksplit) {
    if (hidden <= 0 || n_out <= 0 || batch <= 0 || ksplit <= 0) return 0;
    const size_t n_pad = (static_cast<size_t>(batch) + 15) / 16 * 16;
    const size_t xb = static_cast<size_t>(hidden) * n_pad * 2;
    const size_t part = static_cast<size_t>(ksplit) * n_out * n_pad * 4;
    const size_t ctr = (static_cast<size_t>(n_out) / QP_M) * 4;
    return ((xb + 255) / 256 + (part + 255) / 256 + (ctr + 255) / 256) * 256;
}

extern "C" int scout_qpred_pack_weights(const void* w, int hidden, int n_out, void* w_packed, void* stream) {
    using namespace scout_host;
    if (!w || !w_packed || hidden <= 0 || n_out <= 0 || hidden % QP_KC || n_out % QP_M) {
        set_error(SCOUT_ERR_INVALID_ARGUMENT, "scout_qpred_pack_weights: hidden %% 64 and n_out %% 128 must be 0");
        return SCOUT_ERR_INVALID_ARGUMENT;
    }
    qpred_pack_w_kernel<<<1184, 256, 0, static_cast<cudaStream_t>(stream)>>>(
        static_cast<const __nv_bfloat16*>(w), hidden, n_out, static_cast<__nv_bfloat16*>(w_packed));
    return check_launch("scout_qpred_pack_weights");
}

extern "C" int scout_predict_query(const float* x, int batch, int hidden, const void* w_packed, int n_out,
                                   float* out_f32, void* out_bf16, void* workspace, size_t workspace_bytes,
                                   int ksplit, void* stream) {
    using namespace scout_host;
    if (!x || !w_packed || !workspace || batch <= 0 || batch > QP_MAXN || hidden <= 0 || hidden % QP_KC ||
        n_out <= 0 || n_out % QP_M || (!out_f32 && !out_bf16)) {
        set_error(SCOUT_ERR_INVALID_ARGUMENT,
                  "predict_next_query: bad arguments (batch 1..256, hidden %% 64, n_out %% 128, an output)");
        return SCOUT_ERR_INVALID_ARGUMENT;
    }
    const int nkc = hidden / QP_KC;
    if (ksplit <= 0) ksplit = 2;
    if (ksplit > nkc) ksplit = nkc;
    if (workspace_bytes < scout_qpred_workspace_bytes(hidden, n_out, batch, ksplit)) {
        set_error(SCOUT_ERR_INVALID_ARGUMENT, "predict_next_query: workspace too small");
        return SCOUT_ERR_INVALID_ARGUMENT;
    }
    const int n_pad = (batch + 15) / 16 * 16;
    auto st = static_cast<cudaStream_t>(stream);
    uint8_t* ws = static_cast<uint8_t*>(workspace);
    const size_t xb_bytes = (static_cast<size_t>(hidden) * n_pad * 2 + 255) / 256 * 256;
    const size_t part_bytes = (static_cast<size_t>(ksplit) * n_out * n_pad * 4 + 255) / 256 * 256;
    auto* xb = reinterpret_cast<__nv_bfloat16*>(ws);
    auto* part = reinterpret_cast<float*>(ws + xb_bytes);
    auto* ctr = reinterpret_cast<int*>(ws + xb_bytes + part_bytes);
    qpred_pack_x_kernel<<<n_pad, 256, 0, st>>>(x, hidden, batch, n_pad, xb);
    QpArgs a{static_cast<const __nv_bfloat16*>(w_packed), xb, out_f32, static_cast<__nv_bfloat16*>(out_bf16), part, ctr,
             hidden, n_out, batch, n_pad, ksplit, 0};
    const uint32_t stage = QP_A_BYTES + static_cast<uint32_t>(n_pad) * QP_KC * 2;
    // ring depth: the CTAs of a launch share the SMs' shared memory (ksplit
    // 9 at 64 m-tiles = 4 CTAs per SM); SCOUT_QP_NST overrides (tuning)
    const int per_sm = (n_out / QP_M * ksplit + num_sms_k6() - 1) / num_sms_k6();
    int nst = static_cast<int>((220u * 1024u / static_cast<unsigned>(per_sm < 1 ? 1 : per_sm) - 2048u) / stage);
    if (const char* e = getenv("SCOUT_QP_NST")) nst = atoi(e);
    if (nst > 8) nst = 8;
    if (nst < 2) nst = 2;
    a.nst = nst;
    const size_t smem = static_cast<size_t>(nst) * stage;
    ensure_smem(reinterpret_cast<const void*>(qpred_gemm_kernel), smem);
    launch(qpred_gemm_kernel, dim3(n_out / QP_M, ksplit), dim3(QP_THREADS), smem, st, true, a);
    return check_launch("scout_predict_query");
}
