// CPU co-attention worker: the host half of ScoutAttention.
//
// Two kernels: on CPUs with AMX-BF16 (Sapphire Rapids and later), bf16 block
// images go through the tile unit (run_unit_amx: S = K.Q^T and O += P.V as
// TDPBF16PS tile products, the query split into bf16 hi + lo so scores keep
// ~16 mantissa bits, P rounded to bf16 as K2 does on the GPU); otherwise, and
// for f32 images, an AVX-512 fp32 kernel (run_unit). SCOUT_CPU_AMX=0 forces the
// latter. A persistent thread pool runs the units.
//
// Replaces the reference's scalar-double PrecomputeWorker path
// (proj/include/scout/engine.hpp:88-150, which calls partial_attention,
// attention.hpp:73-95, on the CPU-side blocks of layer i+1 with the predicted
// query) by a multi-threaded AVX-512 kernel over the host tier's block images
// (the pool's bf16 swizzled tile layout, or f32 row-major). One unit's G query
// heads share a pass over its blocks (GQA), as on the GPU: per block, the
// rows are decoded once, S = K (64 x 128) . Q^T (128 x G) in fp32, a
// block-wise online softmax per head, and O += P^T V. The result is K2's
// CPU-partial input: o normalised plus (max logit, denominator), empty
// partials (0, -inf, 0) (attention.hpp:24-36).
#include <immintrin.h>

#include <sys/syscall.h>
#include <unistd.h>

#include <algorithm>
#include <atomic>
#include <chrono>
#include <cmath>
#include <condition_variable>
#include <cstdint>
#include <cstdlib>
#include <cstring>
#include <functional>
#include <limits>
#include <memory>
#include <mutex>
#include <thread>
#include <vector>

#include "../../include/scout_b200.h"
#include "cpu_coattn.h"

namespace scout_host {
void set_error(int code, const char* fmt, ...);
}

namespace {

constexpr int D = SCOUT_HEAD_DIM;
constexpr int BS = SCOUT_BLOCK_SIZE;
constexpr int GMAX = 8;

// element (r, d) of a bf16 tile: [half][slab][row][16-byte chunk ^ (row & 7)][8]
inline int bf16_off(int r, int d) {
    const int h = r >> 5, rr = r & 31, j = d >> 6, c = (d >> 3) & 7, e = d & 7;
    return (((h * 2 + j) * 32 + rr) << 6) + ((c ^ (rr & 7)) << 3) + e;
}

// one row of a block tile into 128 floats
inline void load_row_scalar(const uint8_t* tile, int kv_dtype, int r, float* out) {
    if (kv_dtype == SCOUT_F32) {
        std::memcpy(out, reinterpret_cast<const float*>(tile) + static_cast<size_t>(r) * D, D * sizeof(float));
        return;
    }
    const uint16_t* t = reinterpret_cast<const uint16_t*>(tile);
    for (int d = 0; d < D; ++d) {
        const uint32_t u = static_cast<uint32_t>(t[bf16_off(r, d)]) << 16;
        std::memcpy(&out[d], &u, 4);
    }
}

__attribute__((target("avx512f"))) inline void load_row_avx512(const uint8_t* tile, int kv_dtype, int r, float* out) {
    if (kv_dtype == SCOUT_F32) {
        std::memcpy(out, reinterpret_cast<const float*>(tile) + static_cast<size_t>(r) * D, D * sizeof(float));
        return;
    }
    const uint16_t* t = reinterpret_cast<const uint16_t*>(tile);
    const int h = r >> 5, rr = r & 31;
    for (int j = 0; j < 2; ++j) {
        const uint16_t* row = t + ((h * 2 + j) * 32 + rr) * 64;
        for (int c = 0; c < 8; c += 2) {  // two 16-byte chunks -> 16 floats
            const __m128i a = _mm_loadu_si128(reinterpret_cast<const __m128i*>(row + ((c ^ (rr & 7)) << 3)));
            const __m128i b = _mm_loadu_si128(reinterpret_cast<const __m128i*>(row + (((c + 1) ^ (rr & 7)) << 3)));
            const __m256i ab = _mm256_inserti128_si256(_mm256_castsi128_si256(a), b, 1);
            const __m512i w = _mm512_slli_epi32(_mm512_cvtepu16_epi32(ab), 16);
            _mm512_storeu_ps(out + j * 64 + c * 8, _mm512_castsi512_ps(w));
        }
    }
}

__attribute__((target("avx512f"))) inline float dot128_avx512(const float* a, const float* b) {
    __m512 acc = _mm512_setzero_ps();
    for (int i = 0; i < D; i += 16) acc = _mm512_fmadd_ps(_mm512_loadu_ps(a + i), _mm512_loadu_ps(b + i), acc);
    return _mm512_reduce_add_ps(acc);
}
__attribute__((target("avx512f"))) inline void axpy128_avx512(float* y, float s, const float* x, float alpha) {
    // y = y * alpha + s * x
    const __m512 va = _mm512_set1_ps(alpha), vs = _mm512_set1_ps(s);
    for (int i = 0; i < D; i += 16)
        _mm512_storeu_ps(y + i, _mm512_fmadd_ps(vs, _mm512_loadu_ps(x + i), _mm512_mul_ps(va, _mm512_loadu_ps(y + i))));
}

inline float dot128_scalar(const float* a, const float* b) {
    float s = 0.f;
    for (int i = 0; i < D; ++i) s += a[i] * b[i];
    return s;
}
inline void axpy128_scalar(float* y, float s, const float* x, float alpha) {
    for (int i = 0; i < D; ++i) y[i] = y[i] * alpha + s * x[i];
}

struct Job {
    const uint8_t* host;
    int kv_dtype;
    size_t slot_bytes;
    const int64_t* index;
    const int32_t* rows;
    const int32_t* n_blocks;
    int k_stride, G;
    float scale;
    const void* q;   // f32, or bf16 when q_bf16
    void* o;         // f32, or bf16 when o_bf16
    float* ml;
    bool q_bf16, o_bf16;
};

inline float bf16_to_f(uint16_t h) {
    const uint32_t u = static_cast<uint32_t>(h) << 16;
    float f;
    std::memcpy(&f, &u, 4);
    return f;
}
inline uint16_t f_to_bf16(float f) {  // round to nearest even (finite values)
    uint32_t u;
    std::memcpy(&u, &f, 4);
    if ((u & 0x7F800000u) == 0x7F800000u) return static_cast<uint16_t>(u >> 16);  // inf / nan
    return static_cast<uint16_t>((u + 0x7FFFu + ((u >> 16) & 1u)) >> 16);
}
// unit u's G query rows as f32 (bf16 queries widened exactly into scratch)
inline const float* unit_query(const Job& j, int u, float* scratch) {
    const size_t off = static_cast<size_t>(u) * j.G * D;
    if (!j.q_bf16) return static_cast<const float*>(j.q) + off;
    const uint16_t* qb = static_cast<const uint16_t*>(j.q) + off;
    for (int i = 0; i < j.G * D; ++i) scratch[i] = bf16_to_f(qb[i]);
    return scratch;
}
// head h's normalised output row (K2's CPU-partial o) in the job's o dtype
inline void store_o(const Job& j, size_t h, const float* acc, float inv) {
    if (j.o_bf16) {
        uint16_t* o = static_cast<uint16_t*>(j.o) + h * D;
        for (int d = 0; d < D; ++d) o[d] = f_to_bf16(acc[d] * inv);
    } else {
        float* o = static_cast<float*>(j.o) + h * D;
        for (int d = 0; d < D; ++d) o[d] = acc[d] * inv;
    }
}

// a unit with no CPU-side block: the empty partial (o = 0, (-inf, 0))
inline void store_empty(const Job& j, int u) {
    const size_t h0 = static_cast<size_t>(u) * j.G;
    const size_t esz = j.o_bf16 ? 2 : 4;
    std::memset(static_cast<uint8_t*>(j.o) + h0 * D * esz, 0, j.G * D * esz);
    for (int g = 0; g < j.G; ++g) {
        j.ml[(h0 + g) * 2] = -std::numeric_limits<float>::infinity();
        j.ml[(h0 + g) * 2 + 1] = 0.f;
    }
}
// Per block: the block's rows are decoded once (K and V into fp32), then for
// each head: 64 scores, one block maximum, 64 exponentials and the weighted V
// sum; the running state is rescaled once per block (same result as the
// per-row online softmax of accumulate_token, attention.hpp:38-50, up to fp32
// rounding).
template <bool AVX>
void run_unit(const Job& j, int u) {
    const int G = j.G;
    float m[GMAX], l[GMAX];
    alignas(64) float acc[GMAX][D];
    alignas(64) float kb[BS][D], vb[BS][D];
    float sc[BS];
    for (int g = 0; g < G; ++g) {
        m[g] = -std::numeric_limits<float>::infinity();
        l[g] = 0.f;
        std::memset(acc[g], 0, sizeof(acc[g]));
    }
    const int nb = j.n_blocks[u];
    if (nb <= 0) {
        store_empty(j, u);
        return;
    }
    alignas(64) float qscratch[GMAX * D];
    const float* qu = unit_query(j, u, qscratch);
    for (int i = 0; i < nb; ++i) {
        const size_t idx = static_cast<size_t>(u) * j.k_stride + i;
        const uint8_t* kt = j.host + static_cast<size_t>(j.index[idx]) * j.slot_bytes;
        const uint8_t* vt = kt + j.slot_bytes / 2;
        const int rows = j.rows ? j.rows[idx] : BS;
        for (int r = 0; r < rows; ++r) {
            if (AVX) {
                load_row_avx512(kt, j.kv_dtype, r, kb[r]);
                load_row_avx512(vt, j.kv_dtype, r, vb[r]);
            } else {
                load_row_scalar(kt, j.kv_dtype, r, kb[r]);
                load_row_scalar(vt, j.kv_dtype, r, vb[r]);
            }
        }
        for (int g = 0; g < G; ++g) {
            const float* qg = qu + g * D;
            float mx = -std::numeric_limits<float>::infinity();
            for (int r = 0; r < rows; ++r) {
                sc[r] = (AVX ? dot128_avx512(kb[r], qg) : dot128_scalar(kb[r], qg)) * j.scale;
                mx = std::max(mx, sc[r]);
            }
            const float mn = std::max(m[g], mx);
            const float alpha = std::exp(m[g] - mn);
            float lsum = 0.f;
            for (int r = 0; r < rows; ++r) {
                sc[r] = std::exp(sc[r] - mn);
                lsum += sc[r];
            }
            l[g] = l[g] * alpha + lsum;
            m[g] = mn;
            if (AVX) {
                axpy128_avx512(acc[g], 0.f, vb[0], alpha);  // acc *= alpha
                for (int r = 0; r < rows; ++r) axpy128_avx512(acc[g], sc[r], vb[r], 1.f);
            } else {
                axpy128_scalar(acc[g], 0.f, vb[0], alpha);
                for (int r = 0; r < rows; ++r) axpy128_scalar(acc[g], sc[r], vb[r], 1.f);
            }
        }
    }
    for (int g = 0; g < G; ++g) {
        const size_t h = static_cast<size_t>(u) * G + g;
        const float inv = l[g] > 0.f ? 1.f / l[g] : 0.f;
        store_o(j, h, acc[g], inv);
        j.ml[h * 2] = l[g] > 0.f ? m[g] : -std::numeric_limits<float>::infinity();
        j.ml[h * 2 + 1] = l[g];
    }
}

// ---------------------------------------------------------------- AMX path --
struct alignas(64) TileCfg {
    uint8_t palette, start_row;
    uint8_t rsv[14];
    uint16_t colsb[16];
    uint8_t rows[16];
};

// per-thread scratch of the AMX kernel: one chunk of up to CH blocks (~320 KB, L2)
constexpr int CH = 8;
struct alignas(64) AmxScratch {
    uint16_t kb[CH][BS][D];         // K rows, unswizzled (A operand of S = K.Q^T)
    uint16_t vv[CH][BS / 2][D][2];  // V in VNNI pairs (B operand of O += P.V)
    float sb[CH][BS][16];           // S: cols 0-7 hi heads, 8-15 lo heads
    float pf[BS][GMAX];             // one block's P (bf16-exact fp32), token-major
    uint16_t pa[CH][2][16][32];     // P head-major per 32-token half (A operand; rows >= G zero)
    float ob[16][D];                // the chunk's P.V (rows >= G zero)
    float o[GMAX][D];             // running O
    uint16_t bq[4][16][32];       // Q^T in VNNI, per 32-channel step (hi | lo columns)
};

// qword permutations: a 128-byte slab row whose 16-byte chunk c sits at
// position c ^ x -> channel order (x = row & 7), as (first 64 B, second 64 B)
struct UnswizzleIdx {
    alignas(64) int64_t lo[8][8], hi[8][8];
    UnswizzleIdx() {
        for (int x = 0; x < 8; ++x)
            for (int q = 0; q < 8; ++q) {
                lo[x][q] = ((((q >> 1) ^ x) << 1) | (q & 1));
                hi[x][q] = (((((q + 8) >> 1) ^ x) << 1) | (q & 1));
            }
    }
};
const UnswizzleIdx kUnsw;

inline uint16_t bf16_rne(float f) {
    uint32_t u;
    std::memcpy(&u, &f, 4);
    if ((u & 0x7f800000u) == 0x7f800000u) return static_cast<uint16_t>(u >> 16);  // inf / nan
    return static_cast<uint16_t>((u + 0x7fffu + ((u >> 16) & 1u)) >> 16);
}
inline float bf16_f(uint16_t h) {
    const uint32_t u = static_cast<uint32_t>(h) << 16;
    float f;
    std::memcpy(&f, &u, 4);
    return f;
}

#ifdef SCOUT_CPU_PROF
#include <x86intrin.h>
thread_local unsigned long long g_prof[8];
#define PROF_MARK(i) do { _mm_mfence(); const unsigned long long t_ = __rdtsc(); g_prof[i] += t_ - t_prev; t_prev = t_; } while (0)
#define PROF_START unsigned long long t_prev = __rdtsc()
#else
#define PROF_MARK(i) do {} while (0)
#define PROF_START do {} while (0)
#endif

#define SCOUT_AMX_TARGET __attribute__((target("amx-tile,amx-bf16,avx512f,avx512bw,avx512bf16")))

// row r of a swizzled bf16 tile -> four zmm of 32 channels each
SCOUT_AMX_TARGET inline void unswizzle_row(const uint16_t* t, int r, __m512i out[4]) {
    const int h = r >> 5, rr = r & 31, x = rr & 7;
    const __m512i il = _mm512_load_si512(kUnsw.lo[x]), ih = _mm512_load_si512(kUnsw.hi[x]);
    for (int j = 0; j < 2; ++j) {
        const uint16_t* row = t + ((h * 2 + j) * 32 + rr) * 64;
        const __m512i a = _mm512_loadu_si512(row), b = _mm512_loadu_si512(row + 32);
        out[2 * j] = _mm512_permutex2var_epi64(a, il, b);
        out[2 * j + 1] = _mm512_permutex2var_epi64(a, ih, b);
    }
}

// tokens t, t + 1 of a score tile (hi + lo columns) as one vector: lanes 0-7
// token t, 8-15 token t + 1; rows past the fill -> -inf
SCOUT_AMX_TARGET inline __m512 score_pair(const float* s0, const float* s1, int t, int rows, __m512i pick_hi,
                                          __m512i pick_lo, __m512 ninf) {
    const __m512 a = _mm512_load_ps(s0), c = _mm512_load_ps(s1);
    const __m512 v = _mm512_add_ps(_mm512_permutex2var_ps(a, pick_hi, c), _mm512_permutex2var_ps(a, pick_lo, c));
    const __mmask16 ok = static_cast<__mmask16>((t < rows ? 0x00ffu : 0u) | (t + 1 < rows ? 0xff00u : 0u));
    return _mm512_mask_blend_ps(ok, ninf, v);
}

// unit u's G query rows as f32: bf16 queries widened exactly, 16 lanes at a time
SCOUT_AMX_TARGET inline const float* unit_query_v(const Job& j, int u, float* scratch) {
    const size_t off = static_cast<size_t>(u) * j.G * D;
    if (!j.q_bf16) return static_cast<const float*>(j.q) + off;
    const uint16_t* qb = static_cast<const uint16_t*>(j.q) + off;
    for (int i = 0; i < j.G * D; i += 16)
        _mm512_store_ps(scratch + i, _mm512_castsi512_ps(_mm512_slli_epi32(
                                         _mm512_cvtepu16_epi32(_mm256_loadu_si256(reinterpret_cast<const __m256i*>(qb + i))), 16)));
    return scratch;
}
// store_o, 16 lanes at a time; the bf16 rounding is f_to_bf16's (nearest even,
// inf / nan truncated), bit for bit
SCOUT_AMX_TARGET inline void store_o_v(const Job& j, size_t h, const float* acc, float inv) {
    const __m512 vi = _mm512_set1_ps(inv);
    if (j.o_bf16) {
        uint16_t* o = static_cast<uint16_t*>(j.o) + h * D;
        const __m512i one = _mm512_set1_epi32(1), bias = _mm512_set1_epi32(0x7FFF), ex = _mm512_set1_epi32(0x7F800000);
        for (int d = 0; d < D; d += 16) {
            const __m512i u = _mm512_castps_si512(_mm512_mul_ps(_mm512_load_ps(acc + d), vi));
            const __m512i r = _mm512_add_epi32(_mm512_add_epi32(u, bias), _mm512_and_si512(_mm512_srli_epi32(u, 16), one));
            const __mmask16 special = _mm512_cmpeq_epi32_mask(_mm512_and_si512(u, ex), ex);
            const __m512i v = _mm512_mask_mov_epi32(r, special, u);
            _mm256_storeu_si256(reinterpret_cast<__m256i*>(o + d), _mm512_cvtepi32_epi16(_mm512_srli_epi32(v, 16)));
        }
    } else {
        float* o = static_cast<float*>(j.o) + h * D;
        for (int d = 0; d < D; d += 16) _mm512_storeu_ps(o + d, _mm512_mul_ps(_mm512_load_ps(acc + d), vi));
    }
}
// 16 x 16 transpose of 32-bit words: r[n] word i -> r[i] word n
SCOUT_AMX_TARGET inline void transpose16(__m512i r[16]) {
    __m512i t[16], v[16];
    for (int k = 0; k < 8; ++k) {
        t[2 * k] = _mm512_unpacklo_epi32(r[2 * k], r[2 * k + 1]);
        t[2 * k + 1] = _mm512_unpackhi_epi32(r[2 * k], r[2 * k + 1]);
    }
    for (int k = 0; k < 4; ++k) {
        v[4 * k] = _mm512_unpacklo_epi64(t[4 * k], t[4 * k + 2]);
        v[4 * k + 1] = _mm512_unpackhi_epi64(t[4 * k], t[4 * k + 2]);
        v[4 * k + 2] = _mm512_unpacklo_epi64(t[4 * k + 1], t[4 * k + 3]);
        v[4 * k + 3] = _mm512_unpackhi_epi64(t[4 * k + 1], t[4 * k + 3]);
    }
    // v[4k + c] 128-bit lane L holds word 4L + c of rows 4k..4k+3
    for (int c = 0; c < 4; ++c) {
        const __m512i a0 = _mm512_shuffle_i32x4(v[c], v[4 + c], 0x44), a1 = _mm512_shuffle_i32x4(v[c], v[4 + c], 0xEE);
        const __m512i b0 = _mm512_shuffle_i32x4(v[8 + c], v[12 + c], 0x44),
                      b1 = _mm512_shuffle_i32x4(v[8 + c], v[12 + c], 0xEE);
        r[c] = _mm512_shuffle_i32x4(a0, b0, 0x88);
        r[4 + c] = _mm512_shuffle_i32x4(a0, b0, 0xDD);
        r[8 + c] = _mm512_shuffle_i32x4(a1, b1, 0x88);
        r[12 + c] = _mm512_shuffle_i32x4(a1, b1, 0xDD);
    }
}

SCOUT_AMX_TARGET inline __m512 exp2_ps(__m512 x) {
    x = _mm512_max_ps(x, _mm512_set1_ps(-200.f));  // -inf -> 0 after scalef
    const __m512 xi = _mm512_roundscale_ps(x, _MM_FROUND_TO_NEAREST_INT | _MM_FROUND_NO_EXC);
    const __m512 f = _mm512_sub_ps(x, xi);  // [-0.5, 0.5]
    __m512 p = _mm512_set1_ps(1.5403530e-4f);
    p = _mm512_fmadd_ps(p, f, _mm512_set1_ps(1.3333558e-3f));
    p = _mm512_fmadd_ps(p, f, _mm512_set1_ps(9.6181291e-3f));
    p = _mm512_fmadd_ps(p, f, _mm512_set1_ps(5.5504109e-2f));
    p = _mm512_fmadd_ps(p, f, _mm512_set1_ps(2.4022651e-1f));
    p = _mm512_fmadd_ps(p, f, _mm512_set1_ps(6.9314718e-1f));
    p = _mm512_fmadd_ps(p, f, _mm512_set1_ps(1.f));
    return _mm512_scalef_ps(p, xi);
}

SCOUT_AMX_TARGET void amx_config(int G) {
    TileCfg c{};
    c.palette = 1;
    (void)G;
    for (int t = 0; t < 8; ++t) { c.rows[t] = 16; c.colsb[t] = 64; }
    _tile_loadconfig(&c);
}

// One unit on the tile unit. Scores are in log2 units (the query is scaled by
// scale * log2(e) before the hi/lo split); the result is K2's CPU-partial
// format. The blocks go in chunks of up to CH: all of a chunk's operands are
// staged first (AVX-512), then one tile burst computes every block's S, the
// softmax runs over the whole chunk (one rescale per chunk), and a second
// burst accumulates the chunk's P.V in the tile registers. The tile unit pays
// a wake-up of several hundred cycles after each stretch of vector work, so
// two bursts per chunk instead of two per block matter (measured: an S burst
// of 16 tile products costs ~220 TSC back to back, ~900 after 1200 cycles of
// other work).
#ifndef SCOUT_CPU_PREFETCH
#define SCOUT_CPU_PREFETCH 1
#endif
#ifndef SCOUT_CPU_PF_HINT
#define SCOUT_CPU_PF_HINT _MM_HINT_T1  // into L2: the staging of the current image owns L1
#endif
// the image of block i of unit u (NULL past the unit's blocks)
inline const char* block_image(const Job& j, int u, int i) {
    if (u < 0 || i >= j.n_blocks[u]) return nullptr;
    return reinterpret_cast<const char*>(j.host + static_cast<size_t>(j.index[static_cast<size_t>(u) * j.k_stride + i]) *
                                                      j.slot_bytes);
}

// One unit on the tile unit (`next_u`: the unit this thread runs next, whose
// first block image is prefetched while the last one here is staged; each
// block's image is prefetched while the one before it is staged: a single
// thread's demand misses alone reach ~12 GB/s of host DRAM, one 32 KiB image
// per ~2.6 us)
SCOUT_AMX_TARGET void run_unit_amx(const Job& j, int u, AmxScratch& w, int next_u) {
    const int G = j.G;
    constexpr float LOG2E = 1.4426950408889634f, LN2 = 0.6931471805599453f;
    // ---- Q^T -> VNNI B tiles: column n < 8 = hi of head n, 8 + n = lo of head n;
    // a VNNI word is the (2i, 2i+1) channel pair of one column
    // (w.bq's columns of heads >= G and w.pa's rows >= G stay zero: cleared
    // when the scratch is (re)dedicated to a group size, amx_work)
    const int nb = j.n_blocks[u];
    if (nb <= 0) {
        store_empty(j, u);
        return;
    }
    alignas(64) float qscratch[GMAX * D];
    const float* qu = unit_query_v(j, u, qscratch);
    const __m512 qs = _mm512_set1_ps(j.scale * LOG2E);
    for (int ks = 0; ks < 4; ++ks) {
        // columns: hi words of heads 0..7, then lo words (heads >= G zero);
        // one 16 x 16 word transpose makes the VNNI rows
        __m512i cols[16];
        for (int g = 0; g < GMAX; ++g) {
            if (g >= G) {
                cols[g] = cols[8 + g] = _mm512_setzero_si512();
                continue;
            }
            const __m512 v0 = _mm512_mul_ps(_mm512_loadu_ps(qu + g * D + 32 * ks), qs);
            const __m512 v1 = _mm512_mul_ps(_mm512_loadu_ps(qu + g * D + 32 * ks + 16), qs);
            const __m512i hi = (__m512i)_mm512_cvtne2ps_pbh(v1, v0);
            const __m512 h0 = _mm512_castsi512_ps(_mm512_slli_epi32(_mm512_cvtepu16_epi32(_mm512_castsi512_si256(hi)), 16));
            const __m512 h1 = _mm512_castsi512_ps(
                _mm512_slli_epi32(_mm512_cvtepu16_epi32(_mm512_extracti64x4_epi64(hi, 1)), 16));
            cols[g] = hi;
            cols[8 + g] = (__m512i)_mm512_cvtne2ps_pbh(_mm512_sub_ps(v1, h1), _mm512_sub_ps(v0, h0));
        }
        transpose16(cols);
        for (int i = 0; i < 16; ++i) _mm512_store_si512(w.bq[ks][i], cols[i]);
    }
    bool first = true;  // the first chunk's P.V is the running O (no memset, no rescale of garbage)
    const __m512 ninf = _mm512_set1_ps(-std::numeric_limits<float>::infinity());
    __m512 m = ninf, l = _mm512_setzero_ps();  // lanes g and 8 + g: head g
    const __m512i pick_hi = _mm512_setr_epi32(0, 1, 2, 3, 4, 5, 6, 7, 16, 17, 18, 19, 20, 21, 22, 23);
    const __m512i pick_lo = _mm512_setr_epi32(8, 9, 10, 11, 12, 13, 14, 15, 24, 25, 26, 27, 28, 29, 30, 31);
    const __m512i vp0 = _mm512_setr_epi64(0, 1, 8, 9, 2, 3, 10, 11);
    const __m512i vp1 = _mm512_setr_epi64(4, 5, 12, 13, 6, 7, 14, 15);
    const __m512i gidx = _mm512_mullo_epi32(_mm512_setr_epi32(0, 1, 2, 3, 4, 5, 6, 7, 8, 9, 10, 11, 12, 13, 14, 15),
                                            _mm512_set1_epi32(GMAX));
    for (int c0 = 0; c0 < nb; c0 += CH) {
        const int nc = std::min(CH, nb - c0);
        int rows[CH];
        PROF_START;
        // ---- stage: K rows -> kb, V row pairs -> vv (rows past the fill are
        // zero: stale bytes may be NaN)
        for (int b = 0; b < nc; ++b) {
            const size_t idx = static_cast<size_t>(u) * j.k_stride + c0 + b;
            const uint16_t* kt =
                reinterpret_cast<const uint16_t*>(j.host + static_cast<size_t>(j.index[idx]) * j.slot_bytes);
            const uint16_t* vt = kt + j.slot_bytes / 4;
            rows[b] = std::max(0, std::min(BS, j.rows ? static_cast<int>(j.rows[idx]) : BS));
            // mode 1: the block after this one (the next unit's first after the
            // last); mode 2: block c0 + b of the next unit (a unit's compute ahead)
            const char* pf = SCOUT_CPU_PREFETCH == 0 ? nullptr
                             : SCOUT_CPU_PREFETCH == 2
                                 ? block_image(j, next_u, c0 + b)
                                 : (c0 + b + 1 < nb ? block_image(j, u, c0 + b + 1) : block_image(j, next_u, 0));
            const int pf_lines = static_cast<int>(j.slot_bytes / 64);  // 512: 8 per K row
            for (int r = 0; r < BS; ++r) {
                if (pf)
                    for (int x = 0; x < pf_lines / BS; ++x) _mm_prefetch(pf + 64 * (r * (pf_lines / BS) + x), SCOUT_CPU_PF_HINT);
                __m512i z[4];
                if (r < rows[b]) unswizzle_row(kt, r, z);
                else z[0] = z[1] = z[2] = z[3] = _mm512_setzero_si512();
                for (int q = 0; q < 4; ++q) _mm512_store_si512(&w.kb[b][r][32 * q], z[q]);
            }
            for (int p = 0; p < BS / 2; ++p) {
                __m512i a[4], c[4];
                if (2 * p < rows[b]) unswizzle_row(vt, 2 * p, a);
                else a[0] = a[1] = a[2] = a[3] = _mm512_setzero_si512();
                if (2 * p + 1 < rows[b]) unswizzle_row(vt, 2 * p + 1, c);
                else c[0] = c[1] = c[2] = c[3] = _mm512_setzero_si512();
                for (int q = 0; q < 4; ++q) {
                    const __m512i lo = _mm512_unpacklo_epi16(a[q], c[q]), hi = _mm512_unpackhi_epi16(a[q], c[q]);
                    _mm512_store_si512(&w.vv[b][p][32 * q][0], _mm512_permutex2var_epi64(lo, vp0, hi));
                    _mm512_store_si512(&w.vv[b][p][32 * q + 16][0], _mm512_permutex2var_epi64(lo, vp1, hi));
                }
            }
        }
        PROF_MARK(0);
        // ---- burst 1: S = K . Q^T per block, four 16-token accumulators
        // (tmm0-3), Q^T two 32-channel steps at a time in tmm6/7, K via tmm4/5
#define SCOUT_S_STEP(mt, ks, A, QB)                                 \
    _tile_loadd(A, &w.kb[b][16 * (mt)][32 * (ks)], 2 * D);          \
    _tile_dpbf16ps(mt, A, QB)
        for (int b = 0; b < nc; ++b) {
            _tile_zero(0);
            _tile_zero(1);
            _tile_zero(2);
            _tile_zero(3);
            for (int kp = 0; kp < 2; ++kp) {
                _tile_loadd(6, w.bq[2 * kp], 64);
                _tile_loadd(7, w.bq[2 * kp + 1], 64);
                SCOUT_S_STEP(0, 2 * kp, 4, 6);
                SCOUT_S_STEP(1, 2 * kp, 5, 6);
                SCOUT_S_STEP(2, 2 * kp, 4, 6);
                SCOUT_S_STEP(3, 2 * kp, 5, 6);
                SCOUT_S_STEP(0, 2 * kp + 1, 4, 7);
                SCOUT_S_STEP(1, 2 * kp + 1, 5, 7);
                SCOUT_S_STEP(2, 2 * kp + 1, 4, 7);
                SCOUT_S_STEP(3, 2 * kp + 1, 5, 7);
            }
            _tile_stored(0, &w.sb[b][0][0], 64);
            _tile_stored(1, &w.sb[b][16][0], 64);
            _tile_stored(2, &w.sb[b][32][0], 64);
            _tile_stored(3, &w.sb[b][48][0], 64);
        }
#undef SCOUT_S_STEP
        PROF_MARK(1);
        // ---- softmax over the chunk, two tokens per vector (lanes 0-7: token
        // t, 8-15: t + 1): pass 1 the maximum, pass 2 the bf16-rounded weights
#define score(b, p) score_pair(w.sb[b][2 * (p)], w.sb[b][2 * (p) + 1], 2 * (p), rows[b], pick_hi, pick_lo, ninf)
        __m512 mx = ninf;
        for (int b = 0; b < nc; ++b)
            for (int p = 0; p < BS / 2; ++p) mx = _mm512_max_ps(mx, score(b, p));
        mx = _mm512_max_ps(mx, _mm512_shuffle_f32x4(mx, mx, 0x4e));
        const __m512 mn = _mm512_max_ps(m, mx);
        const __m512 alpha = exp2_ps(_mm512_sub_ps(m, mn));
        m = mn;
        __m512 ls = _mm512_setzero_ps();
        for (int b = 0; b < nc; ++b) {
            for (int p = 0; p < BS / 2; ++p) {
                const __m512 e = exp2_ps(_mm512_sub_ps(score(b, p), mn));
                // round to bf16 once: the sum uses the same weights the tile product sees
                const __m512 pr = _mm512_castsi512_ps(
                    _mm512_slli_epi32(_mm512_cvtepu16_epi32((__m256i)_mm512_cvtneps_pbh(e)), 16));
                ls = _mm512_add_ps(ls, pr);
                _mm512_store_ps(&w.pf[2 * p][0], pr);
            }
            // P -> head-major bf16 (A operand), one row per head
            for (int g = 0; g < G; ++g)
                for (int h = 0; h < 2; ++h) {
                    const __m512 p0 = _mm512_i32gather_ps(gidx, &w.pf[32 * h][g], 4);
                    const __m512 p1 = _mm512_i32gather_ps(gidx, &w.pf[32 * h + 16][g], 4);
                    _mm512_store_si512(w.pa[b][h][g], (__m512i)_mm512_cvtne2ps_pbh(p1, p0));
                }
        }
#undef score
        ls = _mm512_add_ps(ls, _mm512_shuffle_f32x4(ls, ls, 0x4e));
        l = _mm512_fmadd_ps(l, alpha, ls);
        PROF_MARK(2);
        // ---- burst 2: the chunk's P.V, four 16-channel accumulators (tmm0-3)
        // per pass over the blocks, P in tmm4/5 (token halves), V via tmm6/7
#define SCOUT_PV_STEP(c, kt, A, B)                                          \
    _tile_loadd(B, &w.vv[b][16 * (kt)][16 * (cg0 + (c))][0], D * 4);        \
    _tile_dpbf16ps(c, A, B)
        for (int cg0 = 0; cg0 < D / 16; cg0 += 4) {
            _tile_zero(0);
            _tile_zero(1);
            _tile_zero(2);
            _tile_zero(3);
            for (int b = 0; b < nc; ++b) {
                _tile_loadd(4, w.pa[b][0], 64);
                _tile_loadd(5, w.pa[b][1], 64);
                SCOUT_PV_STEP(0, 0, 4, 6);
                SCOUT_PV_STEP(1, 0, 4, 7);
                SCOUT_PV_STEP(2, 0, 4, 6);
                SCOUT_PV_STEP(3, 0, 4, 7);
                SCOUT_PV_STEP(0, 1, 5, 6);
                SCOUT_PV_STEP(1, 1, 5, 7);
                SCOUT_PV_STEP(2, 1, 5, 6);
                SCOUT_PV_STEP(3, 1, 5, 7);
            }
            _tile_stored(0, &w.ob[0][16 * cg0], D * 4);
            _tile_stored(1, &w.ob[0][16 * cg0 + 16], D * 4);
            _tile_stored(2, &w.ob[0][16 * cg0 + 32], D * 4);
            _tile_stored(3, &w.ob[0][16 * cg0 + 48], D * 4);
        }
#undef SCOUT_PV_STEP
        PROF_MARK(3);
        // ---- O = O * alpha + P.V
        alignas(64) float al[16];
        _mm512_store_ps(al, alpha);
        for (int g = 0; g < G; ++g) {
            const __m512 a = _mm512_set1_ps(al[g]);
            for (int c = 0; c < D; c += 16)
                _mm512_store_ps(&w.o[g][c], first ? _mm512_load_ps(&w.ob[g][c])
                                                  : _mm512_fmadd_ps(a, _mm512_load_ps(&w.o[g][c]),
                                                                    _mm512_load_ps(&w.ob[g][c])));
        }
        first = false;
        PROF_MARK(4);
    }
    alignas(64) float mm[16], ll[16];
    _mm512_store_ps(mm, m);
    _mm512_store_ps(ll, l);
    for (int g = 0; g < G; ++g) {
        const size_t h = static_cast<size_t>(u) * G + g;
        const float inv = ll[g] > 0.f ? 1.f / ll[g] : 0.f;
        store_o_v(j, h, w.o[g], inv);
        j.ml[h * 2] = ll[g] > 0.f ? mm[g] * LN2 : -std::numeric_limits<float>::infinity();
        j.ml[h * 2 + 1] = ll[g];
    }
}

SCOUT_AMX_TARGET void amx_work(const Job& j, std::atomic<int>& next, int n_units, int batch) {
    // per-thread scratch, freed when the thread exits (callers' own threads run units too)
    struct Free {
        void operator()(AmxScratch* p) const { std::free(p); }
    };
    static thread_local std::unique_ptr<AmxScratch, Free> owned;
    if (!owned) {
        owned.reset(static_cast<AmxScratch*>(std::aligned_alloc(64, sizeof(AmxScratch))));
        if (!owned) {  // no memory for the tile staging: this thread takes the AVX-512 kernel
            for (int u0; (u0 = next.fetch_add(batch)) < n_units;)
                for (int u = u0; u < std::min(u0 + batch, n_units); ++u) run_unit<true>(j, u);
            return;
        }
    }
    AmxScratch* scratch = owned.get();
    static thread_local int scratch_g = -1;  // the group size the zero padding was laid for
    if (scratch_g != j.G) {
        std::memset(scratch->bq, 0, sizeof(scratch->bq));
        std::memset(scratch->pa, 0, sizeof(scratch->pa));
        scratch_g = j.G;
    }
    amx_config(j.G);
    // units are claimed `batch` at a time (one contended atomic per batch),
    // one batch ahead, so the next unit's first image is in flight while the
    // last unit of a batch finishes
    int u0 = next.fetch_add(batch);
    while (u0 < n_units) {
        const int u1 = std::min(u0 + batch, n_units);
        const int n0 = next.fetch_add(batch);
        for (int u = u0; u < u1; ++u) run_unit_amx(j, u, *scratch, u + 1 < u1 ? u + 1 : (n0 < n_units ? n0 : -1));
        u0 = n0;
    }
    _tile_release();
}

// AMX-BF16 present and the kernel granted the tile state (arch_prctl)
bool amx_ready() {
    static const int v = [] {
        if (!__builtin_cpu_supports("avx512bf16")) return 0;
        unsigned a, b, c, d;
        __asm__ volatile("cpuid" : "=a"(a), "=b"(b), "=c"(c), "=d"(d) : "a"(7), "c"(0));
        if (!((d >> 22) & 1u) || !((d >> 24) & 1u)) return 0;  // AMX-BF16, AMX-TILE
        constexpr long ARCH_REQ_XCOMP_PERM = 0x1023, XFEATURE_XTILEDATA = 18;
        return syscall(SYS_arch_prctl, ARCH_REQ_XCOMP_PERM, XFEATURE_XTILEDATA) == 0 ? 1 : 0;
    }();
    return v != 0;
}

// ----------------------------------------------------------- thread pool --
// Persistent workers (a decode step calls the worker once per layer: thread
// creation per call would cost more than a layer's CPU share).
#ifndef SCOUT_POOL_SPIN_US
#define SCOUT_POOL_SPIN_US 0  // idle workers' spin before sleeping (0: sleep at once)
#endif
class Pool {
public:
    void run(int T, const std::function<void()>& fn) {
        std::lock_guard<std::mutex> call(call_mu_);
        {
            std::unique_lock<std::mutex> lk(mu_);
            while (static_cast<int>(workers_.size()) < T - 1) {
                const int id = static_cast<int>(workers_.size());
                workers_.emplace_back([this, id] { loop(id); });
            }
            fn_ = &fn;
            want_ = T - 1;
            pending_ = T - 1;
            pending_a_.store(T - 1, std::memory_order_relaxed);
            ++gen_;
            gen_a_.store(gen_, std::memory_order_release);
        }
        cv_.notify_all();
        fn();
        // the workers finish within a unit or two of this thread: spin first
        spin_until([&] { return pending_a_.load(std::memory_order_acquire) == 0; });
        std::unique_lock<std::mutex> lk(mu_);
        done_.wait(lk, [&] { return pending_ == 0; });
        fn_ = nullptr;
    }
    ~Pool() {
        {
            std::lock_guard<std::mutex> lk(mu_);
            stop_ = true;
        }
        cv_.notify_all();
        for (auto& t : workers_) t.join();
    }

private:
    void loop(int id) {
        uint64_t seen = 0;
        for (;;) {
            const std::function<void()>* fn;
            // a decode step calls the pool once per layer chunk, back to back:
            // idle workers spin a short while before sleeping on the condvar
            spin_until([&] { return gen_a_.load(std::memory_order_acquire) != seen; });
            {
                std::unique_lock<std::mutex> lk(mu_);
                cv_.wait(lk, [&] { return stop_ || (gen_ != seen && id < want_); });
                if (stop_) return;
                seen = gen_;
                fn = fn_;
            }
            (*fn)();
            std::lock_guard<std::mutex> lk(mu_);
            pending_a_.fetch_sub(1, std::memory_order_release);
            if (--pending_ == 0) done_.notify_one();
        }
    }
    template <typename F>
    static void spin_until(F done) {
        if (SCOUT_POOL_SPIN_US <= 0) return;
        const auto t0 = std::chrono::steady_clock::now();
        for (int i = 0; !done(); ++i) {
            _mm_pause();
            if ((i & 255) == 255 &&
                std::chrono::steady_clock::now() - t0 > std::chrono::microseconds(SCOUT_POOL_SPIN_US))
                return;
        }
    }
    std::atomic<uint64_t> gen_a_{0};
    std::atomic<int> pending_a_{0};
    std::mutex call_mu_, mu_;
    std::condition_variable cv_, done_;
    std::vector<std::thread> workers_;
    const std::function<void()>* fn_ = nullptr;
    uint64_t gen_ = 0;
    int want_ = 0, pending_ = 0;
    bool stop_ = false;
};

Pool& pool() {
    static Pool p;
    return p;
}

bool has_avx512() {
    static const int v = __builtin_cpu_supports("avx512f") ? 1 : 0;
    return v != 0;
}

}  // namespace

int scout_cpu_coattn_run(const CpuCoattnArgs& a) {
    using scout_host::set_error;
    if (a.n_units < 0 || a.k_stride <= 0 || a.group < 1 || a.group > GMAX || !(a.scale > 0.f) ||
        (a.kv_dtype != SCOUT_BF16 && a.kv_dtype != SCOUT_F32) || (a.q_dtype != SCOUT_F32 && a.q_dtype != SCOUT_BF16) ||
        (a.o_dtype != SCOUT_F32 && a.o_dtype != SCOUT_BF16) ||
        (a.n_units > 0 && (!a.host_tier || !a.host_index || !a.n_blocks || !a.q || !a.o || !a.ml))) {
        set_error(SCOUT_ERR_INVALID_ARGUMENT, "scout_cpu_partial_attention: bad arguments");
        return SCOUT_ERR_INVALID_ARGUMENT;
    }
    if (a.n_units == 0) return SCOUT_OK;
    const Job j{static_cast<const uint8_t*>(a.host_tier), a.kv_dtype, scout_slot_bytes(a.kv_dtype), a.host_index,
                a.block_rows, a.n_blocks, a.k_stride, a.group, a.scale, a.q, a.o, a.ml,
                a.q_dtype == SCOUT_BF16, a.o_dtype == SCOUT_BF16};
    const int n_units = a.n_units;
    int T = a.threads > 0 ? a.threads : static_cast<int>(std::thread::hardware_concurrency());
    if (T < 1) T = 1;
    if (T > n_units) T = n_units;
    const char* env = std::getenv("SCOUT_CPU_AMX");
    const bool amx = a.kv_dtype == SCOUT_BF16 && !(env && env[0] == '0') && amx_ready();
    const bool avx = has_avx512();
    std::atomic<int> next{0};
    // claim batch: units with no CPU-side block cost ~0.1 us, so a per-unit
    // atomic shared by 16 threads would dominate them; a batch holds about
    // two blocks' work (load balance at the tail), at most 16 units and at
    // least ~16 claims per thread
    long long total_blocks = 0;
    for (int u = 0; u < n_units; ++u) total_blocks += std::max(0, a.n_blocks[u]);
    const double per_unit = 0.05 + static_cast<double>(total_blocks) / n_units;  // in blocks
    const int batch = std::max(1, std::min({16, n_units / (16 * T), static_cast<int>(2.0 / per_unit)}));
    const std::function<void()> work = [&] {
        if (amx) {
            amx_work(j, next, n_units, batch);
            return;
        }
        for (int u0; (u0 = next.fetch_add(batch)) < n_units;)
            for (int u = u0; u < std::min(u0 + batch, n_units); ++u) {
                if (avx) run_unit<true>(j, u);
                else run_unit<false>(j, u);
            }
    };
    if (T == 1) work();
    else pool().run(T, work);
    return SCOUT_OK;
}

extern "C" int scout_cpu_partial_attention(const void* host_tier, int kv_dtype, const int64_t* host_index,
                                           const int32_t* block_rows, const int32_t* n_blocks, int k_stride,
                                           const float* q, int group, float scale, int n_units, float* o, float* ml,
                                           int threads) {
    CpuCoattnArgs a{};
    a.host_tier = host_tier;
    a.kv_dtype = kv_dtype;
    a.host_index = host_index;
    a.block_rows = block_rows;
    a.n_blocks = n_blocks;
    a.k_stride = k_stride;
    a.q = q;
    a.q_dtype = SCOUT_F32;
    a.group = group;
    a.scale = scale;
    a.n_units = n_units;
    a.o = o;
    a.o_dtype = SCOUT_F32;
    a.ml = ml;
    a.threads = threads;
    return scout_cpu_coattn_run(a);
}

extern "C" int scout_cpu_partial_attention_ex(const void* host_tier, int kv_dtype, const int64_t* host_index,
                                              const int32_t* block_rows, const int32_t* n_blocks, int k_stride,
                                              const void* q, int q_dtype, int group, float scale, int n_units, void* o,
                                              int o_dtype, float* ml, int threads) {
    CpuCoattnArgs a{};
    a.host_tier = host_tier;
    a.kv_dtype = kv_dtype;
    a.host_index = host_index;
    a.block_rows = block_rows;
    a.n_blocks = n_blocks;
    a.k_stride = k_stride;
    a.q = q;
    a.q_dtype = q_dtype;
    a.group = group;
    a.scale = scale;
    a.n_units = n_units;
    a.o = o;
    a.o_dtype = o_dtype;
    a.ml = ml;
    a.threads = threads;
    return scout_cpu_coattn_run(a);
}

extern "C" int scout_cpu_coattn_kernel(int kv_dtype) {
    const char* env = std::getenv("SCOUT_CPU_AMX");
    if (kv_dtype == SCOUT_BF16 && !(env && env[0] == '0') && amx_ready()) return 2;
    return has_avx512() ? 1 : 0;
}
