// CPU co-attention worker: the host half of ScoutAttention.
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

#include <algorithm>
#include <atomic>
#include <cmath>
#include <cstdint>
#include <cstring>
#include <limits>
#include <thread>
#include <vector>

#include "../../include/scout_b200.h"

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
    const float* q;
    float* o;
    float* ml;
};

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
    const float* qu = j.q + static_cast<size_t>(u) * G * D;
    const int nb = j.n_blocks[u];
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
        for (int d = 0; d < D; ++d) j.o[h * D + d] = acc[g][d] * inv;
        j.ml[h * 2] = l[g] > 0.f ? m[g] : -std::numeric_limits<float>::infinity();
        j.ml[h * 2 + 1] = l[g];
    }
}

bool has_avx512() {
    static const int v = __builtin_cpu_supports("avx512f") ? 1 : 0;
    return v != 0;
}

}  // namespace

extern "C" int scout_cpu_partial_attention(const void* host_tier, int kv_dtype, const int64_t* host_index,
                                           const int32_t* block_rows, const int32_t* n_blocks, int k_stride,
                                           const float* q, int group, float scale, int n_units, float* o, float* ml,
                                           int threads) {
    using scout_host::set_error;
    if (n_units < 0 || k_stride <= 0 || group < 1 || group > GMAX || !(scale > 0.f) ||
        (kv_dtype != SCOUT_BF16 && kv_dtype != SCOUT_F32) ||
        (n_units > 0 && (!host_tier || !host_index || !n_blocks || !q || !o || !ml))) {
        set_error(SCOUT_ERR_INVALID_ARGUMENT, "scout_cpu_partial_attention: bad arguments");
        return SCOUT_ERR_INVALID_ARGUMENT;
    }
    if (n_units == 0) return SCOUT_OK;
    const Job j{static_cast<const uint8_t*>(host_tier), kv_dtype, scout_slot_bytes(kv_dtype), host_index, block_rows,
                n_blocks, k_stride, group, scale, q, o, ml};
    int T = threads > 0 ? threads : static_cast<int>(std::thread::hardware_concurrency());
    if (T < 1) T = 1;
    if (T > n_units) T = n_units;
    const bool avx = has_avx512();
    std::atomic<int> next{0};
    auto work = [&] {
        for (int u; (u = next.fetch_add(1)) < n_units;) {
            if (avx) run_unit<true>(j, u);
            else run_unit<false>(j, u);
        }
    };
    if (T == 1) {
        work();
        return SCOUT_OK;
    }
    std::vector<std::thread> pool;
    pool.reserve(T - 1);
    for (int t = 1; t < T; ++t) pool.emplace_back(work);
    work();
    for (auto& th : pool) th.join();
    return SCOUT_OK;
}
