// K0 — KV slot writes and block-digest build.
//
// Replaces the data movement of TieredKvCache::append_token
// (reference proj/include/scout/kv_store.hpp:90-117) and build_digest
// (digest.hpp:34-60), which the reference re-runs over the whole open block on
// every append (kv_store.hpp:108). min/max is exact in any dtype, so the bf16
// digests equal the reference's double digests of the same bf16 keys.
#include "scout_common.cuh"

using namespace scout_dev;

namespace {

template <typename T>
__device__ __forceinline__ size_t elem_index(int r, int d);
template <>
__device__ __forceinline__ size_t elem_index<__nv_bfloat16>(int r, int d) {
    return static_cast<size_t>(bf16_tile_offset(r, d));
}
template <>
__device__ __forceinline__ size_t elem_index<float>(int r, int d) {
    return static_cast<size_t>(r) * D + d;
}

template <typename T>
__device__ __forceinline__ T from_f32(float x);
template <>
__device__ __forceinline__ __nv_bfloat16 from_f32<__nv_bfloat16>(float x) {
    return __float2bfloat16_rn(x);
}
template <>
__device__ __forceinline__ float from_f32<float>(float x) {
    return x;
}
__device__ __forceinline__ float to_f32(__nv_bfloat16 x) { return __bfloat162float(x); }
__device__ __forceinline__ float to_f32(float x) { return x; }

// std::min / std::max as build_digest folds them (digest.hpp:45-46): the
// running value is kept unless the new row compares strictly below / above,
// so signed zeros and NaNs fold exactly as in the reference.
__device__ __forceinline__ float ref_min(float acc, float v) { return v < acc ? v : acc; }
__device__ __forceinline__ float ref_max(float acc, float v) { return acc < v ? v : acc; }

// One CTA of 128 threads per token row: thread = channel.
template <typename T>
__global__ void kv_write_kernel(uint8_t* pool, const int32_t* slots, const int32_t* rows,
                                const float* k_rows, const float* v_rows, int n) {
    const int i = blockIdx.x;
    if (i >= n) return;
    const int c = threadIdx.x;
    const size_t tile = BS * D;
    T* base = reinterpret_cast<T*>(pool + static_cast<size_t>(slots[i]) * (2 * tile * sizeof(T)));
    const size_t off = elem_index<T>(rows[i], c);
    base[off] = from_f32<T>(k_rows[static_cast<size_t>(i) * D + c]);
    base[tile + off] = from_f32<T>(v_rows[static_cast<size_t>(i) * D + c]);
}

template <typename T>
__global__ void kv_read_kernel(const uint8_t* pool, const int32_t* slots, const int32_t* rows, float* k_rows,
                               float* v_rows, int n) {
    const int i = blockIdx.x;
    if (i >= n) return;
    const int c = threadIdx.x;
    const size_t tile = BS * D;
    const T* base = reinterpret_cast<const T*>(pool + static_cast<size_t>(slots[i]) * (2 * tile * sizeof(T)));
    const size_t off = elem_index<T>(rows[i], c);
    k_rows[static_cast<size_t>(i) * D + c] = to_f32(base[off]);
    v_rows[static_cast<size_t>(i) * D + c] = to_f32(base[tile + off]);
}

// minmax digest: thread = channel, sequential over rows (exact).
template <typename T>
__global__ void digest_minmax_kernel(const uint8_t* pool, int n, const int32_t* slots, const int32_t* block_rows,
                                     const int32_t* units, const int32_t* block_ids, T* digests, int nb_stride) {
    const int i = blockIdx.x;
    if (i >= n) return;
    const int c = threadIdx.x;
    const T* k = reinterpret_cast<const T*>(pool + static_cast<size_t>(slots[i]) * (2 * BS * D * sizeof(T)));
    const int rows = block_rows[i];
    float lo = to_f32(k[elem_index<T>(0, c)]);
    float hi = lo;
    for (int r = 1; r < rows; ++r) {
        const float v = to_f32(k[elem_index<T>(r, c)]);
        lo = ref_min(lo, v);
        hi = ref_max(hi, v);
    }
    T* dig = digests + static_cast<size_t>(units[i]) * 2 * D * nb_stride;
    dig[static_cast<size_t>(c) * nb_stride + block_ids[i]] = from_f32<T>(lo);
    dig[static_cast<size_t>(D + c) * nb_stride + block_ids[i]] = from_f32<T>(hi);
}

// mean digest (digest.hpp:52-57): column sum from 0.0 in row order, then / rows.
template <typename T>
__global__ void digest_mean_kernel(const uint8_t* pool, int n, const int32_t* slots, const int32_t* block_rows,
                                   const int32_t* units, const int32_t* block_ids, double* digests, int nb_stride) {
    const int i = blockIdx.x;
    if (i >= n) return;
    const int c = threadIdx.x;
    const T* k = reinterpret_cast<const T*>(pool + static_cast<size_t>(slots[i]) * (2 * BS * D * sizeof(T)));
    const int rows = block_rows[i];
    double s = 0.0;
    for (int r = 0; r < rows; ++r) s = __dadd_rn(s, static_cast<double>(to_f32(k[elem_index<T>(r, c)])));
    s = __ddiv_rn(s, static_cast<double>(rows));
    digests[static_cast<size_t>(units[i]) * D * nb_stride + static_cast<size_t>(c) * nb_stride + block_ids[i]] = s;
}

// Append one token to the open block of each unit (append_token,
// kv_store.hpp:90-117, one layer): the row lands at row n_tokens[u] % 64 of
// slot open_slot[u]; the digest column of block n_tokens[u] / 64 continues the
// reference's fold by one row (minmax: the fold of build_digest over the rows
// so far, bit-identical to rebuilding the open block as kv_store.hpp:108 does;
// mean: sequential double column sum over the stored rows / rows).
// Thread = channel, CTA = unit.
template <typename T, int METHOD>
__global__ void kv_append_kernel(uint8_t* pool, const int32_t* open_slot, int32_t* n_tokens, const float* k_rows,
                                 const float* v_rows, void* digests, int nb_stride, int advance) {
    const int u = blockIdx.x, c = threadIdx.x;
    const int pos = n_tokens[u];
    const int r = pos % BS, blk = pos / BS;
    const size_t tile = BS * D;
    T* base = reinterpret_cast<T*>(pool + static_cast<size_t>(open_slot[u]) * (2 * tile * sizeof(T)));
    const size_t off = elem_index<T>(r, c);
    const T kq = from_f32<T>(k_rows[static_cast<size_t>(u) * D + c]);
    base[off] = kq;
    base[tile + off] = from_f32<T>(v_rows[static_cast<size_t>(u) * D + c]);
    if constexpr (METHOD == SCOUT_DIGEST_MINMAX) {
        T* dig = static_cast<T*>(digests) + static_cast<size_t>(u) * 2 * D * nb_stride;
        T& lo = dig[static_cast<size_t>(c) * nb_stride + blk];
        T& hi = dig[static_cast<size_t>(D + c) * nb_stride + blk];
        const float v = to_f32(kq);
        if (r == 0) {
            lo = kq;
            hi = kq;
        } else {
            lo = from_f32<T>(ref_min(to_f32(lo), v));
            hi = from_f32<T>(ref_max(to_f32(hi), v));
        }
    } else {
        // the row just written is read back with the others (same stream order)
        __syncthreads();
        double s = 0.0;
        for (int rr = 0; rr <= r; ++rr) s = __dadd_rn(s, static_cast<double>(to_f32(base[elem_index<T>(rr, c)])));
        static_cast<double*>(digests)[static_cast<size_t>(u) * D * nb_stride + static_cast<size_t>(c) * nb_stride + blk] =
            __ddiv_rn(s, static_cast<double>(r + 1));
    }
    if (advance) {
        __syncthreads();
        if (c == 0) n_tokens[u] = pos + 1;
    }
}

}  // namespace

extern "C" int scout_kv_append(void* kv_pool, int kv_dtype, int method, int n_units, const int32_t* open_slot,
                               int32_t* n_tokens, const float* k_rows, const float* v_rows, void* digests,
                               int nb_stride, int advance, void* stream) {
    using namespace scout_host;
    if (n_units < 0 || nb_stride <= 0 ||
        (n_units > 0 && (!kv_pool || !open_slot || !n_tokens || !k_rows || !v_rows || !digests))) {
        set_error(SCOUT_ERR_INVALID_ARGUMENT, "append_token: bad arguments");
        return SCOUT_ERR_INVALID_ARGUMENT;
    }
    if (n_units == 0) return SCOUT_OK;
    auto st = static_cast<cudaStream_t>(stream);
    auto pool = static_cast<uint8_t*>(kv_pool);
    const int adv = advance ? 1 : 0;
    if (method == SCOUT_DIGEST_MINMAX && kv_dtype == SCOUT_BF16)
        kv_append_kernel<__nv_bfloat16, SCOUT_DIGEST_MINMAX><<<n_units, D, 0, st>>>(pool, open_slot, n_tokens, k_rows, v_rows, digests, nb_stride, adv);
    else if (method == SCOUT_DIGEST_MINMAX && kv_dtype == SCOUT_F32)
        kv_append_kernel<float, SCOUT_DIGEST_MINMAX><<<n_units, D, 0, st>>>(pool, open_slot, n_tokens, k_rows, v_rows, digests, nb_stride, adv);
    else if (method == SCOUT_DIGEST_MEAN && kv_dtype == SCOUT_BF16)
        kv_append_kernel<__nv_bfloat16, SCOUT_DIGEST_MEAN><<<n_units, D, 0, st>>>(pool, open_slot, n_tokens, k_rows, v_rows, digests, nb_stride, adv);
    else if (method == SCOUT_DIGEST_MEAN && kv_dtype == SCOUT_F32)
        kv_append_kernel<float, SCOUT_DIGEST_MEAN><<<n_units, D, 0, st>>>(pool, open_slot, n_tokens, k_rows, v_rows, digests, nb_stride, adv);
    else {
        set_error(SCOUT_ERR_UNSUPPORTED, "scout_kv_append: method %d / kv dtype %d unsupported", method, kv_dtype);
        return SCOUT_ERR_UNSUPPORTED;
    }
    return check_launch("scout_kv_append");
}

extern "C" int scout_kv_write_tokens(void* kv_pool, int kv_dtype, const int32_t* slots, const int32_t* rows,
                                     const float* k_rows, const float* v_rows, int n, void* stream) {
    using namespace scout_host;
    if (n < 0 || (n > 0 && (!kv_pool || !slots || !rows || !k_rows || !v_rows))) {
        set_error(SCOUT_ERR_INVALID_ARGUMENT, "scout_kv_write_tokens: null buffer or n < 0");
        return SCOUT_ERR_INVALID_ARGUMENT;
    }
    if (n == 0) return SCOUT_OK;
    auto st = static_cast<cudaStream_t>(stream);
    if (kv_dtype == SCOUT_BF16)
        kv_write_kernel<__nv_bfloat16><<<n, D, 0, st>>>(static_cast<uint8_t*>(kv_pool), slots, rows, k_rows, v_rows, n);
    else if (kv_dtype == SCOUT_F32)
        kv_write_kernel<float><<<n, D, 0, st>>>(static_cast<uint8_t*>(kv_pool), slots, rows, k_rows, v_rows, n);
    else {
        set_error(SCOUT_ERR_UNSUPPORTED, "scout_kv_write_tokens: kv dtype %d unsupported", kv_dtype);
        return SCOUT_ERR_UNSUPPORTED;
    }
    return check_launch("scout_kv_write_tokens");
}

extern "C" int scout_kv_read_tokens(const void* kv_pool, int kv_dtype, const int32_t* slots, const int32_t* rows,
                                    float* k_rows, float* v_rows, int n, void* stream) {
    using namespace scout_host;
    if (n < 0 || (n > 0 && (!kv_pool || !slots || !rows || !k_rows || !v_rows))) {
        set_error(SCOUT_ERR_INVALID_ARGUMENT, "scout_kv_read_tokens: null buffer or n < 0");
        return SCOUT_ERR_INVALID_ARGUMENT;
    }
    if (n == 0) return SCOUT_OK;
    auto st = static_cast<cudaStream_t>(stream);
    if (kv_dtype == SCOUT_BF16)
        kv_read_kernel<__nv_bfloat16><<<n, D, 0, st>>>(static_cast<const uint8_t*>(kv_pool), slots, rows, k_rows, v_rows, n);
    else if (kv_dtype == SCOUT_F32)
        kv_read_kernel<float><<<n, D, 0, st>>>(static_cast<const uint8_t*>(kv_pool), slots, rows, k_rows, v_rows, n);
    else {
        set_error(SCOUT_ERR_UNSUPPORTED, "scout_kv_read_tokens: kv dtype %d unsupported", kv_dtype);
        return SCOUT_ERR_UNSUPPORTED;
    }
    return check_launch("scout_kv_read_tokens");
}

extern "C" int scout_digest_build(const void* kv_pool, int kv_dtype, int method, int n, const int32_t* slots,
                                  const int32_t* block_rows, const int32_t* units, const int32_t* block_ids,
                                  void* digests, int nb_stride, void* stream) {
    using namespace scout_host;
    if (n < 0 || nb_stride <= 0 ||
        (n > 0 && (!kv_pool || !slots || !block_rows || !units || !block_ids || !digests))) {
        set_error(SCOUT_ERR_INVALID_ARGUMENT, "scout_digest_build: bad arguments");
        return SCOUT_ERR_INVALID_ARGUMENT;
    }
    if (n == 0) return SCOUT_OK;
    auto st = static_cast<cudaStream_t>(stream);
    auto pool = static_cast<const uint8_t*>(kv_pool);
    if (method == SCOUT_DIGEST_MINMAX) {
        if (kv_dtype == SCOUT_BF16)
            digest_minmax_kernel<__nv_bfloat16><<<n, D, 0, st>>>(pool, n, slots, block_rows, units, block_ids,
                                                                 static_cast<__nv_bfloat16*>(digests), nb_stride);
        else if (kv_dtype == SCOUT_F32)
            digest_minmax_kernel<float><<<n, D, 0, st>>>(pool, n, slots, block_rows, units, block_ids,
                                                         static_cast<float*>(digests), nb_stride);
        else {
            set_error(SCOUT_ERR_UNSUPPORTED, "scout_digest_build: kv dtype %d unsupported", kv_dtype);
            return SCOUT_ERR_UNSUPPORTED;
        }
    } else if (method == SCOUT_DIGEST_MEAN) {
        if (kv_dtype == SCOUT_BF16)
            digest_mean_kernel<__nv_bfloat16><<<n, D, 0, st>>>(pool, n, slots, block_rows, units, block_ids,
                                                               static_cast<double*>(digests), nb_stride);
        else if (kv_dtype == SCOUT_F32)
            digest_mean_kernel<float><<<n, D, 0, st>>>(pool, n, slots, block_rows, units, block_ids,
                                                       static_cast<double*>(digests), nb_stride);
        else {
            set_error(SCOUT_ERR_UNSUPPORTED, "scout_digest_build: kv dtype %d unsupported", kv_dtype);
            return SCOUT_ERR_UNSUPPORTED;
        }
    } else {
        set_error(SCOUT_ERR_INVALID_ARGUMENT, "scout_digest_build: unknown method %d", method);
        return SCOUT_ERR_INVALID_ARGUMENT;
    }
    return check_launch("scout_digest_build");
}
