// K3 — standalone LSE merge of partial sets; K4 — periodic-recall gather.
//
// K3 replaces merge (reference proj/include/scout/attention.hpp:100-114) for
// callers that keep GPU and CPU partials apart (the fused path lives in K2).
// Partials are (o normalised, m, l): the reference's (o_acc, max_logit, denom)
// with o = o_acc / denom. Empty operands are exact identities (:101-102); both
// empty give o = 0 (engine.hpp:273) and ml = (-inf, 0).
//
// K4 moves the bytes that TieredKvCache::begin_layer (kv_store.hpp:201-218)
// only flags: whole block images from device-mapped pinned host memory into
// freed pool slots, on a side stream, 16-byte loads over PCIe / C2C.
#include "scout_common.cuh"
#include "k4_batch.h"

#include <math_constants.h>

#include <vector>

using namespace scout_dev;

namespace {

__global__ void merge_kernel(const float* __restrict__ a_o, const float* __restrict__ a_ml,
                             const float* __restrict__ b_o, const float* __restrict__ b_ml, float* out_o,
                             float* out_ml, int n_rows) {
    const int row = blockIdx.x;
    if (row >= n_rows) return;
    const int d = threadIdx.x;  // 0..127
    const float ma = a_ml[2 * row], la = a_ml[2 * row + 1];
    const float mb = b_ml[2 * row], lb = b_ml[2 * row + 1];
    const float oa = a_o[static_cast<size_t>(row) * D + d], ob = b_o[static_cast<size_t>(row) * D + d];
    float o, m, l;
    if (!(la > 0.f) && !(lb > 0.f)) {
        o = 0.f; m = -CUDART_INF_F; l = 0.f;
    } else if (!(la > 0.f)) {
        o = ob; m = mb; l = lb;
    } else if (!(lb > 0.f)) {
        o = oa; m = ma; l = la;
    } else {
        m = fmaxf(ma, mb);
        const float wa = la * expf(ma - m), wb = lb * expf(mb - m);
        l = wa + wb;
        o = (wa * oa + wb * ob) / l;
    }
    __syncthreads();  // out may alias a
    out_o[static_cast<size_t>(row) * D + d] = o;
    if (d == 0) { out_ml[2 * row] = m; out_ml[2 * row + 1] = l; }
}

// One CTA per recalled block; each thread keeps 4 x 16 B loads in flight.
__global__ void __launch_bounds__(256) recall_gather_kernel(uint8_t* pool, const uint8_t* host, const int64_t* src,
                                                            const int32_t* dst, int n, size_t slot_bytes) {
    const int i = blockIdx.x;
    if (i >= n) return;
    const int4* s = reinterpret_cast<const int4*>(host + static_cast<size_t>(src[i]) * slot_bytes);
    int4* d = reinterpret_cast<int4*>(pool + static_cast<size_t>(dst[i]) * slot_bytes);
    const int nvec = static_cast<int>(slot_bytes / 16);
    for (int base = threadIdx.x; base < nvec; base += 4 * blockDim.x) {
        int4 v[4];
#pragma unroll
        for (int k = 0; k < 4; ++k) {
            const int idx = base + k * blockDim.x;
            if (idx < nvec) v[k] = __ldcv(s + idx);
        }
#pragma unroll
        for (int k = 0; k < 4; ++k) {
            const int idx = base + k * blockDim.x;
            if (idx < nvec) d[idx] = v[k];
        }
    }
}

}  // namespace

extern "C" int scout_merge_partials(const float* a_o, const float* a_ml, const float* b_o, const float* b_ml,
                                    float* out_o, float* out_ml, int n_rows, void* stream) {
    using namespace scout_host;
    if (n_rows < 0 || (n_rows > 0 && (!a_o || !a_ml || !b_o || !b_ml || !out_o || !out_ml))) {
        set_error(SCOUT_ERR_INVALID_ARGUMENT, "scout_merge_partials: bad arguments");
        return SCOUT_ERR_INVALID_ARGUMENT;
    }
    if (n_rows == 0) return SCOUT_OK;
    merge_kernel<<<n_rows, D, 0, static_cast<cudaStream_t>(stream)>>>(a_o, a_ml, b_o, b_ml, out_o, out_ml, n_rows);
    return check_launch("scout_merge_partials");
}

extern "C" int scout_recall_gather(void* kv_pool, int kv_dtype, const void* host_blocks, const int64_t* src_index,
                                   const int32_t* dst_slots, int n, void* stream) {
    using namespace scout_host;
    if (kv_dtype != SCOUT_BF16 && kv_dtype != SCOUT_F32) {
        set_error(SCOUT_ERR_UNSUPPORTED, "scout_recall_gather: kv dtype %d unsupported", kv_dtype);
        return SCOUT_ERR_UNSUPPORTED;
    }
    if (n < 0 || (n > 0 && (!kv_pool || !host_blocks || !src_index || !dst_slots))) {
        set_error(SCOUT_ERR_INVALID_ARGUMENT, "scout_recall_gather: bad arguments");
        return SCOUT_ERR_INVALID_ARGUMENT;
    }
    if (n == 0) return SCOUT_OK;
    // pinned host memory is mapped under UVA; translate in case the mapping differs
    void* dev_view = nullptr;
    if (cudaHostGetDevicePointer(&dev_view, const_cast<void*>(host_blocks), 0) == cudaSuccess && dev_view)
        host_blocks = dev_view;
    else
        cudaGetLastError();  // not a registered host pointer: use as given (e.g. device memory)
    recall_gather_kernel<<<n, 256, 0, static_cast<cudaStream_t>(stream)>>>(
        static_cast<uint8_t*>(kv_pool), static_cast<const uint8_t*>(host_blocks), src_index, dst_slots, n,
        slot_bytes(kv_dtype));
    return check_launch("scout_recall_gather");
}

extern "C" int scout_recall_copy(void* kv_pool, int kv_dtype, const void* host_blocks, const int64_t* src_index,
                                 const int32_t* dst_slots, int n, void* stream) {
    using namespace scout_host;
    if (kv_dtype != SCOUT_BF16 && kv_dtype != SCOUT_F32) {
        set_error(SCOUT_ERR_UNSUPPORTED, "scout_recall_copy: kv dtype %d unsupported", kv_dtype);
        return SCOUT_ERR_UNSUPPORTED;
    }
    if (n < 0 || (n > 0 && (!kv_pool || !host_blocks || !src_index || !dst_slots)) || stream == nullptr) {
        set_error(SCOUT_ERR_INVALID_ARGUMENT, "scout_recall_copy: bad arguments (a non-default stream is required)");
        return SCOUT_ERR_INVALID_ARGUMENT;
    }
    if (n == 0) return SCOUT_OK;
    // one cudaMemcpyAsync per run of consecutive (source image, destination
    // slot) pairs: the copy engines pay a fixed cost per call (~5 us), so a
    // scattered list moves at a few GB/s -- the SM gather (scout_recall_gather)
    // is the fast path for scattered recalls
    const size_t sb = slot_bytes(kv_dtype);
    auto* pool = static_cast<uint8_t*>(kv_pool);
    const auto* host = static_cast<const uint8_t*>(host_blocks);
    for (int i = 0; i < n;) {
        int j = i + 1;
        while (j < n && src_index[j] == src_index[j - 1] + 1 && dst_slots[j] == dst_slots[j - 1] + 1) ++j;
        if (cudaMemcpyAsync(pool + static_cast<size_t>(dst_slots[i]) * sb, host + static_cast<size_t>(src_index[i]) * sb,
                            static_cast<size_t>(j - i) * sb, cudaMemcpyHostToDevice,
                            static_cast<cudaStream_t>(stream)) != cudaSuccess) {
            set_error(SCOUT_ERR_CUDA, "scout_recall_copy: %s", cudaGetErrorString(cudaGetLastError()));
            return SCOUT_ERR_CUDA;
        }
        i = j;
    }
    return SCOUT_OK;
}

// ---------------------------------------------------------------------------
// Device-driven tier data movement (the engine's device-tier mode): the block
// lists live in HBM (K1's CPU-side ids, K5's slots), so the copies are issued
// by kernels instead of host copy descriptors.
//   host tier layout: block (layer, unit, id) at index (layer * n_units + unit) * nb_stride + id,
//   modulo host_blocks when host_blocks > 0 (a bounded synthetic tier: images alias)
namespace {

__device__ __forceinline__ long long host_index(long long base, int u, int nb_stride, int id, long long host_blocks) {
    const long long i = base + static_cast<long long>(u) * nb_stride + id;
    return host_blocks > 0 ? i % host_blocks : i;
}

// recall: unit u's n_ids[u] blocks ids[u][i] -> pool slots dst[u][i] (-1:
// rejected ticket). A small fixed grid loops over the units: the copies are
// PCIe-bound anyway, and a narrow footprint leaves the SMs' thread / register
// room to the persistent K2 that runs next to it (a wide grid of gather CTAs
// held K2's CTAs back from launching).
__global__ void __launch_bounds__(256) recall_ids_kernel(uint8_t* pool, const uint8_t* host, long long host_base,
                                                         int nb_stride, long long host_blocks, const int32_t* ids,
                                                         const int32_t* n_ids, const int32_t* dst, int k_stride,
                                                         size_t slot_bytes, int n_units) {
    const int nvec = static_cast<int>(slot_bytes / 16);
    for (int u = blockIdx.x; u < n_units; u += gridDim.x) {
        const int n = n_ids[u];
        for (int i = 0; i < n; ++i) {
            const int slot = dst[static_cast<size_t>(u) * k_stride + i];
            if (slot < 0) continue;
            const long long hb = host_index(host_base, u, nb_stride, ids[static_cast<size_t>(u) * k_stride + i], host_blocks);
            const int4* s = reinterpret_cast<const int4*>(host + static_cast<size_t>(hb) * slot_bytes);
            int4* d = reinterpret_cast<int4*>(pool + static_cast<size_t>(slot) * slot_bytes);
            for (int base = threadIdx.x; base < nvec; base += 4 * blockDim.x) {
                int4 v[4];
#pragma unroll
                for (int k = 0; k < 4; ++k) {
                    const int idx = base + k * blockDim.x;
                    if (idx < nvec) v[k] = __ldcv(s + idx);
                }
#pragma unroll
                for (int k = 0; k < 4; ++k) {
                    const int idx = base + k * blockDim.x;
                    if (idx < nvec) d[idx] = v[k];
                }
            }
        }
    }
}

// every due layer of a step in one launch (k4_batch.h): blockIdx.y picks the
// layer, the CTAs of a layer loop over its units as recall_ids_kernel does;
// the last CTA of a layer to finish publishes the layer's flag (release
// after a fence, so the next K2 sees the copies once it sees the flag)
__global__ void __launch_bounds__(256) recall_layers_kernel(const RecallLayersArgs a) {
    const int layer = a.layer[blockIdx.y];
    const int nvec = static_cast<int>(a.slot_bytes / 16);
    const size_t lu = static_cast<size_t>(layer) * a.n_units;
    const long long hbase = a.host_base0 + static_cast<long long>(layer) * a.host_layer_stride;
    for (int u = blockIdx.x; u < a.n_units; u += gridDim.x) {
        const int n = a.n_ids[lu + u];
        const size_t row = (lu + u) * a.k_stride;
        for (int i = 0; i < n; ++i) {
            const int slot = a.dst[row + i];
            if (slot < 0) continue;  // a warm slot (its image is in place) or a rejected ticket
            const long long hb = host_index(hbase, u, a.nb_stride, a.ids[row + i], a.host_blocks);
            const int4* s = reinterpret_cast<const int4*>(a.host + static_cast<size_t>(hb) * a.slot_bytes);
            int4* d = reinterpret_cast<int4*>(a.pool + static_cast<size_t>(slot) * a.slot_bytes);
            for (int base = threadIdx.x; base < nvec; base += 4 * blockDim.x) {
                int4 v[4];
#pragma unroll
                for (int k = 0; k < 4; ++k) {
                    const int idx = base + k * blockDim.x;
                    if (idx < nvec) v[k] = __ldcv(s + idx);
                }
#pragma unroll
                for (int k = 0; k < 4; ++k) {
                    const int idx = base + k * blockDim.x;
                    if (idx < nvec) d[idx] = v[k];
                }
            }
        }
    }
    __syncthreads();
    if (threadIdx.x == 0) {
        __threadfence();
        if (atomicAdd(a.ctr + layer, 1u) == gridDim.x - 1) {
            a.ctr[layer] = 0;
            __threadfence();
            asm volatile("st.release.gpu.global.u32 [%0], %1;" ::"l"(a.flags + layer), "r"(a.token) : "memory");
        }
    }
}

// seal write-through: the block unit u sealed (sealed_id[u] >= 0, slot
// open_slot[u]) is copied to its host-tier image, which becomes the slow copy
__global__ void __launch_bounds__(256) writeback_kernel(const uint8_t* pool, uint8_t* host, long long host_base,
                                                        int nb_stride, long long host_blocks, const int32_t* open_slot,
                                                        const int32_t* sealed_id, size_t slot_bytes) {
    const int u = blockIdx.x;
    const int id = sealed_id[u];
    if (id < 0) return;
    const int4* s = reinterpret_cast<const int4*>(pool + static_cast<size_t>(open_slot[u]) * slot_bytes);
    int4* d = reinterpret_cast<int4*>(host + static_cast<size_t>(host_index(host_base, u, nb_stride, id, host_blocks)) *
                                      slot_bytes);
    const int nvec = static_cast<int>(slot_bytes / 16);
    for (int i = threadIdx.x; i < nvec; i += blockDim.x) d[i] = __ldcg(s + i);
}

const void* device_view(const void* host) {
    void* dv = nullptr;
    if (cudaHostGetDevicePointer(&dv, const_cast<void*>(host), 0) == cudaSuccess && dv) return dv;
    cudaGetLastError();
    return host;
}

}  // namespace

extern "C" int scout_recall_gather_ids(void* kv_pool, int kv_dtype, const void* host_tier, long long host_base,
                                       int nb_stride, long long host_blocks, int n_units, const int32_t* ids, const int32_t* n_ids,
                                       const int32_t* dst_slots, int k_stride, int ctas, void* stream) {
    using namespace scout_host;
    if (kv_dtype != SCOUT_BF16 && kv_dtype != SCOUT_F32) {
        set_error(SCOUT_ERR_UNSUPPORTED, "scout_recall_gather_ids: kv dtype %d unsupported", kv_dtype);
        return SCOUT_ERR_UNSUPPORTED;
    }
    if (n_units < 0 || nb_stride <= 0 || k_stride <= 0 ||
        (n_units > 0 && (!kv_pool || !host_tier || !ids || !n_ids || !dst_slots))) {
        set_error(SCOUT_ERR_INVALID_ARGUMENT, "scout_recall_gather_ids: bad arguments");
        return SCOUT_ERR_INVALID_ARGUMENT;
    }
    if (n_units == 0) return SCOUT_OK;
    int grid = ctas > 0 ? ctas : 32;
    if (grid > n_units) grid = n_units;
    recall_ids_kernel<<<grid, 256, 0, static_cast<cudaStream_t>(stream)>>>(
        static_cast<uint8_t*>(kv_pool), static_cast<const uint8_t*>(device_view(host_tier)), host_base, nb_stride,
        host_blocks, ids, n_ids, dst_slots, k_stride, slot_bytes(kv_dtype), n_units);
    return check_launch("scout_recall_gather_ids");
}

int scout_recall_gather_layers(RecallLayersArgs a, const void* host_tier, int kv_dtype, int ctas, cudaStream_t st) {
    using namespace scout_host;
    if ((kv_dtype != SCOUT_BF16 && kv_dtype != SCOUT_F32) || a.n < 1 || a.n > K4_MAX_LAYERS || a.n_units < 1 ||
        !host_tier || !a.pool || !a.flags || !a.ctr) {
        set_error(SCOUT_ERR_INVALID_ARGUMENT, "recall gather (layers): bad arguments");
        return SCOUT_ERR_INVALID_ARGUMENT;
    }
    a.host = static_cast<const uint8_t*>(device_view(host_tier));
    a.slot_bytes = slot_bytes(kv_dtype);
    int grid = ctas > 0 ? ctas : 32;
    if (grid > a.n_units) grid = a.n_units;
    recall_layers_kernel<<<dim3(grid, a.n), 256, 0, st>>>(a);
    return check_launch("recall gather (layers)");
}

extern "C" int scout_kv_writeback(const void* kv_pool, int kv_dtype, void* host_tier, long long host_base, int nb_stride,
                                  long long host_blocks, int n_units, const int32_t* open_slot, const int32_t* sealed_id, void* stream) {
    using namespace scout_host;
    if (kv_dtype != SCOUT_BF16 && kv_dtype != SCOUT_F32) {
        set_error(SCOUT_ERR_UNSUPPORTED, "scout_kv_writeback: kv dtype %d unsupported", kv_dtype);
        return SCOUT_ERR_UNSUPPORTED;
    }
    if (n_units < 0 || nb_stride <= 0 || (n_units > 0 && (!kv_pool || !host_tier || !open_slot || !sealed_id))) {
        set_error(SCOUT_ERR_INVALID_ARGUMENT, "scout_kv_writeback: bad arguments");
        return SCOUT_ERR_INVALID_ARGUMENT;
    }
    if (n_units == 0) return SCOUT_OK;
    writeback_kernel<<<n_units, 256, 0, static_cast<cudaStream_t>(stream)>>>(
        static_cast<const uint8_t*>(kv_pool), static_cast<uint8_t*>(const_cast<void*>(device_view(host_tier))), host_base,
        nb_stride, host_blocks, open_slot, sealed_id, slot_bytes(kv_dtype));
    return check_launch("scout_kv_writeback");
}
