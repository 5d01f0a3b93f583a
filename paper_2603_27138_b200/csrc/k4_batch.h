// Internal: one recall-gather launch over every due layer of a step (device
// tier mode, SM gather): grid = (ctas, layers); the last CTA of a layer
// publishes its recall flag, so neither per-layer launches nor per-layer
// stream writes sit between the step's bookkeeping and the next K2.
#pragma once
#include <cuda_runtime.h>

#include <cstddef>
#include <cstdint>

constexpr int K4_MAX_LAYERS = 128;

struct RecallLayersArgs {
    uint8_t* pool;
    const uint8_t* host;            // host tier (device view set at launch)
    size_t slot_bytes;
    int nb_stride, n_units, k_stride;
    long long host_blocks;          // > 0: image indices modulo host_blocks
    long long host_base0;           // host_base(layer) = host_base0 + layer * host_layer_stride
    long long host_layer_stride;
    const int32_t* ids;             // [layers][n_units][k_stride]
    const int32_t* n_ids;           // [layers][n_units]
    const int32_t* dst;             // [layers][n_units][k_stride]: pool slot, < 0: nothing to copy
    unsigned* flags;                // [layers]: recall flag, = token once the layer's copies landed
    unsigned* ctr;                  // [layers]: CTAs done (reset by the last one)
    unsigned token;
    int n;                          // due layers
    int16_t layer[K4_MAX_LAYERS];
};

int scout_recall_gather_layers(RecallLayersArgs a, const void* host_tier, int kv_dtype, int ctas, cudaStream_t st);
