// Internal (engine <-> K2) interface of the persistent multi-layer K2 launch.
// Not part of the public C ABI: scout_sparse_decode wraps it for one layer,
// the engine drives it for a whole decode step.
#pragma once
#include <cuda_runtime.h>
#include <stdint.h>

constexpr int K2_MAX_LAYERS = 96;  // kernel parameters carry the per-layer I/O by value

struct K2Layer {
    const void* q;           // [U*G][128] true query of the layer (f32, or bf16 if q_bf16)
    const int32_t* res_slots;
    const int32_t* res_ids;
    const int32_t* n_res;
    const void* cpu_o;       // optional CPU partial (f32, or bf16 when K2StepArgs::cpu_bf16)
    const float* cpu_ml;
    float* o;
    float* ml;
    const unsigned* in_flag;  // optional: inputs of this layer landed when *in_flag >= token
    unsigned recall_token;    // > 0: wait recall_flag[layer] >= recall_token before streaming
    unsigned pad;
};

// NL: layer slots. The struct is the kernel's parameter block: a single-layer
// launch uses the 1-slot form (~170 B of parameters instead of ~8 KB)
template <int NL>
struct K2StepArgsT {
    int n_units, group, k_stride, n_layers;
    float scale;
    const void* kv_pool;
    const int32_t* n_tokens;
    void* workspace;          // n_layers consecutive per-layer workspaces
    size_t ws_layer_bytes;
    const unsigned* k1_flag;  // optional [n_layers]: K1 published layer L when >= token
    const unsigned* recall_flag;  // optional [n_layers]
    unsigned* layer_done;     // optional [n_layers]: += 1 per CTA when its share of layer L is written
    unsigned token;
    int max_ctas;
    int q_bf16;               // queries are bf16 (else f32)
    int cpu_bf16;             // CPU partial o is bf16 (else f32); its (m, l) stay f32
    unsigned long long* prof; // optional [grid][16] cycle counters (SCOUT_K2_PROF diagnostics)
    int l2_prefetch;          // blocks the producer prefetches into L2 ahead of the ring (0: none)
    unsigned done_extra;      // CTA 0 adds this to layer_done too (a launch narrower than the
                              // engine's grid still counts `grid` per layer)
    K2Layer layers[NL];
};
using K2StepArgs = K2StepArgsT<K2_MAX_LAYERS>;

// per-layer workspace bytes for n_units units and a grid of `grid` CTAs
size_t scout_k2_ws_layer_bytes(int n_units, int grid);
// grid the launch will use for n_units / k_stride (persistent: <= one CTA per SM unless the
// per-CTA plan limits force more)
int scout_k2_grid(int n_units, int k_stride, int max_ctas);
// launch the bf16 tensor-core K2 over a.n_layers layers
int scout_k2_launch(const K2StepArgs& a, cudaStream_t st, bool pdl);
