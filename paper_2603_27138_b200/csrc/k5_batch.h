// Internal (engine <-> K5) multi-layer launches of the device tier mode. Not
// part of the public C ABI: the engine drives them for a whole decode step.
#pragma once
#include <cuda_runtime.h>
#include <stdint.h>

#include "../../include/scout_b200.h"

constexpr int K5_MAX_LAYERS = 96;

struct TierPostArgs {
    const scout_tier_layer* layers;  // device array [n_layers]
    int n_layers, nbs, k, step, ticket_base;
    int layer0;                      // first layer of this launch (grid.y layers from it)
    const int32_t* n_tokens;         // count before the append (advanced after the launch)
    uint8_t* pool;                   // KV pool: bf16 tile slots, or f32 row-major slots (kv_f32)
    int kv_f32;
    const float* k_new;              // [L][U][128]
    const float* v_new;
    void* digests[K5_MAX_LAYERS];    // per layer [U][2][128][nbs] in the KV dtype
    uint8_t* host_tier;              // device view of the pinned host tier (nullptr: no write-through)
    long long host_blocks;
    int host_units, host_unit0;      // image index ((l * host_units + host_unit0 + u) * nbs + id) % host_blocks
    const int32_t* sel_ids;          // [L][U][k] K1's selection of this step (the layer's predicted set)
    const int32_t* n_sel;            // [L][U]
    int32_t* rc_ids;                 // [L][U][k] out: the recalled ids (predicted \ residency after the
    int32_t* rc_n;                   //   append, maybe_schedule_recall recall.hpp:114-126), count [L][U]
    int32_t* dst;                    // [L][U][k] recall destination slots (-2 - slot: warm, no copy; -1 rejected)
    unsigned long long* rc_stats;    // optional [2]: recalled blocks served warm / to copy (summed)
    // K1's split of this step, checked against the selection (check_split,
    // engine.hpp:317-329): [L][U][k] ascending lists and [L][U] counts
    const int32_t *res_ids, *n_res, *cpu_ids, *n_cpu, *res_tok, *cpu_tok;
    int32_t* plan_out;               // optional [L][U][nbs]: the planning view of step plan_step,
    int plan_step;                   //   written once the layer's bookkeeping is done
    uint8_t recall_due[K5_MAX_LAYERS];
};

// begin_layer's ticket application for several layers in one launch
struct TierApplyArgs {
    const scout_tier_layer* layers;  // device array [n_layers]
    int nbs, n;
    const int32_t* n_tokens;
    int layer[K5_MAX_LAYERS];        // the layers with a ticket due
    int due_tick[K5_MAX_LAYERS];
};

// GpuSidePolicy::all_resident: every fast block of layers [layer0, layer0 +
// n) in ascending id order (ids / slots [L][U][stride], counts n [L][U],
// indexed by absolute layer). layers (tier mode, device array) or tables
// (static mode: per-layer block tables [U][nbs], slot or -1).
struct ResidentListArgs {
    const scout_tier_layer* layers;
    const int32_t* tables[K5_MAX_LAYERS];
    int nbs, layer0, stride;
    const int32_t* n_tokens;
    int32_t *ids, *slots, *n;
};
int scout_tier_resident_lists(const ResidentListArgs& a, int n_units, int n_layers_launch, cudaStream_t st);

int scout_tier_plan_layers(const scout_tier_layer* layers_dev, int n_layers, int n_units, int nb_stride,
                           const int32_t* n_tokens, int step, int32_t* tables, cudaStream_t st);
// post-attention bookkeeping of layers [a.layer0, a.layer0 + n_layers_launch)
int scout_tier_post_layers(const TierPostArgs& a, int n_units, int n_layers_launch, cudaStream_t st);
int scout_tier_apply_layers(const TierApplyArgs& a, int n_units, cudaStream_t st);
// n_tokens += 1 once every layer has appended
int scout_tier_advance(int32_t* n_tokens, int n_units, cudaStream_t st);
