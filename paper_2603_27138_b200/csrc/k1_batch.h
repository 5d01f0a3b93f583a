// Internal: one K1 launch over many layers (grid = units x layers); the
// per-layer arguments travel by value in the kernel parameters.
#pragma once
#include <cuda_runtime.h>

#include "../../include/scout_b200.h"

constexpr int K1_MAX_LAYERS = 96;

// NA: argument slots. The whole struct is the kernel's parameter block, so a
// single-layer launch uses the 1-slot form: ~200 B instead of ~17 KB of
// parameters for the driver to copy into the command queue per launch (the
// 17 KB form cost ~45 us of host time per launch in the layer-by-layer mode)
template <int NA>
struct K1BatchT {
    int n;
    int nbuf;   // digest ring depth (set at launch)
    int chunk;  // digest chunk bytes (set at launch)
    int persist;  // persistent grid over (layer, unit) items (set at launch)
    int direct;   // bf16 digests read straight from global memory, no ring (set at launch)
    scout_topk_args a[NA];
};
using K1Batch = K1BatchT<K1_MAX_LAYERS>;
using K1Batch1 = K1BatchT<1>;

int scout_k1_launch_batch(const scout_topk_args* layers, int n, cudaStream_t st);
