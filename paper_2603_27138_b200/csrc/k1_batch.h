// Internal: one K1 launch over many layers (grid = units x layers); the
// per-layer arguments travel by value in the kernel parameters.
#pragma once
#include <cuda_runtime.h>

#include "../../include/scout_b200.h"

constexpr int K1_MAX_LAYERS = 96;

struct K1Batch {
    int n;
    int nbuf;   // digest ring depth (set at launch)
    int chunk;  // digest chunk bytes (set at launch)
    int persist;  // persistent grid over (layer, unit) items (set at launch)
    int direct;   // bf16 digests read straight from global memory, no ring (set at launch)
    scout_topk_args a[K1_MAX_LAYERS];
};

int scout_k1_launch_batch(const scout_topk_args* layers, int n, cudaStream_t st);
