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
    int nowait;   // publish without griddepcontrol.wait (launched as a programmatic dependent of a
                  // grid that itself waits for this one's flags: the overlapped step)
    int slots;    // > 0: persistent grid of exactly this many CTAs; < 0: resident CTAs on -slots SMs
    unsigned* all_ctr;   // optional: layers published so far (reset by the last)
    unsigned* all_flag;  // optional: = all_token once every layer of the launch has published
    unsigned all_token;
    scout_topk_args a[NA];
};
using K1Batch = K1BatchT<K1_MAX_LAYERS>;
using K1Batch1 = K1BatchT<1>;

int scout_k1_launch_batch(const scout_topk_args* layers, int n, cudaStream_t st);
// the overlapped step's K1: a persistent grid on `sms` SMs, launched as a
// programmatic dependent of the running K2, publishing without waiting for it
int scout_k1_launch_batch_beside(const scout_topk_args* layers, int n, int sms, cudaStream_t st,
                                 unsigned* all_ctr = nullptr, unsigned* all_flag = nullptr, unsigned all_token = 0);
