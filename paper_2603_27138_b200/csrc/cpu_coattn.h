// Internal (engine <-> CPU co-attention worker) interface: the worker with
// the element types the engine's host path moves (bf16 queries in, bf16 or
// f32 partials out). The C ABI scout_cpu_partial_attention is its f32 case.
#pragma once
#include <stdint.h>

struct CpuCoattnArgs {
    const void* host_tier;      // block images (pool slot layout)
    int kv_dtype;               // SCOUT_BF16 / SCOUT_F32
    const int64_t* host_index;  // [n_units][k_stride] image index of block i of unit u
    const int32_t* block_rows;  // optional [n_units][k_stride] valid rows (NULL: 64)
    const int32_t* n_blocks;    // [n_units]
    int k_stride;
    const void* q;              // [n_units][G][128] in q_dtype
    int q_dtype;                // SCOUT_F32 / SCOUT_BF16
    int group;
    float scale;
    int n_units;
    void* o;                    // [n_units][G][128] normalised, in o_dtype
    int o_dtype;                // SCOUT_F32 / SCOUT_BF16
    float* ml;                  // [n_units][G][2] (max logit, denominator); empty = (-inf, 0)
    int threads;                // 0: all hardware threads
};

int scout_cpu_coattn_run(const CpuCoattnArgs& a);
