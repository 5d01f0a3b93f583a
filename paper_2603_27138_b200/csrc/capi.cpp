// C-ABI plumbing shared by the kernels: thread-local last error, version,
// slot geometry. (Status convention: include/scout_b200.h.)
#include <cstdarg>
#include <cstdio>
#include <mutex>
#include <unordered_map>

#include <cuda_runtime.h>

#include "../../include/scout_b200.h"

namespace {
thread_local char g_last_error[512] = "";
}

namespace scout_host {
void set_error(int code, const char* fmt, ...) {
    (void)code;
    va_list ap;
    va_start(ap, fmt);
    std::vsnprintf(g_last_error, sizeof g_last_error, fmt, ap);
    va_end(ap);
}

int check_launch(const char* what) {
    const cudaError_t e = cudaGetLastError();
    if (e != cudaSuccess) {
        set_error(SCOUT_ERR_CUDA, "%s: %s", what, cudaGetErrorString(e));
        return SCOUT_ERR_CUDA;
    }
    return SCOUT_OK;
}
void ensure_smem(const void* kernel, size_t bytes) {
    static std::mutex mu;
    static std::unordered_map<const void*, size_t> done;
    std::lock_guard<std::mutex> lk(mu);
    size_t& have = done[kernel];
    if (bytes > have) {
        cudaFuncSetAttribute(kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, static_cast<int>(bytes));
        have = bytes;
    }
}
}  // namespace scout_host

extern "C" const char* scout_last_error(void) { return g_last_error; }
extern "C" int scout_version(void) { return 1; }
extern "C" size_t scout_slot_bytes(int kv_dtype) {
    if (kv_dtype == SCOUT_BF16) return 2u * 64u * 128u * 2u;
    if (kv_dtype == SCOUT_F32) return 2u * 64u * 128u * 4u;
    return 0;
}

// calibrate_intervals (recall.hpp:66-95) over a recall-free profiling trace:
// per layer, the longest run of leading steps whose CPU ratio cpu / budget
// stays at or below beta (equal counts), floor 1. cpu_tokens / budget_tokens
// [layers][steps] in step order (RatioTrace::record's samples, recall.hpp:29-45).
extern "C" int scout_calibrate_intervals(const int64_t* cpu_tokens, const int64_t* budget_tokens, int layers,
                                         int steps, double beta, int32_t* intervals) {
    using scout_host::set_error;
    if (!(beta > 0.0) || !(beta < 1.0)) {
        set_error(SCOUT_ERR_INVALID_ARGUMENT, "calibrate_intervals: beta must be in (0, 1)");
        return SCOUT_ERR_INVALID_ARGUMENT;
    }
    if (layers <= 0 || steps <= 0 || !cpu_tokens || !budget_tokens || !intervals) {
        set_error(SCOUT_ERR_INVALID_ARGUMENT, "calibrate_intervals: no samples");
        return SCOUT_ERR_INVALID_ARGUMENT;
    }
    for (int l = 0; l < layers; ++l)
        for (int t = 0; t < steps; ++t)
            if (budget_tokens[static_cast<size_t>(l) * steps + t] <= 0 || cpu_tokens[static_cast<size_t>(l) * steps + t] < 0) {
                set_error(SCOUT_ERR_INVALID_ARGUMENT, "RatioTrace::record: zero budget (layer %d, step %d)", l, t);
                return SCOUT_ERR_INVALID_ARGUMENT;
            }
    for (int l = 0; l < layers; ++l) {
        int n = 0;
        while (n < steps) {
            const size_t i = static_cast<size_t>(l) * steps + n;
            const double ratio = static_cast<double>(cpu_tokens[i]) / static_cast<double>(budget_tokens[i]);
            if (!(ratio <= beta)) break;
            ++n;
        }
        intervals[l] = n > 1 ? n : 1;
    }
    return SCOUT_OK;
}
