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
