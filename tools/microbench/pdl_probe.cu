// Does a programmatic dependent launch start while its primary still runs?
// A (primary) triggers launch_dependents, then spins on a flag only B (the
// secondary, launched with programmatic stream serialization) sets.
#include <cstdio>
#include <cuda_runtime.h>
__device__ unsigned long long gns() { unsigned long long t; asm volatile("mov.u64 %0, %globaltimer;" : "=l"(t)); return t; }
__global__ void A(volatile unsigned* flag, int* timed_out, int smem_pad) {
    extern __shared__ char s[];
    if (smem_pad) s[threadIdx.x] = 0;
    asm volatile("griddepcontrol.launch_dependents;" ::: "memory");
    if (threadIdx.x == 0) {
        unsigned long long t0 = gns();
        while (*flag == 0) { if (gns() - t0 > 2000000000ull) { atomicExch(timed_out, 1); break; } }
    }
}
__global__ void B(unsigned* flag) { if (blockIdx.x == 0 && threadIdx.x == 0) { __threadfence(); atomicExch(flag, 1u); } }
int main() {
    unsigned* flag; int* to; cudaMalloc(&flag, 4); cudaMalloc(&to, 4);
    cudaStream_t st; cudaStreamCreateWithFlags(&st, cudaStreamNonBlocking);
    int sms; cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
    const int big = 200 * 1024;
    cudaFuncSetAttribute(A, cudaFuncAttributeMaxDynamicSharedMemorySize, big);
    struct Case { const char* name; int grid, smem; cudaStream_t s; } cases[] = {
        {"A 4 CTAs, own stream", 4, 0, st}, {"A sms-20 CTAs x 200KB, own stream", sms - 20, big, st},
        {"A 4 CTAs, legacy stream", 4, 0, 0}};
    for (auto& c : cases) {
        cudaMemset(flag, 0, 4); cudaMemset(to, 0, 4); cudaDeviceSynchronize();
        A<<<c.grid, 128, c.smem, c.s>>>(flag, to, c.smem);
        cudaLaunchConfig_t cfg = {}; cfg.gridDim = dim3(8); cfg.blockDim = dim3(128); cfg.stream = c.s;
        cudaLaunchAttribute at[1]; at[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
        at[0].val.programmaticStreamSerializationAllowed = 1; cfg.attrs = at; cfg.numAttrs = 1;
        cudaError_t e = cudaLaunchKernelEx(&cfg, B, flag);
        cudaError_t e2 = cudaDeviceSynchronize();
        int h = -1; cudaMemcpy(&h, to, 4, cudaMemcpyDeviceToHost);
        printf("%-40s launch %s sync %s -> %s\n", c.name, cudaGetErrorString(e), cudaGetErrorString(e2),
               h ? "A TIMED OUT (B waited for A)" : "B ran beside A");
    }
}
