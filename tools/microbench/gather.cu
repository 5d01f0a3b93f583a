// Gather bandwidth of random KV-slot pieces via 1-D bulk copies (TMA engine):
// how chunk size / randomness affects achievable HBM read throughput.
// nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o gather gather.cu
#include <cstdio>
#include <cstdint>
#include <vector>
#include <random>
#include <cuda_runtime.h>
#define CK(x) do { cudaError_t e = (x); if (e != cudaSuccess) { printf("err %s line %d\n", cudaGetErrorString(e), __LINE__); return 1; } } while (0)
__device__ __forceinline__ void mbar_init(uint64_t* bar, int count) { asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" :: "r"((uint32_t)__cvta_generic_to_shared(bar)), "r"(count)); }
__device__ __forceinline__ void mbar_expect_tx(uint64_t* bar, uint32_t bytes) { asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" :: "r"((uint32_t)__cvta_generic_to_shared(bar)), "r"(bytes)); }
__device__ __forceinline__ void mbar_wait(uint64_t* bar, uint32_t parity) {
    uint32_t a = (uint32_t)__cvta_generic_to_shared(bar);
    asm volatile("{\n.reg .pred p;\nW: mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n@!p bra W;\n}\n" :: "r"(a), "r"(parity)); }
__device__ __forceinline__ void bulk_g2s(void* dst, const void* src, uint32_t bytes, uint64_t* bar) {
    asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];"
                 :: "r"((uint32_t)__cvta_generic_to_shared(dst)), "l"(src), "r"(bytes), "r"((uint32_t)__cvta_generic_to_shared(bar)) : "memory"); }
// each CTA processes n items; item i copies PIECES pieces of PB bytes from src + off[i*PIECES+p]
template <int NST, int PIECES, int PB>
__global__ void gather(const uint8_t* src, const long long* off, int n_per_cta, float* out) {
    extern __shared__ __align__(128) uint8_t smem[];
    __shared__ uint64_t full[NST];
    const long long* my = off + (long long)blockIdx.x * n_per_cta * PIECES;
    if (threadIdx.x == 0) { for (int i = 0; i < NST; ++i) mbar_init(&full[i], 1); asm volatile("fence.mbarrier_init.release.cluster;"); }
    __syncthreads();
    float acc = 0;
    auto issue = [&](int i) { int s = i % NST; mbar_expect_tx(&full[s], PIECES * PB);
        for (int p = 0; p < PIECES; ++p) bulk_g2s(smem + s * PIECES * PB + p * PB, src + my[i * PIECES + p], PB, &full[s]); };
    if (threadIdx.x == 0) for (int i = 0; i < NST && i < n_per_cta; ++i) issue(i);
    for (int i = 0; i < n_per_cta; ++i) {
        int s = i % NST;
        mbar_wait(&full[s], (i / NST) & 1);
        acc += ((const float*)(smem + s * PIECES * PB))[threadIdx.x];
        __syncthreads();
        if (threadIdx.x == 0 && i + NST < n_per_cta) issue(i + NST);
    }
    if (acc == 1234.5f) out[0] = acc;
}
template <int NST, int PIECES, int PB>
int run(const uint8_t* src, size_t bytes, int mode, int sms, float* dout, const char* name) {
    // mode 0: random slots; 1: sequential; 2: unit-clustered (each CTA walks
    // units of 512 contiguous slots = 16 MB, taking 64 random slots of each in
    // ascending order: K2's access pattern if a unit's blocks were allocated
    // together)
    const int per = 200;  // items per CTA
    const int grid = sms;
    const int nitems = grid * per;
    std::vector<long long> off((size_t)nitems * PIECES);
    std::mt19937_64 rng(1);
    const long long nslots = bytes / 32768;
    std::vector<long long> unit_slots;
    for (int i = 0; i < nitems; ++i) {
        long long slot;
        if (mode == 2) {
            if (i % 64 == 0) {  // next unit: 64 of its 512 slots, ascending
                const long long base = (long long)(rng() % (nslots / 512)) * 512;
                std::vector<char> pick(512, 0);
                for (int c = 0; c < 64;) { int r = (int)(rng() % 512); if (!pick[r]) { pick[r] = 1; ++c; } }
                unit_slots.clear();
                for (int r = 0; r < 512; ++r) if (pick[r]) unit_slots.push_back(base + r);
            }
            slot = unit_slots[i % 64];
        } else {
            slot = mode == 0 ? (long long)(rng() % nslots) : (long long)i % nslots;
        }
        for (int p = 0; p < PIECES; ++p) off[(size_t)i * PIECES + p] = slot * 32768 + (long long)p * (PIECES == 2 ? 16384 : PB);
    }
    long long* doff; CK(cudaMalloc(&doff, off.size() * 8)); CK(cudaMemcpy(doff, off.data(), off.size() * 8, cudaMemcpyHostToDevice));
    auto k = gather<NST, PIECES, PB>; int smem = NST * PIECES * PB;
    CK(cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, smem));
    cudaEvent_t e0, e1; cudaEventCreate(&e0); cudaEventCreate(&e1);
    k<<<grid, 128, smem>>>(src, doff, per, dout);
    float best = 1e9;
    for (int r = 0; r < 5; ++r) { cudaEventRecord(e0); k<<<grid, 128, smem>>>(src, doff, per, dout); cudaEventRecord(e1); CK(cudaEventSynchronize(e1)); float ms; cudaEventElapsedTime(&ms, e0, e1); best = ms < best ? ms : best; }
    printf("%-34s NST=%2d pieces=%d x %5d B: %.0f GB/s\n", name, NST, PIECES, PB, (double)nitems * PIECES * PB / best / 1e6);
    cudaFree(doff);
    return 0;
}
int main() {
    int sms; cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
    size_t bytes = (size_t)40 << 30;
    uint8_t* src; CK(cudaMalloc(&src, bytes)); CK(cudaMemset(src, 1, bytes));
    float* dout; CK(cudaMalloc(&dout, 64));
    run<13, 2, 8192>(src, bytes, 0, sms, dout, "random slot, K+V halves (2x8KB)");
    run<13, 2, 8192>(src, bytes, 1, sms, dout, "sequential slot, K+V halves");
    run<13, 1, 16384>(src, bytes, 0, sms, dout, "random 16KB contiguous");
    run<6, 1, 32768>(src, bytes, 0, sms, dout, "random 32KB contiguous");
    run<6, 1, 32768>(src, bytes, 2, sms, dout, "unit-clustered 32KB (64 of 512)");
    run<5, 1, 32768>(src, bytes, 0, sms, dout, "random 32KB, 5 stages");
    run<7, 1, 32768>(src, bytes, 0, sms, dout, "random 32KB, 7 stages (224 KB)");
    run<6, 1, 32768>(src, bytes, 1, sms, dout, "sequential 32KB");
    run<26, 1, 8192>(src, bytes, 0, sms, dout, "random 8KB");
    run<13, 4, 4096>(src, bytes, 0, sms, dout, "random 4x4KB");
    run<12, 1, 16384>(src, bytes, 1, sms, dout, "sequential 16KB");
    return 0;
}
