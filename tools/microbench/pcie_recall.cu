// Host->device recall bandwidth: how fast can a burst of scattered 32 KiB
// block images (bf16 K+V of one 64-token block) move from pinned host memory
// into scattered pool slots?
//   (a) one contiguous cudaMemcpyAsync (the link's ceiling)
//   (b') one cudaMemcpyAsync per scattered 32 KiB copy
//   (the batched-copy driver API measured in round 2a is closed on this GPU
//   pool and was removed from this file)
//   (c) an SM gather kernel over the mapped host pointer (zero-copy loads),
//       various grid sizes and load depths
// nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o pcie_recall pcie_recall.cu
#include <cuda_runtime.h>

#include <algorithm>
#include <cstdint>
#include <cstdio>
#include <numeric>
#include <random>
#include <vector>

#define CK(x)                                                                              \
    do {                                                                                   \
        cudaError_t e = (x);                                                               \
        if (e != cudaSuccess) {                                                            \
            printf("err %s line %d\n", cudaGetErrorString(e), __LINE__);                   \
            return 1;                                                                      \
        }                                                                                  \
    } while (0)

constexpr size_t SB = 32768;

template <int DEPTH>
__global__ void __launch_bounds__(256) gather_host(uint8_t* pool, const uint8_t* host, const long long* src,
                                                   const int* dst, int n) {
    constexpr int NV = SB / 16;
    // one warp per block image at a time: each lane DEPTH x 16 B in flight per round
    const int warps = gridDim.x * (blockDim.x / 32);
    const int w = blockIdx.x * (blockDim.x / 32) + (threadIdx.x >> 5);
    const int lane = threadIdx.x & 31;
    for (int i = w; i < n; i += warps) {
        const int4* s = reinterpret_cast<const int4*>(host + src[i] * SB);
        int4* d = reinterpret_cast<int4*>(pool + static_cast<size_t>(dst[i]) * SB);
        for (int base = lane; base < NV; base += 32 * DEPTH) {
            int4 v[DEPTH];
#pragma unroll
            for (int k = 0; k < DEPTH; ++k) v[k] = __ldcv(s + base + k * 32);
#pragma unroll
            for (int k = 0; k < DEPTH; ++k) d[base + k * 32] = v[k];
        }
    }
}

int main(int argc, char** argv) {
    const int n = argc > 1 ? atoi(argv[1]) : 48000;       // blocks in the burst
    const int host_n = argc > 2 ? atoi(argv[2]) : 65536;  // host images (2 GiB)
    const int pool_n = 200000;                            // pool slots (6.1 GiB)
    uint8_t *host, *pool;
    CK(cudaHostAlloc(&host, host_n * SB, cudaHostAllocMapped));
    memset(host, 1, host_n * SB);
    CK(cudaMalloc(&pool, static_cast<size_t>(pool_n) * SB));
    uint8_t* hdev;
    CK(cudaHostGetDevicePointer((void**)&hdev, host, 0));
    std::mt19937_64 rng(7);
    std::vector<long long> src(n);
    std::vector<int> dst(n);
    for (int i = 0; i < n; ++i) src[i] = rng() % host_n;
    std::vector<int> perm(pool_n);
    std::iota(perm.begin(), perm.end(), 0);
    std::shuffle(perm.begin(), perm.end(), rng);
    for (int i = 0; i < n; ++i) dst[i] = perm[i];
    long long* dsrc;
    int* ddst;
    CK(cudaMalloc(&dsrc, n * 8));
    CK(cudaMalloc(&ddst, n * 4));
    CK(cudaMemcpy(dsrc, src.data(), n * 8, cudaMemcpyHostToDevice));
    CK(cudaMemcpy(ddst, dst.data(), n * 4, cudaMemcpyHostToDevice));
    cudaStream_t st;
    CK(cudaStreamCreateWithFlags(&st, cudaStreamNonBlocking));
    cudaEvent_t a, b;
    cudaEventCreate(&a);
    cudaEventCreate(&b);
    const double gb = static_cast<double>(n) * SB / 1e9;
    auto report = [&](const char* name) {
        float ms;
        cudaEventSynchronize(b);
        cudaEventElapsedTime(&ms, a, b);
        printf("%-58s %7.2f ms  %6.1f GB/s\n", name, ms, gb / (ms / 1e3));
    };
    // (a) contiguous
    for (int r = 0; r < 2; ++r) {
        cudaEventRecord(a, st);
        CK(cudaMemcpyAsync(pool, host, std::min<size_t>(static_cast<size_t>(n), host_n) * SB, cudaMemcpyHostToDevice, st));
        cudaEventRecord(b, st);
    }
    report("(a) one contiguous cudaMemcpyAsync");
    // (b) batch
    std::vector<void*> ds(n), ss(n);
    std::vector<size_t> sz(n, SB);
    for (int i = 0; i < n; ++i) {
        ds[i] = pool + static_cast<size_t>(dst[i]) * SB;
        ss[i] = host + src[i] * SB;
    }
    for (int r = 0; r < 2; ++r) {
        cudaEventRecord(a, st);
        for (int i = 0; i < n; ++i) CK(cudaMemcpyAsync(ds[i], ss[i], SB, cudaMemcpyHostToDevice, st));
        cudaEventRecord(b, st);
    }
    report("(b') per-block cudaMemcpyAsync");
    // (c) SM gather over the mapped pointer
    for (int grid : {8, 16, 32, 64, 148, 296}) {
        for (int r = 0; r < 2; ++r) {
            cudaEventRecord(a, st);
            gather_host<8><<<grid, 256, 0, st>>>(pool, hdev, dsrc, ddst, n);
            cudaEventRecord(b, st);
        }
        CK(cudaGetLastError());
        char nm[96];
        snprintf(nm, sizeof nm, "(c) SM gather, %d CTAs x 8 warps, 8 x 16 B per lane", grid);
        report(nm);
    }
    for (int grid : {32, 148}) {
        for (int r = 0; r < 2; ++r) {
            cudaEventRecord(a, st);
            gather_host<4><<<grid, 256, 0, st>>>(pool, hdev, dsrc, ddst, n);
            cudaEventRecord(b, st);
        }
        char nm[96];
        snprintf(nm, sizeof nm, "(c) SM gather, %d CTAs x 8 warps, 4 x 16 B per lane", grid);
        report(nm);
    }
    CK(cudaDeviceSynchronize());
    return 0;
}
