// Host DRAM read bandwidth on the GPU box's cores: the roofline of the CPU
// co-attention worker, which streams whole 32 KiB block images (bf16 K+V of a
// 64-token block) from the pinned host tier.
//   (a) sequential read of a 2 GiB buffer, T threads
//   (b) random 32 KiB images out of a 2 GiB pool (the worker's access shape)
// g++ -O3 -march=native -fopenmp -o host_bw host_bw.cpp
#include <immintrin.h>
#include <omp.h>

#include <chrono>
#include <cstdint>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <random>
#include <vector>

int main() {
    const size_t bytes = size_t(2) << 30, blk = 32768, nblk = bytes / blk;
    auto* buf = static_cast<uint8_t*>(std::aligned_alloc(4096, bytes));
    std::memset(buf, 1, bytes);
    const int maxT = omp_get_max_threads();
    for (int T = 1; T <= maxT; T *= 2) {
        if (T * 2 > maxT && T != maxT) {}
        for (int pass = 0; pass < 2; ++pass) {
            long long acc = 0;
            const auto t0 = std::chrono::steady_clock::now();
#pragma omp parallel num_threads(T) reduction(+ : acc)
            {
                const int t = omp_get_thread_num();
                const size_t lo = bytes / T * t, hi = bytes / T * (t + 1);
                __m512i a = _mm512_setzero_si512();
                for (size_t i = lo; i < hi; i += 64) a = _mm512_add_epi64(a, _mm512_load_si512(buf + i));
                acc += _mm512_reduce_add_epi64(a);
            }
            const double s = std::chrono::duration<double>(std::chrono::steady_clock::now() - t0).count();
            volatile long long sink = acc;
            (void)sink;
            if (pass) printf("(a) sequential read, %2d threads: %7.1f GB/s\n", T, bytes / s / 1e9);
        }
        const size_t reads = nblk;  // as many images as the pool holds, random order
        std::vector<uint32_t> order(reads);
        std::mt19937 rng(T);
        for (auto& x : order) x = rng() % nblk;
        for (int pass = 0; pass < 2; ++pass) {
            long long acc = 0;
            const auto t0 = std::chrono::steady_clock::now();
#pragma omp parallel for num_threads(T) reduction(+ : acc) schedule(dynamic, 64)
            for (size_t r = 0; r < reads; ++r) {
                const uint8_t* p = buf + size_t(order[r]) * blk;
                __m512i a = _mm512_setzero_si512();
                for (size_t i = 0; i < blk; i += 64) a = _mm512_add_epi64(a, _mm512_load_si512(p + i));
                acc += _mm512_reduce_add_epi64(a);
            }
            const double s = std::chrono::duration<double>(std::chrono::steady_clock::now() - t0).count();
            volatile long long sink = acc;
            (void)sink;
            if (pass) printf("(b) random 32 KiB images, %2d threads: %7.1f GB/s (%.2f M images/s)\n", T,
                             reads * blk / s / 1e9, reads / s / 1e6);
        }
        if (T < maxT && T * 2 > maxT) T = maxT / 2;  // end on maxT
    }
    return 0;
}
