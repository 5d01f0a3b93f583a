// local microbench + bit-compare harness for scout_cpu_coattn_run
// CPU co-attention worker harness (host only): 16 cases (q dtype x o dtype x
// Poisson blocks per unit) over a bf16 / f32 host tier; times each call and
// writes the outputs for a bit-for-bit A/B of two builds.
// Env: HB host images (8192), KVDT 1 bf16 / 0 f32, REPS timed calls (20).
// Args: [output file] [threads]
#include "cpu_coattn.h"
extern "C" const char* scout_last_error(void);
#include <chrono>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <random>
#include <vector>
#include <cstdint>
int bench_main(int argc, char** argv) {
    const char* out = argc > 1 ? argv[1] : nullptr;
    int T = argc > 2 ? atoi(argv[2]) : 1;
    const int G = 8, D = 128, K = 64; const int HB = getenv("HB") ? atoi(getenv("HB")) : 8192;
    const size_t sb = (getenv("KVDT") && atoi(getenv("KVDT")) == 0) ? 65536 : 32768;
    std::vector<uint16_t> host(HB * sb / 2);
    std::mt19937 rng(7);
    std::normal_distribution<float> nd;
    auto bf = [](float f) { uint32_t u; memcpy(&u, &f, 4); return (uint16_t)((u + 0x7fff + ((u >> 16) & 1)) >> 16); };
    for (auto& h : host) h = bf(nd(rng));
    FILE* fo = out ? fopen(out, "wb") : nullptr;
    double lam[] = {0.0, 0.8, 3.4, 8.0};
    for (int dt = 0; dt < 4; ++dt) {
        const int qd = (dt & 1) ? 1 : 0, od = (dt & 2) ? 1 : 0;  // 1 = bf16
        for (double L : lam) {
            const int U = 1024;
            std::poisson_distribution<int> pd(L > 0 ? L : 1e-9);
            std::vector<int32_t> nb(U), rows(U * K);
            std::vector<int64_t> idx(U * K);
            for (int u = 0; u < U; ++u) {
                nb[u] = L > 0 ? std::min(K, pd(rng)) : 0;
                for (int i = 0; i < K; ++i) { idx[u * K + i] = rng() % HB; rows[u * K + i] = (i == 0 && u % 7 == 0) ? 33 : 64; }
            }
            std::vector<float> qf(U * G * D);
            std::vector<uint16_t> qb(U * G * D);
            for (size_t i = 0; i < qf.size(); ++i) { qf[i] = nd(rng); qb[i] = bf(qf[i]); }
            std::vector<float> of(U * G * D), ml(U * G * 2);
            std::vector<uint16_t> ob(U * G * D);
            CpuCoattnArgs a{};
            a.host_tier = host.data(); a.kv_dtype = 1 /*placeholder*/;
            a.host_index = idx.data(); a.block_rows = rows.data(); a.n_blocks = nb.data(); a.k_stride = K;
            a.q = qd ? (const void*)qb.data() : (const void*)qf.data(); a.group = G; a.scale = 0.0883883f; a.n_units = U;
            a.o = od ? (void*)ob.data() : (void*)of.data(); a.ml = ml.data(); a.threads = T;
            a.kv_dtype = atoi(getenv("KVDT") ? getenv("KVDT") : "1");
            a.q_dtype = qd ? 1 : 0; a.o_dtype = od ? 1 : 0;
            int rc = scout_cpu_coattn_run(a);
            if (rc) { printf("rc %d %s\n", rc, scout_last_error()); return 1; }
            auto t0 = std::chrono::steady_clock::now();
            int reps = getenv("REPS") ? atoi(getenv("REPS")) : 20;
            for (int r = 0; r < reps; ++r) scout_cpu_coattn_run(a);
            double us = std::chrono::duration<double, std::micro>(std::chrono::steady_clock::now() - t0).count() / reps;
            long tb = 0; for (int x : nb) tb += x;
            printf("q%s o%s lambda %.1f: %8.1f us per call (%ld blocks, %.2f us/unit)\n", qd ? "bf16" : "f32", od ? "bf16" : "f32", L, us, tb, us / U);
            if (fo) { fwrite(od ? (void*)ob.data() : (void*)of.data(), 1, od ? ob.size() * 2 : of.size() * 4, fo); fwrite(ml.data(), 4, ml.size(), fo); }
        }
    }
    if (fo) fclose(fo);
return 0;
}
