// Host-side decode-step orchestration in C++ (the GPU side of
// ScoutEngine::decode_step, reference proj/include/scout/engine.hpp:205-314).
//
// A decode step (device path, scout_engine_decode_step):
//   1. K1 for every layer in ONE launch (grid units x layers): K1(0) with the
//      true query (layer 0 is pinned resident, engine.hpp:227-233), K1(i>=1)
//      with the predicted query (engine.hpp:236-251);
//   2. ONE persistent K2 launch that walks all layers (per-layer launch cost
//      and pipeline drain gone);
//   3. side stream: per-layer recall copies (copy engines) gated on the
//      layer's K2 completion counter via cuStreamWaitValue32 (issued after the
//      layer's attention, kv_store.hpp:175-197), each publishing a recall flag
//      the next step's K2 waits on before it streams the layer (visible at
//      (m+1, i), kv_store.hpp:201-218).
// Host-buffer path (scout_engine_decode_step_host): q_pred lands first and
// releases one K1 launch over all layers; K2 starts once K1 is done and polls
// per-chunk input flags for q_true / CPU partials still in flight; the outputs
// (4 layers at a time) and the host worker's CPU-side ids leave as soon as they
// exist. A step's input copies start at the call, so in steady state they run
// under the previous step's K2.
// K1 outputs are double-buffered by step parity; K2 workspaces are per layer.
// Nothing here allocates or synchronises the host inside a step.
#include <cuda.h>
#include <cuda_runtime.h>

#include <algorithm>
#include <chrono>
#include <condition_variable>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <deque>
#include <mutex>
#include <new>
#include <thread>
#include <vector>

#include "../../include/scout_b200.h"
#include "cpu_coattn.h"
#include "k1_batch.h"
#include "k2_step.h"
#include "k4_batch.h"
#include "k5_batch.h"

namespace scout_host {
void set_error(int code, const char* fmt, ...);
}

namespace {

struct Buf {
    void* p = nullptr;
    ~Buf() {
        if (p) cudaFree(p);
    }
    int alloc(size_t n) {
        if (n == 0) n = 16;
        return cudaMalloc(&p, n) == cudaSuccess ? 0 : -1;
    }
};

#define CU(x)                                                                              \
    do {                                                                                   \
        cudaError_t e_ = (x);                                                              \
        if (e_ != cudaSuccess) {                                                           \
            scout_host::set_error(SCOUT_ERR_CUDA, "%s: %s", #x, cudaGetErrorString(e_)); \
            return SCOUT_ERR_CUDA;                                                         \
        }                                                                                  \
    } while (0)

#define CU_RC(x)                        \
    do {                                \
        const int rc_ = (x);            \
        if (rc_ != SCOUT_OK) return rc_; \
    } while (0)

// stream memory operations (driver API, resolved at run time)
using WaitValueFn = CUresult (*)(CUstream, CUdeviceptr, cuuint32_t, unsigned int);
using WriteValueFn = CUresult (*)(CUstream, CUdeviceptr, cuuint32_t, unsigned int);
WaitValueFn g_wait = nullptr;
WriteValueFn g_write = nullptr;

bool load_stream_memops() {
    if (g_wait && g_write) return true;
    cudaDriverEntryPointQueryResult q1, q2;
    void* f1 = nullptr;
    void* f2 = nullptr;
    if (cudaGetDriverEntryPoint("cuStreamWaitValue32", &f1, cudaEnableDefault, &q1) != cudaSuccess ||
        cudaGetDriverEntryPoint("cuStreamWriteValue32", &f2, cudaEnableDefault, &q2) != cudaSuccess || !f1 || !f2)
        return false;
    g_wait = reinterpret_cast<WaitValueFn>(f1);
    g_write = reinterpret_cast<WriteValueFn>(f2);
    return true;
}

int wait_value(cudaStream_t st, const unsigned* addr, unsigned v) {
    if (g_wait(st, reinterpret_cast<CUdeviceptr>(addr), v, CU_STREAM_WAIT_VALUE_GEQ) != CUDA_SUCCESS) {
        scout_host::set_error(SCOUT_ERR_CUDA, "cuStreamWaitValue32 failed");
        return SCOUT_ERR_CUDA;
    }
    return SCOUT_OK;
}
int write_value(cudaStream_t st, unsigned* addr, unsigned v) {
    if (g_write(st, reinterpret_cast<CUdeviceptr>(addr), v, CU_STREAM_WRITE_VALUE_DEFAULT) != CUDA_SUCCESS) {
        scout_host::set_error(SCOUT_ERR_CUDA, "cuStreamWriteValue32 failed");
        return SCOUT_ERR_CUDA;
    }
    return SCOUT_OK;
}

}  // namespace

struct scout_engine {
    scout_engine_config cfg{};
    std::vector<scout_layer_desc> layers;
    int U = 0, G = 0, UG = 0, grid = 0, nch = 0;
    // per-layer K1 outputs, two sets (step parity)
    Buf sel_ids[2], n_sel[2], res_slots[2], res_ids[2], n_res[2], cpu_ids[2], n_cpu[2], res_tok[2], cpu_tok[2];
    // GpuSidePolicy::all_resident: every layer's whole fast tier at attention
    // time, [L][U][nb_stride] (K2 reads these instead of K1's resident share)
    bool all_res = false;
    Buf ar_ids[2], ar_slots[2], ar_n[2];
    int resident_lists(int par, int l0, int n, cudaStream_t s) {
        ResidentListArgs a{};
        a.layers = tier_mode ? static_cast<const scout_tier_layer*>(tier_dev.p) : nullptr;
        if (!tier_mode)
            for (int i = 0; i < n; ++i) a.tables[l0 + i] = layers[l0 + i].block_table;
        a.nbs = cfg.nb_stride;
        a.layer0 = l0;
        a.stride = cfg.nb_stride;
        a.n_tokens = cfg.n_tokens;
        a.ids = I(ar_ids[par]);
        a.slots = I(ar_slots[par]);
        a.n = I(ar_n[par]);
        ++launches;
        return scout_tier_resident_lists(a, U, n, s);
    }
    Buf ws;  // per-layer K2 workspaces
    size_t ws_layer = 0;
    Buf flags;  // k1_flag[L] | k1_ctr[L] | recall_flag[L] | layer_done[L] | in_flag[nch] | rc_ctr[L] |
                // k1_all_ctr | k1_all_flag
    unsigned *k1_flag = nullptr, *k1_ctr = nullptr, *recall_flag = nullptr, *layer_done = nullptr, *in_flag = nullptr,
             *rc_ctr = nullptr, *k1_all_ctr = nullptr, *k1_all_flag = nullptr;
    unsigned token = 0;  // number of steps launched
    std::vector<unsigned> rc_token;  // per layer: token of its last recall (0: none)
    // recall cadence (engine.hpp:35, recall.hpp:97-126): per-layer interval
    // (0: never) and the step of the layer's last trigger (0: prefill)
    std::vector<int> rc_int, last_recall;
    // recall plans (host arrays for the copy engines, device for the SM kernel)
    std::vector<std::vector<int64_t>> rc_src;
    std::vector<std::vector<int32_t>> rc_dst;
    std::vector<Buf> rc_dev;
    // streams / events
    cudaStream_t k1s = nullptr, side = nullptr, h2d = nullptr, d2h = nullptr, rc_list = nullptr;
    cudaEvent_t ev_start = nullptr, ev_k1_end = nullptr, ev_tmp = nullptr;
    cudaEvent_t ev_k2[2] = {nullptr, nullptr};
    bool k2_recorded[2] = {false, false};
    std::vector<cudaEvent_t> ev_k1;     // per layer: K1 done (host path: CPU-side id copies)
    std::vector<cudaEvent_t> chunk_ev;  // host path: input chunk landed
    // host path staging (per step parity): q_true | q_pred | cpu_o | cpu_ml | out_o | out_ml
    Buf stage[2];
    cudaEvent_t stage_free[2] = {nullptr, nullptr};
    bool stage_recorded[2] = {false, false};
    // recall issuer thread: a layer's recall is ~1300 block copies whose
    // descriptors cost the CPU ~0.6 us each; a worker enqueues them on the side
    // stream so the caller's thread goes straight on to the next step
    int device = 0;
    std::thread rc_thread;
    std::mutex rc_mu;
    std::condition_variable rc_cv, rc_idle;
    struct RcJob {
        int layer;
        unsigned token;
        int slot;   // device tier mode: pinned list slot (-1: static recall plan)
        int chunk;  // ... and the post chunk whose lists it waits for
    };
    std::deque<RcJob> rc_jobs;
    // device tier mode recalls on the copy engines: the post-attention kernel's
    // lists (K1's CPU-side ids, K5's slots) come back to pinned slots, and the
    // issuer thread turns them into copy descriptors
    static constexpr int RC_SLOTS = 4;
    uint8_t* rc_pinned = nullptr;  // RC_SLOTS x (ids [L][U][k] | n [L][U] | dst [L][U][k]) int32
    size_t rc_slot_bytes = 0;
    static constexpr int MAX_CH = K2_MAX_LAYERS;  // post chunks (layer-by-layer mode: one per layer)
    cudaEvent_t ev_chunk[RC_SLOTS][MAX_CH] = {};  // post chunk done (post stream)
    cudaEvent_t ev_list[RC_SLOTS][MAX_CH] = {};   // its lists landed (pinned)
    cudaEvent_t ev_post = nullptr, ev_pre = nullptr;
    bool post_recorded = false;
    cudaStream_t post_s = nullptr;
    int rc_slot_jobs[RC_SLOTS] = {};
    bool rc_stop = false, rc_busy = false;
    // SCOUT_RECALL_PROF=1: the issuer thread's CPU time and blocks, printed at destroy
    double rc_prof_ms = 0.0;
    long long rc_prof_blocks = 0, rc_prof_jobs = 0;
    int rc_err = SCOUT_OK;
    char rc_msg[256] = {0};
    // device tier mode (cfg.tier != nullptr)
    bool tier_mode = false;
    std::vector<scout_tier_layer> tier;
    Buf plan_tab;                  // [L][U][nbs] residency planning view (K1's block tables)
    Buf open_slot, sealed_id;      // [L][U] append bookkeeping
    Buf tier_dst;                  // [L][U][k] recall destination slots
    Buf tier_rc_ids, tier_rc_n;    // [L][U][k] / [L][U] the recalled ids (predicted \ residency)
    Buf tier_dev;                  // [L] scout_tier_layer (device copy for the multi-layer launches)
    Buf rc_stats;                  // [2] u64: recalled blocks served by a warm image / copied (K5 counts)
    uint8_t* host_dev = nullptr;   // device view of the pinned host tier
    std::vector<int> pending;      // per layer: ready tick of its in-flight recall ticket, -1 none
    int n_tickets = 0;
    cudaEvent_t ev_side_end = nullptr, ev_kvin = nullptr;
    bool side_recorded = false;
    int tick(int step, int layer) const { return step * cfg.layers + layer; }
    // first host-tier image index of (layer, unit) (cfg.host_units / host_unit0)
    long long host_row(int l, int u) const {
        const long long hu = cfg.host_units > 0 ? cfg.host_units : U;
        return (static_cast<long long>(l) * hu + cfg.host_unit0 + u) * cfg.nb_stride;
    }
    // ---- in-engine CPU co-attention worker (cfg.cpu_worker; the reference's
    // PrecomputeWorker, engine.hpp:88-150): per step, once K1 has selected
    // and its CPU-side ids are on the host, a worker thread computes layer
    // chunk c's partials (q_pred over the host tier images) on the CPU pool,
    // copies them into the step's device staging and publishes in_flag[c];
    // the running K2 merges each chunk's layers as they land.
    bool cw_on = false;
    std::thread cw_thread;
    std::mutex cw_mu;
    std::condition_variable cw_cv, cw_done_cv;
    struct CwJob {
        unsigned token;
        int par;
        const void* h_q_pred;
    };
    std::deque<CwJob> cw_jobs;
    bool cw_stop = false;
    unsigned cw_done = 0;  // token of the last finished job
    int cw_err = SCOUT_OK;
    char cw_msg[256] = {0};
    uint8_t* cw_pinned = nullptr;  // per parity: ids [L][U][k] | n [L][U] | o [L][UG][128] | ml [L][UG][2]
    size_t cw_par_bytes = 0, cw_off_o = 0, cw_off_ml = 0;
    cudaStream_t cw_s = nullptr;
    cudaEvent_t cw_ids_ev[2] = {}, cw_qt_ev[2] = {}, cw_copy_ev[2] = {};
    bool cw_copy_rec[2] = {false, false};  // worker thread only
    std::vector<int64_t> cw_index;         // worker thread only: [L][U][k] host image indices
    double cw_ms = 0.0;                    // CPU time of the worker's partials (summed, reset by stats)
    int cw_steps = 0;

    // K6 in the layer-by-layer mode (cfg.hidden > 0): the predictor's
    // workspace and one layer's q_pred (q dtype)
    Buf qp_ws, qp_buf;
    size_t qp_ws_bytes = 0;
    // K6 CTAs inside decode_layer_x: one per 128-feature tile (each CTA the
    // whole K), at most the SMs K2 of the layer leaves free, so the GEMM runs
    // in one wave beside K2 (its default grid, two CTAs per tile, took two
    // waves there: 9.19-9.40 ms per step against 9.08-9.25, r02g8 sweep).
    // SCOUT_LW_QP_CTAS overrides (0: K6's default grid).
    int qp_ctas() const {
        static const int env = [] {
            const char* s = getenv("SCOUT_LW_QP_CTAS");
            return s ? atoi(s) : -1;
        }();
        if (env >= 0) return env;
        const int tiles = cfg.hq * SCOUT_HEAD_DIM / 128;
        return tiles < LW_FREE_SMS ? tiles : LW_FREE_SMS;
    }
    // layer-by-layer mode (scout_engine_decode_layer): the layer expected next
    // and the step in progress
    int lw_next = 0, lw_step = -1;
    // SCOUT_LW_HOSTPROF=1: host time of decode_layer by section, printed at destroy
    double lw_host[6] = {0, 0, 0, 0, 0, 0};
    long long lw_calls = 0;
    // K2 CTAs of a single-layer launch (cfg.layer_ctas; SCOUT_LW_K2_CTAS
    // overrides): 0 = automatic, the grid less LW_FREE_SMS for K1 of the next
    // layer (measured per 64-layer step: 148 CTAs 13.9 ms, 120 12.3 ms before
    // the victim cache; after it 148 10.9, 120 10.0, 96 9.1-9.4, 80 8.94-8.99,
    // 72 8.97-8.99, 64 9.2: profiles/r02m_lw_ctas.txt)
    static constexpr int LW_FREE_SMS = 68;
    int layer_ctas() const {
        static const int env = [] {
            const char* s = getenv("SCOUT_LW_K2_CTAS");
            return s ? atoi(s) : 0;
        }();
        const int v = env != 0 ? env : cfg.layer_ctas;
        if (v < 0) return 0;
        if (v > 0) return v;
        return grid > 2 * LW_FREE_SMS ? grid - LW_FREE_SMS : 0;
    }

    // instrumentation
    bool timing = false;
    std::vector<cudaEvent_t> tev;
    size_t tev_used = 0;
    long long launches = 0;

    size_t lk(int layer) const { return static_cast<size_t>(layer) * U * cfg.k; }
    size_t lu(int layer) const { return static_cast<size_t>(layer) * U; }
    int32_t* I(const Buf& b) const { return static_cast<int32_t*>(b.p); }

    // SCOUT_K2_PROF diagnostics: [grid][16] cycle sums (producer: total, plan
    // waits, free-stage waits, blocks; consumers, summed over the warps: data
    // waits, Q loads, segment ends, plans + layer ends; combiner: waiting, busy)
    unsigned long long* k2_prof = nullptr;
    void report_k2_prof() {
        std::vector<unsigned long long> h(static_cast<size_t>(grid) * 16);
        if (cudaMemcpy(h.data(), k2_prof, h.size() * 8, cudaMemcpyDeviceToHost) != cudaSuccess) return;
        double s[16] = {0};
        for (int c = 0; c < grid; ++c)
            for (int i = 0; i < 16; ++i) s[i] += static_cast<double>(h[static_cast<size_t>(c) * 16 + i]);
        const double tot = s[0] > 0 ? s[0] : 1.0, nw = 6.0;
        fprintf(stderr,
                "[k2 prof] %d CTAs, %.0f blocks/CTA, %.0f cycles/block | producer: plan wait %.1f%%, stage wait "
                "%.1f%% | consumers: data wait %.1f%%, Q load %.1f%%, segment end %.1f%%, plan+layer end %.1f%% | "
                "combiners (each): waiting %.1f%%, busy %.1f%% | planner: buffer wait %.1f%%, planning %.1f%%\n",
                grid, s[3] / grid, s[0] / (s[3] > 0 ? s[3] : 1), 100 * s[1] / tot, 100 * s[2] / tot,
                100 * s[4] / nw / tot, 100 * s[5] / nw / tot, 100 * s[6] / nw / tot, 100 * s[7] / nw / tot,
                100 * s[8] / 2 / tot, 100 * s[9] / 2 / tot, 100 * s[10] / tot, 100 * s[11] / tot);
    }

    ~scout_engine() {
        if (lw_calls > 0 && getenv("SCOUT_LW_HOSTPROF"))
            fprintf(stderr,
                    "[lw host] %lld calls, us per call: step start %.1f, apply %.1f, K2 launch %.1f, K1 launch %.1f, "
                    "post %.1f, total %.1f\n",
                    lw_calls, lw_host[0] / lw_calls, lw_host[1] / lw_calls, lw_host[2] / lw_calls,
                    lw_host[3] / lw_calls, lw_host[4] / lw_calls, lw_host[5] / lw_calls);
        stop_worker();
        stop_recalls();
        if (cw_pinned) cudaFreeHost(cw_pinned);
        if (cw_s) cudaStreamDestroy(cw_s);
        for (auto* evs : {cw_ids_ev, cw_qt_ev, cw_copy_ev})
            for (int i = 0; i < 2; ++i)
                if (evs[i]) cudaEventDestroy(evs[i]);
        if (k2_prof) cudaFree(k2_prof);
        for (auto& row : ev_chunk)
            for (auto ev : row)
                if (ev) cudaEventDestroy(ev);
        for (auto& row : ev_list)
            for (auto ev : row)
                if (ev) cudaEventDestroy(ev);
        if (ev_post) cudaEventDestroy(ev_post);
        if (ev_pre) cudaEventDestroy(ev_pre);
        if (ev_rcg) cudaEventDestroy(ev_rcg);
        if (post_s) cudaStreamDestroy(post_s);
        if (rc_pinned) cudaFreeHost(rc_pinned);
        for (cudaStream_t s : {k1s, side, h2d, d2h, rc_list})
            if (s) cudaStreamDestroy(s);
        for (cudaEvent_t e : {ev_start, ev_k1_end, ev_tmp, ev_k2[0], ev_k2[1], stage_free[0], stage_free[1], ev_side_end, ev_kvin})
            if (e) cudaEventDestroy(e);
        for (auto e : ev_k1) cudaEventDestroy(e);
        for (auto e : chunk_ev) cudaEventDestroy(e);
        for (auto e : tev) cudaEventDestroy(e);
    }

    // ---------------------------------------------------------------- K1
    size_t qbytes() const { return cfg.q_dtype == SCOUT_BF16 ? 2 : 4; }
    size_t cbytes() const { return cfg.cpu_dtype == SCOUT_BF16 ? 2 : 4; }  // CPU-partial o element bytes
    // layer l's query block of a [L][U*G][128] query array
    const void* qlayer(const void* q, int l) const {
        return static_cast<const uint8_t*>(q) + static_cast<size_t>(l) * UG * SCOUT_HEAD_DIM * qbytes();
    }

    scout_topk_args k1_args(int layer, const void* q, int step, int par) {
        scout_topk_args a{};
        a.n_units = U;
        a.group = G;
        a.digest_dtype = cfg.kv_dtype;
        a.method = SCOUT_DIGEST_MINMAX;
        a.k = cfg.k;
        a.k_stride = cfg.k;
        a.nb_stride = cfg.nb_stride;
        a.step = step;
        a.q = q;
        a.digests = layers[layer].digests;
        a.n_tokens = cfg.n_tokens;
        a.block_table = tier_mode ? I(plan_tab) + static_cast<size_t>(layer) * U * cfg.nb_stride : layers[layer].block_table;
        if (tier_mode) a.last_selected = tier[layer].last_sel;  // mark_selected (kv_store.hpp:222-228)
        a.sel_ids = I(sel_ids[par]) + lk(layer);
        a.n_sel = I(n_sel[par]) + lu(layer);
        a.res_slots = I(res_slots[par]) + lk(layer);
        a.res_ids = I(res_ids[par]) + lk(layer);
        a.n_res = I(n_res[par]) + lu(layer);
        a.cpu_ids = I(cpu_ids[par]) + lk(layer);
        a.n_cpu = I(n_cpu[par]) + lu(layer);
        a.res_tokens = I(res_tok[par]) + lu(layer);
        a.cpu_tokens = I(cpu_tok[par]) + lu(layer);
        a.done_flag = k1_flag + layer;
        a.done_ctr = k1_ctr + layer;
        a.done_token = token;
        a.q_dtype = cfg.q_dtype;
        return a;
    }
    // K1 over layers [l0, l0+n) in one launch (grid units x layers): layer 0
    // selects with the true query, the others with the predicted one
    int select_batch(int l0, int n, const void* q_true, const void* q_pred, int step, int par, cudaStream_t st) {
        std::vector<scout_topk_args> v(n);
        for (int i = 0; i < n; ++i) {
            const int l = l0 + i;
            v[i] = k1_args(l, l == 0 ? q_true : qlayer(q_pred, l), step, par);
        }
        ++launches;
        return scout_k1_launch_batch(v.data(), n, st);
    }

    // ---------------------------------------------------------------- K2
    // K2 over layers [l0, l0 + n) in one persistent launch (the per-layer
    // arrays q .. inflag are indexed from l0): the whole step (0, L), or one
    // layer in the layer-by-layer mode
    int launch_k2(int par, const void* const* q, const void* const* co, const float* const* cml, float* const* o,
                  float* const* ml, const unsigned* const* inflag, bool poll_k1, cudaStream_t st, int l0 = 0,
                  int n = -1, int ctas = 0, bool records = true) {
        if (n < 0) n = cfg.layers;
        K2StepArgs a{};
        a.n_units = U;
        a.group = G;
        a.k_stride = all_res ? cfg.nb_stride : cfg.k;
        a.n_layers = n;
        a.scale = cfg.scale;
        a.kv_pool = cfg.kv_pool;
        a.n_tokens = cfg.n_tokens;
        a.workspace = static_cast<uint8_t*>(ws.p) + static_cast<size_t>(l0) * ws_layer;
        a.ws_layer_bytes = ws_layer;
        a.k1_flag = poll_k1 ? k1_flag + l0 : nullptr;
        a.recall_flag = recall_flag + l0;
        a.layer_done = layer_done + l0;
        a.token = token;
        a.max_ctas = cfg.max_ctas;
        if (ctas > 0 && ctas < grid) {  // a narrower launch (layer-by-layer mode) still counts `grid` per layer
            a.max_ctas = ctas;
            a.done_extra = static_cast<unsigned>(grid - ctas);
        }
        a.q_bf16 = cfg.q_dtype == SCOUT_BF16;
        a.cpu_bf16 = cfg.cpu_dtype == SCOUT_BF16;
        a.prof = k2_prof;
        static const int l2pf = [] {
            const char* e = getenv("SCOUT_K2_L2PF");
            return e ? atoi(e) : 0;
        }();
        a.l2_prefetch = l2pf;
        for (int j = 0; j < n; ++j) {
            const int i = l0 + j;
            const size_t lr = static_cast<size_t>(i) * U * cfg.nb_stride;
            a.layers[j] = all_res ? K2Layer{q[j], I(ar_slots[par]) + lr, I(ar_ids[par]) + lr, I(ar_n[par]) + lu(i),
                                            co[j], cml[j], o[j], ml[j], inflag ? inflag[j] : nullptr, rc_token[i], 0u}
                                  : K2Layer{q[j], I(res_slots[par]) + lk(i), I(res_ids[par]) + lk(i), I(n_res[par]) + lu(i),
                                            co[j], cml[j], o[j], ml[j], inflag ? inflag[j] : nullptr, rc_token[i], 0u};
        }
        if (cfg.recall_mode == 1 && (cfg.recall_interval > 0 || cfg.recall_intervals)) {
            // SM-gather recalls need SMs: a persistent K2 that polls their flags
            // while holding every SM would wait for them forever, so K2 starts
            // only after every recall kernel queued so far (copy-engine recalls,
            // the default, need no SM and overlap K2 freely)
            drain_recalls();
            CU(cudaEventRecord(ev_tmp, side));
            CU(cudaStreamWaitEvent(st, ev_tmp, 0));
        }
        cudaEvent_t e0 = nullptr, e1 = nullptr;
        if (timing) {
            while (tev.size() < tev_used + 2) {
                cudaEvent_t e;
                CU(cudaEventCreate(&e));
                tev.push_back(e);
            }
            e0 = tev[tev_used++];
            e1 = tev[tev_used++];
            CU(cudaEventRecord(e0, st));
        }
        if (cfg.kv_dtype == SCOUT_F32) {
            // f32 KV: one CUDA-core split-K launch per layer (scout_sparse_decode),
            // with the persistent kernel's device-side gates done as stream
            // operations: the layer's recall flag and input chunk before it,
            // the layer_done count the post-attention launches wait for after it
            for (int j = 0; j < n; ++j) {
                const K2Layer& ly = a.layers[j];
                if (ly.recall_token) CU_RC(wait_value(st, recall_flag + l0 + j, ly.recall_token));
                if (ly.in_flag) CU_RC(wait_value(st, ly.in_flag, token));
                scout_decode_args d{};
                d.n_units = U;
                d.group = G;
                d.kv_dtype = SCOUT_F32;
                d.k_stride = a.k_stride;
                d.scale = cfg.scale;
                d.q = ly.q;
                d.kv_pool = cfg.kv_pool;
                d.res_slots = ly.res_slots;
                d.res_ids = ly.res_ids;
                d.n_res = ly.n_res;
                d.n_tokens = cfg.n_tokens;
                d.cpu_o = static_cast<const float*>(ly.cpu_o);
                d.cpu_ml = ly.cpu_ml;
                d.o = ly.o;
                d.ml = ly.ml;
                d.workspace = static_cast<uint8_t*>(a.workspace) + static_cast<size_t>(j) * ws_layer;
                d.workspace_bytes = ws_layer;
                d.max_ctas = cfg.max_ctas;
                d.q_dtype = SCOUT_F32;
                ++launches;
                const int rc = scout_sparse_decode(&d, st);
                if (rc != SCOUT_OK) return rc;
                CU_RC(write_value(st, layer_done + l0 + j, token * static_cast<unsigned>(grid)));
            }
            if (timing) CU(cudaEventRecord(e1, st));
            CU(cudaEventRecord(ev_k2[par], st));
            k2_recorded[par] = true;
            return SCOUT_OK;
        }
        ++launches;
        const int rc = scout_k2_launch(a, st, false);
        if (rc != SCOUT_OK) return rc;
        k2_e1 = e1;
        // records = false: the caller queues K1 right behind this launch as
        // its programmatic dependent (nothing may sit between them in the
        // stream) and records afterwards (k2_records)
        return records ? k2_records(par, st) : SCOUT_OK;
    }
    cudaEvent_t k2_e1 = nullptr;
    bool k1k2_loaded = false;  // K1 and K2 have launched once (their modules are loaded)
    int ov_setting = -1;       // scout_engine_set_overlap: -1 environment / default, 0 off, > 0 K1's SMs
    long long ov_steps = 0;    // overlapped steps since the last scout_engine_overlap_stats reset
    int ov_last_sms = 0;
    // The overlapped step (K1 beside K2, §6.1 of DESIGN.md): how many SMs K1
    // gets this step, 0 = the ordinary order. K2 runs on the rest of the grid,
    // polling K1's per-layer flags; K1 is K2's programmatic dependent (a
    // persistent grid on the SMs K2 leaves, publishing without waiting for
    // it), so K1's digest stream runs under K2's instead of before it.
    // Conditions: bf16 KV, the predicted-top-k policy, no ticket due this
    // step (begin_layer's application follows K1's marks and precedes the
    // layer's post), the full grid, K1's register-resident paths (<= 1024
    // blocks per unit: the 2048-block variant streams too slowly on a third
    // of the SMs), and one ordinary step first (a kernel's first launch loads
    // its module, which would wait for the running K2 that waits for it).
    // SCOUT_K1K2_OVERLAP=<SMs> overrides the default (35% of the grid), 0 disables.
    int overlap_sms(int step) const {
        static const bool serialising = [] {
            // kernel-serialising tools (a profiler / sanitizer injected into the
            // process, or blocking launches) would run K2 to its end before K1
            // starts: K2 would wait for K1's flags until its 10 s trap
            const char* inj = getenv("CUDA_INJECTION64_PATH");
            const char* blk = getenv("CUDA_LAUNCH_BLOCKING");
            return (inj && *inj) || (blk && atoi(blk) != 0);
        }();
        static const int env_sms = [] {
            const char* v = getenv("SCOUT_K1K2_OVERLAP");
            return v ? atoi(v) : -1;
        }();
        const int want = ov_setting >= 0 ? ov_setting : env_sms;  // -1: the default share
        // static view: only without recall plans (their copies follow K2's layers)
        const bool static_recalls = !tier_mode && (cfg.recall_interval > 0 || cfg.recall_intervals);
        if (serialising || !k1k2_loaded || want == 0 || static_recalls || all_res || cfg.kv_dtype != SCOUT_BF16 ||
            cfg.max_ctas > 0 || cfg.nb_stride > 1024 || grid < 100)
            return 0;
        if (tier_mode)
            for (int i = 0; i < cfg.layers; ++i)
                if (pending[i] >= 0 && pending[i] <= tick(step, i)) return 0;
        const int sms = want > 0 ? want : (grid * 35 + 50) / 100;
        return sms < grid ? sms : 0;
    }
    // plan (when due) on st, then on ks: K2 over the grid less `sms`, K1 as its
    // programmatic dependent, the K2 records. ev_pre (after the plan) gates
    // the post launches; done = true publishes k1_all_flag once K1 is complete.
    int overlapped_pair(int step, int par, int sms, const void* q_true, const void* q_pred, const void* const* q,
                        const void* const* co, const float* const* cml, float* const* o, float* const* ml,
                        const unsigned* const* inflag, cudaStream_t st, cudaStream_t ks, bool done) {
        const int L = cfg.layers;
        int rc;
        if (tier_mode && planned_step != step) {
            ++launches;
            if ((rc = scout_tier_plan_layers(static_cast<const scout_tier_layer*>(tier_dev.p), L, U, cfg.nb_stride,
                                             cfg.n_tokens, step, I(plan_tab), st)) != SCOUT_OK)
                return rc;
        }
        // ev_pre (device tier mode) gates the post launches; the static view
        // has no post, only the order of ks after st
        cudaEvent_t pre = tier_mode ? ev_pre : ev_tmp;
        CU(cudaEventRecord(pre, st));
        if (ks != st) CU(cudaStreamWaitEvent(ks, pre, 0));
        if ((rc = launch_k2(par, q, co, cml, o, ml, inflag, true, ks, 0, L, grid - sms, false)) != SCOUT_OK) return rc;
        std::vector<scout_topk_args> v(L);
        for (int i = 0; i < L; ++i) v[i] = k1_args(i, i == 0 ? q_true : qlayer(q_pred, i), step, par);
        ++launches;
        if ((rc = scout_k1_launch_batch_beside(v.data(), L, sms, ks, done ? k1_all_ctr : nullptr,
                                               done ? k1_all_flag : nullptr, token)) != SCOUT_OK)
            return rc;
        ++ov_steps;
        ov_last_sms = sms;
        return k2_records(par, ks);
    }
    int k2_records(int par, cudaStream_t st) {
        if (timing && k2_e1) CU(cudaEventRecord(k2_e1, st));
        k2_e1 = nullptr;
        CU(cudaEventRecord(ev_k2[par], st));
        k2_recorded[par] = true;
        return SCOUT_OK;
    }

    // ---------------------------------------------------------------- K4
    // Is layer i due for a recall at this step? The reference's trigger
    // (maybe_schedule_recall, recall.hpp:114-126): step - last_recall >=
    // interval, which resets the cadence even when nothing moves; or, opt-in,
    // round 1's stagger (step + i) % interval == 0. Call once per (step, layer).
    bool recall_due(int step, int i) {
        const int n = rc_int[i];
        if (n <= 0) return false;
        if (cfg.recall_stagger) return (step + i) % n == 0;
        if (step - last_recall[i] < n) return false;
        last_recall[i] = step;
        return true;
    }
    // A failure of the recall issuer thread (reported by the next call, before
    // anything of that call is launched: the failed layer's flag was still
    // published, so no K2 waits for it forever)
    int issuer_status() {
        std::lock_guard<std::mutex> lk(rc_mu);
        if (rc_err == SCOUT_OK) return SCOUT_OK;
        scout_host::set_error(rc_err, "recall issuer: %s", rc_msg);
        return rc_err;
    }
    // static mode: the due layers' recall plans; the copy waits for every CTA
    // to finish layer i of this launch
    int issue_recalls(int step) {
        bool any = false;
        for (int i = 0; i < cfg.layers; ++i) {
            const scout_layer_desc& L = layers[i];
            if (L.recall_n <= 0 || rc_src[i].empty() || !recall_due(step, i)) continue;
            rc_token[i] = token;  // the next step's K2 waits for it before streaming layer i
            std::lock_guard<std::mutex> lk(rc_mu);
            rc_jobs.push_back(RcJob{i, token, -1, 0});
            any = true;
        }
        if (any) rc_cv.notify_one();
        return SCOUT_OK;
    }
    // one layer's recall on the side stream (issuer thread)
    int run_recall(int i, unsigned tok) {
        const scout_layer_desc& L = layers[i];
        int rc = wait_value(side, layer_done + i, tok * static_cast<unsigned>(grid));
        if (rc != SCOUT_OK) return rc;
        if (cfg.recall_mode == 1) {
            const int64_t* src = static_cast<const int64_t*>(rc_dev[i].p);
            const int32_t* dst = reinterpret_cast<const int32_t*>(src + L.recall_n);
            rc = scout_recall_gather(cfg.kv_pool, cfg.kv_dtype, cfg.host_tier, src, dst, L.recall_n, side);
        } else {
            rc = scout_recall_copy(cfg.kv_pool, cfg.kv_dtype, cfg.host_tier, rc_src[i].data(), rc_dst[i].data(),
                                   L.recall_n, side);
        }
        if (rc != SCOUT_OK) return rc;
        return write_value(side, recall_flag + i, tok);
    }
    void recall_loop() {
        cudaSetDevice(device);
        std::unique_lock<std::mutex> lk(rc_mu);
        for (;;) {
            rc_cv.wait(lk, [&] { return rc_stop || !rc_jobs.empty(); });
            if (rc_jobs.empty()) break;  // stopping and drained
            const auto job = rc_jobs.front();
            rc_jobs.pop_front();
            rc_busy = true;
            lk.unlock();
            const int rc = job.slot < 0 ? run_recall(job.layer, job.token) : run_tier_recall(job);
            if (rc != SCOUT_OK)  // publish the flag anyway: the next K2 must not wait for it forever
                write_value(side, recall_flag + job.layer, job.token);
            lk.lock();
            rc_busy = false;
            if (job.slot >= 0 && --rc_slot_jobs[job.slot] == 0) rc_idle.notify_all();
            if (rc != SCOUT_OK && rc_err == SCOUT_OK) {
                rc_err = rc;
                std::snprintf(rc_msg, sizeof(rc_msg), "%s", scout_last_error());
            }
            if (rc_jobs.empty()) rc_idle.notify_all();
        }
    }
    // device tier mode: one layer's recall from a pinned list slot (issuer thread)
    int run_tier_recall(const RcJob& job) {
        if (cudaEventSynchronize(ev_list[job.slot][job.chunk]) != cudaSuccess) {
            scout_host::set_error(SCOUT_ERR_CUDA, "recall lists: %s", cudaGetErrorString(cudaGetLastError()));
            return SCOUT_ERR_CUDA;
        }
        const int L = cfg.layers, k = cfg.k, i = job.layer;
        const int32_t* ids = reinterpret_cast<const int32_t*>(rc_pinned + job.slot * rc_slot_bytes);
        const int32_t* nn = ids + static_cast<size_t>(L) * U * k;
        const int32_t* dst = nn + static_cast<size_t>(L) * U;
        std::vector<int64_t> src_v;
        std::vector<int32_t> dst_v;
        src_v.reserve(static_cast<size_t>(U) * 8);
        dst_v.reserve(static_cast<size_t>(U) * 8);
        for (int u = 0; u < U; ++u) {
            const int n = nn[static_cast<size_t>(i) * U + u];
            for (int j = 0; j < n; ++j) {
                const size_t o = (static_cast<size_t>(i) * U + u) * k + j;
                if (dst[o] < 0) continue;
                long long hi = host_row(i, u) + ids[o];
                if (cfg.host_blocks > 0) hi %= cfg.host_blocks;
                src_v.push_back(hi);
                dst_v.push_back(dst[o]);
            }
        }
        int rc = SCOUT_OK;
        static const bool prof = getenv("SCOUT_RECALL_PROF") != nullptr;
        const auto t0 = std::chrono::steady_clock::now();
        if (!src_v.empty())
            rc = scout_recall_copy(cfg.kv_pool, cfg.kv_dtype, cfg.host_tier, src_v.data(), dst_v.data(),
                                   static_cast<int>(src_v.size()), side);
        if (prof) {
            rc_prof_ms += std::chrono::duration<double, std::milli>(std::chrono::steady_clock::now() - t0).count();
            rc_prof_blocks += static_cast<long long>(src_v.size());
            ++rc_prof_jobs;
        }
        if (rc != SCOUT_OK) return rc;
        return write_value(side, recall_flag + i, job.token);
    }
    // every queued recall enqueued on the side stream
    void drain_recalls() {
        std::unique_lock<std::mutex> lk(rc_mu);
        rc_idle.wait(lk, [&] { return rc_jobs.empty() && !rc_busy; });
    }
    void stop_recalls() {
        if (!rc_thread.joinable()) return;
        {
            std::lock_guard<std::mutex> lk(rc_mu);
            rc_stop = true;
        }
        rc_cv.notify_all();
        rc_thread.join();
    }

    // ------------------------------------------------------ host staging
    struct Stage {
        uint8_t *qt, *qp, *co;
        float *cm, *o, *oml, *kn, *vn;
    };
    // device staging of one step parity: q_true | q_pred (q dtype) | cpu_o
    // (cpu dtype, sized for f32) | cpu_ml | out_o | out_ml | k_new | v_new
    Stage stage_of(int par) const {
        const size_t qd = static_cast<size_t>(UG) * SCOUT_HEAD_DIM, md = static_cast<size_t>(UG) * 2;
        const size_t L = static_cast<size_t>(cfg.layers), qb = qbytes();
        Stage g{};
        g.qt = static_cast<uint8_t*>(stage[par].p);
        g.qp = g.qt + L * qd * qb;
        g.co = g.qp + L * qd * qb;
        g.cm = reinterpret_cast<float*>(g.co + L * qd * 4);
        g.o = g.cm + L * md;
        g.oml = g.o + L * qd;
        g.kn = g.oml + L * md;
        g.vn = g.kn + L * U * SCOUT_HEAD_DIM;
        return g;
    }

    // ------------------------------------------------------ CPU worker
    int32_t* cw_ids(int par) const { return reinterpret_cast<int32_t*>(cw_pinned + par * cw_par_bytes); }
    int32_t* cw_n(int par) const { return cw_ids(par) + static_cast<size_t>(cfg.layers) * U * cfg.k; }
    uint8_t* cw_o(int par) const { return cw_pinned + par * cw_par_bytes + cw_off_o; }
    float* cw_ml(int par) const { return reinterpret_cast<float*>(cw_pinned + par * cw_par_bytes + cw_off_ml); }
    int worker_status() {
        std::lock_guard<std::mutex> lk(cw_mu);
        if (cw_err == SCOUT_OK) return SCOUT_OK;
        scout_host::set_error(cw_err, "CPU co-attention worker: %s", cw_msg);
        return cw_err;
    }
    void cw_loop() {
        cudaSetDevice(device);
        std::unique_lock<std::mutex> lk(cw_mu);
        for (;;) {
            cw_cv.wait(lk, [&] { return cw_stop || !cw_jobs.empty(); });
            if (cw_jobs.empty()) break;  // stopping and drained
            const CwJob job = cw_jobs.front();
            cw_jobs.pop_front();
            lk.unlock();
            const int rc = cw_run(job);
            lk.lock();
            if (rc != SCOUT_OK && cw_err == SCOUT_OK) {
                cw_err = rc;
                std::snprintf(cw_msg, sizeof(cw_msg), "%s", scout_last_error());
            }
            cw_done = job.token;
            cw_done_cv.notify_all();
        }
    }
    // One step's CPU share, chunk by chunk (engine.hpp:243-251: layer i's task
    // covers cpu[i] = predicted[i] \ residency with q_pred[i]). A failure still
    // publishes the flags (with whatever the partials hold) so no K2 waits
    // forever; the error is reported by the next call.
    int cw_run(const CwJob& job) {
        const int par = job.par, L = cfg.layers, CH = cfg.chunk_layers, k = cfg.k;
        int rc = SCOUT_OK;
        if (cudaEventSynchronize(cw_ids_ev[par]) != cudaSuccess ||
            (cw_copy_rec[par] && cudaEventSynchronize(cw_copy_ev[par]) != cudaSuccess)) {
            scout_host::set_error(SCOUT_ERR_CUDA, "CPU worker: %s", cudaGetErrorString(cudaGetLastError()));
            rc = SCOUT_ERR_CUDA;
        }
        const Stage g = stage_of(par);
        const size_t qd = static_cast<size_t>(UG) * SCOUT_HEAD_DIM, md = static_cast<size_t>(UG) * 2;
        const int32_t* ids = cw_ids(par);
        const int32_t* nn = cw_n(par);
        double ms = 0.0;
        for (int c = 0, lo = 0; lo < L; ++c, lo += CH) {
            const int n = std::min(CH, L - lo);
            if (rc == SCOUT_OK) {
                const auto t0 = std::chrono::steady_clock::now();
                for (int l = lo; l < lo + n; ++l)
                    for (int u = 0; u < U; ++u) {
                        const size_t row = (static_cast<size_t>(l) * U + u) * k;
                        const long long base = host_row(l, u);
                        for (int i = 0; i < nn[static_cast<size_t>(l) * U + u]; ++i) {
                            long long hi = base + ids[row + i];
                            if (cfg.host_blocks > 0) hi %= cfg.host_blocks;
                            cw_index[row + i] = hi;
                        }
                    }
                CpuCoattnArgs a{};
                a.host_tier = cfg.host_tier;
                a.kv_dtype = cfg.kv_dtype;
                a.host_index = cw_index.data() + lk(lo);
                a.n_blocks = nn + lu(lo);
                a.k_stride = k;
                a.q = static_cast<const uint8_t*>(job.h_q_pred) + lo * qd * qbytes();
                a.q_dtype = cfg.q_dtype;
                a.group = G;
                a.scale = cfg.scale;
                a.n_units = n * U;
                a.o = cw_o(par) + lo * qd * cbytes();
                a.o_dtype = cfg.cpu_dtype;
                a.ml = cw_ml(par) + lo * md;
                a.threads = cfg.cpu_threads;
                const auto t1 = std::chrono::steady_clock::now();
                rc = scout_cpu_coattn_run(a);
                const auto t2 = std::chrono::steady_clock::now();
                ms += std::chrono::duration<double, std::milli>(t2 - t0).count();
                static const bool cwprof = getenv("SCOUT_CW_PROF") != nullptr;
                if (cwprof) {
                    long long nbk = 0;
                    for (int i = 0; i < n * U; ++i) nbk += nn[lu(lo) + i];
                    fprintf(stderr, "[cw] step token %u chunk %d: %d units, %lld blocks, index %.3f ms, run %.3f ms\n",
                            job.token, c, n * U, nbk, std::chrono::duration<double, std::milli>(t1 - t0).count(),
                            std::chrono::duration<double, std::milli>(t2 - t1).count());
                }
            }
            if (cudaMemcpyAsync(g.co + lo * qd * cbytes(), cw_o(par) + lo * qd * cbytes(), n * qd * cbytes(),
                                cudaMemcpyHostToDevice, cw_s) != cudaSuccess ||
                cudaMemcpyAsync(g.cm + lo * md, cw_ml(par) + lo * md, n * md * 4, cudaMemcpyHostToDevice, cw_s) !=
                    cudaSuccess) {
                if (rc == SCOUT_OK) {
                    scout_host::set_error(SCOUT_ERR_CUDA, "CPU worker copies: %s", cudaGetErrorString(cudaGetLastError()));
                    rc = SCOUT_ERR_CUDA;
                }
            }
            const int wr = write_value(cw_s, in_flag + c, job.token);
            if (rc == SCOUT_OK) rc = wr;
        }
        if (cudaEventRecord(cw_copy_ev[par], cw_s) == cudaSuccess) cw_copy_rec[par] = true;
        {
            std::lock_guard<std::mutex> l(cw_mu);
            cw_ms += ms;
            ++cw_steps;
        }
        return rc;
    }
    void stop_worker() {
        if (!cw_thread.joinable()) return;
        {
            std::lock_guard<std::mutex> lk(cw_mu);
            cw_stop = true;
        }
        cw_cv.notify_all();
        cw_thread.join();
    }

    // ------------------------------------------------------- device tier mode
    // 1. residency planning view of every layer at this step (residency_set at
    //    (step, i-1) == at step start: the step's later ops touch other layers);
    // 2. select + split + mark_selected for every layer (one launch);
    // 3. begin_layer: tickets due at (step, i), applied after the marks
    //    The planning view is usually written already: the previous step's
    //    post-attention launches compute it for `step` as each layer's
    //    bookkeeping ends (planned_step); a step number out of sequence (or the
    //    first step) plans here.
    int planned_step = -1;
    bool prefilled = false;  // scout_engine_prefill ran (ScoutEngine::prefilled_)
    int tier_pre(int step, int par, const void* q_true, const void* q_pred, cudaStream_t s) {
        const int L = cfg.layers, nbs = cfg.nb_stride;
        int rc;
        if (planned_step != step) {
            ++launches;
            if ((rc = scout_tier_plan_layers(static_cast<const scout_tier_layer*>(tier_dev.p), L, U, nbs, cfg.n_tokens,
                                             step, I(plan_tab), s)) != SCOUT_OK)
                return rc;
        }
        if (ph_ev[0]) cudaEventRecord(ph_ev[0], s);
        if ((rc = select_batch(0, L, q_true, q_pred, step, par, s)) != SCOUT_OK) return rc;
        if (ph_ev[1]) cudaEventRecord(ph_ev[1], s);
        TierApplyArgs ap{};
        ap.layers = static_cast<const scout_tier_layer*>(tier_dev.p);
        ap.nbs = nbs;
        ap.n_tokens = cfg.n_tokens;
        for (int i = 0; i < L; ++i) {
            if (pending[i] < 0 || pending[i] > tick(step, i)) continue;
            ap.layer[ap.n] = i;
            ap.due_tick[ap.n] = tick(step, i);
            ++ap.n;
            pending[i] = -1;
        }
        if (ap.n > 0) {  // every due layer in one launch (independent layer states)
            ++launches;
            if ((rc = scout_tier_apply_layers(ap, U, s)) != SCOUT_OK) return rc;
        }
        // all_resident: the fast tier after begin_layer's tickets
        if (all_res && (rc = resident_lists(par, 0, L, s)) != SCOUT_OK) return rc;
        return SCOUT_OK;
    }
    // 5. as K2 finishes each chunk of layers (layer_done flags), one launch per
    //    chunk on the post stream: append the token (open / seal + LRU
    //    eviction, write-through) and, when due, schedule the recall of the
    //    layer's CPU-side selected blocks (maybe_schedule_recall,
    //    recall.hpp:114-126) -- issued right after the layer's attention, as in
    //    engine.hpp:299-307, so the copies get a whole step before the next
    //    K2 needs them; n_tokens advances once every layer has appended;
    // 6. the recall copies: copy engines (lists back to a pinned slot, the
    //    issuer thread builds the descriptors) or the SM gather (recall_mode 1).
    //    The next step's K2 waits for a layer's flag before streaming it.
    // `pre`: an event recorded on the step's stream after phases 1-3 (before K2).
    static constexpr int POST_CH = 8, POST_TAIL = 2;
    cudaEvent_t ph_ev[2] = {};  // SCOUT_ENGINE_PHASES: after the plan, after K1
    // The post-attention bookkeeping of one step: post_begin sets up the
    // step's arguments and recall list slot, post_chunk handles layers
    // [lo, lo+n) once K2 finished them, post_end advances n_tokens and orders
    // the next step after all of it. recall_due is decided per layer as its
    // chunk is posted (each (step, layer) once).
    TierPostArgs pa_step{};
    int post_slot = 0;
    bool post_ce = false;
    int32_t *post_hid = nullptr, *post_hn = nullptr, *post_hd = nullptr;
    int post_begin(int step, int par, unsigned tok, const float* k_new, const float* v_new) {
        const int L = cfg.layers;
        TierPostArgs& pa = pa_step;
        pa = TierPostArgs{};
        pa.layers = static_cast<const scout_tier_layer*>(tier_dev.p);
        pa.n_layers = L;
        pa.nbs = cfg.nb_stride;
        pa.k = cfg.k;
        pa.step = step;
        pa.ticket_base = n_tickets;
        n_tickets += L;
        pa.n_tokens = cfg.n_tokens;
        pa.pool = static_cast<uint8_t*>(cfg.kv_pool);
        pa.kv_f32 = cfg.kv_dtype == SCOUT_F32;
        pa.k_new = k_new;
        pa.v_new = v_new;
        for (int i = 0; i < L; ++i) pa.digests[i] = const_cast<void*>(layers[i].digests);
        pa.host_tier = host_dev;
        pa.host_blocks = cfg.host_blocks;
        pa.host_units = cfg.host_units > 0 ? cfg.host_units : U;
        pa.host_unit0 = cfg.host_unit0;
        pa.sel_ids = I(sel_ids[par]);
        pa.n_sel = I(n_sel[par]);
        pa.rc_ids = I(tier_rc_ids);
        pa.rc_n = I(tier_rc_n);
        pa.dst = I(tier_dst);
        pa.rc_stats = static_cast<unsigned long long*>(rc_stats.p);
        pa.res_ids = all_res ? nullptr : I(res_ids[par]);  // check_split only for the predicted policy
        pa.n_res = I(n_res[par]);
        pa.cpu_ids = I(cpu_ids[par]);
        pa.n_cpu = I(n_cpu[par]);
        pa.res_tok = I(res_tok[par]);
        pa.cpu_tok = I(cpu_tok[par]);
        pa.plan_out = I(plan_tab);  // the next step's planning view (K1 of this step has read its own)
        pa.plan_step = step + 1;
        post_ce = cfg.recall_mode == 0 && rc_pinned != nullptr;
        post_slot = static_cast<int>(tok % RC_SLOTS);
        if (post_ce) {  // this step's list slot must be free (the issuer thread is done with it)
            std::unique_lock<std::mutex> lk(rc_mu);
            rc_idle.wait(lk, [&] { return rc_slot_jobs[post_slot] == 0; });
        }
        post_hid = post_ce ? reinterpret_cast<int32_t*>(rc_pinned + post_slot * rc_slot_bytes) : nullptr;
        post_hn = post_ce ? post_hid + static_cast<size_t>(L) * U * cfg.k : nullptr;
        post_hd = post_ce ? post_hn + static_cast<size_t>(L) * U : nullptr;
        return SCOUT_OK;
    }
    int post_chunk(int step, unsigned tok, int c, int lo, int n) {
        TierPostArgs& pa = pa_step;
        for (int i = lo; i < lo + n; ++i) pa.recall_due[i] = recall_due(step, i);
        int rc;
        if ((rc = wait_value(post_s, layer_done + lo + n - 1, tok * static_cast<unsigned>(grid))) != SCOUT_OK) return rc;
        pa.layer0 = lo;
        ++launches;
        if ((rc = scout_tier_post_layers(pa, U, n, post_s)) != SCOUT_OK) return rc;
        bool due = false;
        for (int i = lo; i < lo + n; ++i) due |= pa.recall_due[i] != 0;
        if (!due) return SCOUT_OK;
        const int slot = post_slot;
        if (post_ce) {
            // the lists travel on their own stream; `side` carries only the
            // issuer thread's copies and flags (which the next step's K2
            // waits for), so nothing of the next step may queue ahead there
            CU(cudaEventRecord(ev_chunk[slot][c], post_s));
            CU(cudaStreamWaitEvent(rc_list, ev_chunk[slot][c], 0));
            for (int i = lo; i < lo + n; ++i) {
                if (!pa.recall_due[i]) continue;
                CU(cudaMemcpyAsync(post_hid + lk(i), pa.rc_ids + lk(i), static_cast<size_t>(U) * cfg.k * 4,
                                   cudaMemcpyDeviceToHost, rc_list));
                CU(cudaMemcpyAsync(post_hn + lu(i), pa.rc_n + lu(i), static_cast<size_t>(U) * 4, cudaMemcpyDeviceToHost,
                                   rc_list));
                CU(cudaMemcpyAsync(post_hd + lk(i), pa.dst + lk(i), static_cast<size_t>(U) * cfg.k * 4,
                                   cudaMemcpyDeviceToHost, rc_list));
            }
            CU(cudaEventRecord(ev_list[slot][c], rc_list));
            {
                std::lock_guard<std::mutex> lk(rc_mu);
                for (int i = lo; i < lo + n; ++i) {
                    if (!pa.recall_due[i]) continue;
                    rc_jobs.push_back(RcJob{i, tok, slot, c});
                    ++rc_slot_jobs[slot];
                }
            }
            rc_cv.notify_one();
        } else {
            // SM gather: the step's due layers go out in one launch after its
            // last chunk (post_end). Gathers cannot run beside the persistent
            // K2 (it holds every SM) nor ahead of the next K1's grid anyway,
            // and one launch per layer cost ~16 us each after K1 (64 layers:
            // ~0.7 ms on the step after a recall, most of them with nothing
            // to copy once the victim cache serves the recall)
            for (int i = lo; i < lo + n; ++i)
                if (pa.recall_due[i]) rc_gather_layers.push_back(i);
        }
        for (int i = lo; i < lo + n; ++i) {
            if (!pa.recall_due[i]) continue;
            rc_token[i] = tok;  // the next step's K2 waits for it before streaming layer i
            pending[i] = tick(step + 1, i);
        }
        return SCOUT_OK;
    }
    std::vector<int> rc_gather_layers;  // this step's due layers (SM gather), launched by post_end
    cudaEvent_t ev_rcg = nullptr;
    int post_end(int step, cudaStream_t s) {
        int rc;
        if (!rc_gather_layers.empty()) {
            CU(cudaEventRecord(ev_rcg, post_s));  // after every chunk's post launch
            CU(cudaStreamWaitEvent(side, ev_rcg, 0));
            for (size_t b = 0; b < rc_gather_layers.size(); b += K4_MAX_LAYERS) {
                RecallLayersArgs ra{};
                ra.pool = static_cast<uint8_t*>(cfg.kv_pool);
                ra.nb_stride = cfg.nb_stride;
                ra.n_units = U;
                ra.k_stride = cfg.k;
                ra.host_blocks = cfg.host_blocks;
                ra.host_base0 = host_row(0, 0);
                ra.host_layer_stride = host_row(1, 0) - host_row(0, 0);
                ra.ids = pa_step.rc_ids;
                ra.n_ids = pa_step.rc_n;
                ra.dst = pa_step.dst;
                ra.flags = recall_flag;
                ra.ctr = rc_ctr;
                ra.token = token;
                for (size_t j = b; j < rc_gather_layers.size() && ra.n < K4_MAX_LAYERS; ++j)
                    ra.layer[ra.n++] = static_cast<int16_t>(rc_gather_layers[j]);
                ++launches;
                if ((rc = scout_recall_gather_layers(ra, cfg.host_tier, cfg.kv_dtype, 0, side)) != SCOUT_OK) return rc;
            }
            rc_gather_layers.clear();
        }
        ++launches;
        if ((rc = scout_tier_advance(const_cast<int32_t*>(cfg.n_tokens), U, post_s)) != SCOUT_OK) return rc;
        planned_step = step + 1;
        // the next step (planning, K1) follows the bookkeeping
        CU(cudaEventRecord(ev_post, post_s));
        post_recorded = true;
        CU(cudaStreamWaitEvent(s, ev_post, 0));
        return SCOUT_OK;
    }
    // the whole step's bookkeeping in chunks of POST_CH layers as K2 finishes
    // them, the last one only POST_TAIL long: it runs after K2 has ended, on
    // the critical path to the next step
    int tier_post(int step, int par, unsigned tok, const float* k_new, const float* v_new, cudaEvent_t pre,
                  cudaStream_t s) {
        const int L = cfg.layers;
        int rc;
        if ((rc = post_begin(step, par, tok, k_new, v_new)) != SCOUT_OK) return rc;
        CU(cudaStreamWaitEvent(post_s, pre, 0));
        for (int c = 0, lo = 0, n = 0; lo < L; ++c, lo += n) {
            n = L - lo <= POST_TAIL ? L - lo : std::min(POST_CH, L - lo - POST_TAIL);
            if ((rc = post_chunk(step, tok, c, lo, n)) != SCOUT_OK) return rc;
        }
        return post_end(step, s);
    }

    // K1 lists of this parity were read by the K2 two steps back: wait for it;
    // inputs recorded on `st` before the step are visible to the K1 stream
    // Device tier mode: the engine owns every buffer K1 reads, so K1 follows
    // the previous step's bookkeeping (ev_post) instead of everything queued on
    // the caller's stream -- in particular not the previous step's output
    // copies, whose tail would otherwise sit in front of every step.
    int begin_step(cudaStream_t st, int par) {
        if (tier_mode) {
            if (post_recorded) CU(cudaStreamWaitEvent(k1s, ev_post, 0));
        } else {
            CU(cudaEventRecord(ev_start, st));
            CU(cudaStreamWaitEvent(k1s, ev_start, 0));
        }
        if (k2_recorded[par]) CU(cudaStreamWaitEvent(k1s, ev_k2[par], 0));
        return SCOUT_OK;
    }
    int end_step(cudaStream_t st) {
        CU(cudaEventRecord(ev_k1_end, k1s));
        CU(cudaStreamWaitEvent(st, ev_k1_end, 0));
        return SCOUT_OK;
    }
};

extern "C" int scout_engine_create(const scout_engine_config* cfg, const scout_layer_desc* layers,
                                   scout_engine** out) {
    using scout_host::set_error;
    if (!cfg || !layers || !out) {
        set_error(SCOUT_ERR_INVALID_ARGUMENT, "scout_engine_create: null argument");
        return SCOUT_ERR_INVALID_ARGUMENT;
    }
    const scout_engine_config& c = *cfg;
    if (c.layers <= 0 || c.layers > K2_MAX_LAYERS || c.batch <= 0 || c.hkv <= 0 || c.hq % c.hkv != 0 || c.k <= 0 ||
        c.k > SCOUT_MAX_K || c.nb_stride <= 0 || !c.kv_pool || !c.n_tokens || !(c.scale > 0.f) ||
        (c.kv_dtype != SCOUT_BF16 && c.kv_dtype != SCOUT_F32) || (c.q_dtype != SCOUT_F32 && c.q_dtype != SCOUT_BF16) ||
        (c.cpu_dtype != SCOUT_F32 && c.cpu_dtype != SCOUT_BF16) || c.recall_interval < 0) {
        set_error(SCOUT_ERR_INVALID_ARGUMENT, "scout_engine_create: bad config (layers 1..%d, bf16 / f32 KV, k 1..%d)",
                  K2_MAX_LAYERS, SCOUT_MAX_K);
        return SCOUT_ERR_INVALID_ARGUMENT;
    }
    if (c.kv_dtype == SCOUT_F32 && (c.q_dtype != SCOUT_F32 || c.cpu_dtype != SCOUT_F32 || c.hidden > 0)) {
        // the f32 attention path (per-layer CUDA-core split-K) takes f32 queries and partials
        set_error(SCOUT_ERR_INVALID_ARGUMENT, "scout_engine_create: f32 KV needs f32 queries and CPU partials");
        return SCOUT_ERR_INVALID_ARGUMENT;
    }
    if (const int G = c.hq / c.hkv; G != 1 && G != 2 && G != 4 && G != 8) {
        set_error(SCOUT_ERR_INVALID_ARGUMENT, "scout_engine_create: GQA group %d not in {1,2,4,8}", G);
        return SCOUT_ERR_INVALID_ARGUMENT;
    }
    if (c.gpu_side_policy != SCOUT_GPU_SIDE_PREDICTED && c.gpu_side_policy != SCOUT_GPU_SIDE_ALL_RESIDENT) {
        set_error(SCOUT_ERR_INVALID_ARGUMENT, "scout_engine_create: gpu_side_policy %d unknown", c.gpu_side_policy);
        return SCOUT_ERR_INVALID_ARGUMENT;
    }
    if (c.recall_intervals)
        for (int l = 0; l < c.layers; ++l)
            if (c.recall_intervals[l] < 1) {  // engine.hpp:177-178
                set_error(SCOUT_ERR_INVALID_ARGUMENT, "scout_engine_create: recall interval of layer %d must be >= 1", l);
                return SCOUT_ERR_INVALID_ARGUMENT;
            }
    if (c.tier && c.tier[0].capacity > 0) {
        // layer 0 is pinned resident (engine.hpp:181): its begin_layer tickets are
        // applied after the step's selection, which only a pinned layer allows
        set_error(SCOUT_ERR_INVALID_ARGUMENT, "scout_engine_create: device tier mode needs layer 0 pinned (capacity <= 0)");
        return SCOUT_ERR_INVALID_ARGUMENT;
    }
    const bool any_recall = c.recall_interval > 0 || c.recall_intervals != nullptr;
    if (c.cpu_worker && (!c.tier || !c.host_staging || !c.host_tier || c.cpu_threads < 0)) {
        set_error(SCOUT_ERR_INVALID_ARGUMENT,
                  "scout_engine_create: cpu_worker needs device tier mode, host_staging and a host tier");
        return SCOUT_ERR_INVALID_ARGUMENT;
    }
    if (c.host_unit0 < 0 || c.host_units < 0 || (c.host_units > 0 && c.host_unit0 + c.batch * c.hkv > c.host_units)) {
        set_error(SCOUT_ERR_INVALID_ARGUMENT, "scout_engine_create: host_unit0 + U must fit host_units");
        return SCOUT_ERR_INVALID_ARGUMENT;
    }
    if ((any_recall || c.tier) && !c.host_tier) {
        set_error(SCOUT_ERR_INVALID_ARGUMENT, "scout_engine_create: recall needs a host tier");
        return SCOUT_ERR_INVALID_ARGUMENT;
    }
    if (!load_stream_memops()) {
        set_error(SCOUT_ERR_UNSUPPORTED, "scout_engine_create: driver lacks stream memory operations");
        return SCOUT_ERR_UNSUPPORTED;
    }
    auto* e = new (std::nothrow) scout_engine();
    if (!e) {
        set_error(SCOUT_ERR_CUDA, "scout_engine_create: out of host memory");
        return SCOUT_ERR_CUDA;
    }
    e->cfg = c;
    if (e->cfg.chunk_layers <= 0) e->cfg.chunk_layers = 8;
    e->layers.assign(layers, layers + c.layers);
    e->U = c.batch * c.hkv;
    e->G = c.hq / c.hkv;
    e->UG = e->U * e->G;
    e->grid = scout_k2_grid(e->U, c.k, c.max_ctas);
    e->all_res = c.gpu_side_policy == SCOUT_GPU_SIDE_ALL_RESIDENT;
    if (const char* pe = getenv("SCOUT_K2_PROF"); pe && atoi(pe) != 0) {
        // diagnostics: K2 cycle accounting, summed over every launch, printed at destroy
        CU(cudaMalloc(&e->k2_prof, static_cast<size_t>(e->grid) * 16 * sizeof(unsigned long long)));
        CU(cudaMemset(e->k2_prof, 0, static_cast<size_t>(e->grid) * 16 * sizeof(unsigned long long)));
    }
    e->nch = (c.layers + e->cfg.chunk_layers - 1) / e->cfg.chunk_layers;
    const size_t lk = static_cast<size_t>(c.layers) * e->U * c.k * 4, lu = static_cast<size_t>(c.layers) * e->U * 4;
    int bad = 0;
    for (int p = 0; p < 2; ++p)
        bad |= e->sel_ids[p].alloc(lk) | e->res_slots[p].alloc(lk) | e->res_ids[p].alloc(lk) |
               e->cpu_ids[p].alloc(lk) | e->n_sel[p].alloc(lu) | e->n_res[p].alloc(lu) | e->n_cpu[p].alloc(lu) |
               e->res_tok[p].alloc(lu) | e->cpu_tok[p].alloc(lu);
    if (e->all_res) {
        const size_t lr = static_cast<size_t>(c.layers) * e->U * c.nb_stride * 4;
        for (int p = 0; p < 2; ++p) bad |= e->ar_ids[p].alloc(lr) | e->ar_slots[p].alloc(lr) | e->ar_n[p].alloc(lu);
    }
    e->ws_layer = scout_k2_ws_layer_bytes(e->U, e->grid);
    if (c.kv_dtype == SCOUT_F32)  // per-layer launches of the f32 path (scout_sparse_decode)
        e->ws_layer = std::max(e->ws_layer, (scout_sparse_decode_workspace_bytes(e->U, e->G, c.max_ctas) + 255) / 256 * 256);
    bad |= e->ws.alloc(e->ws_layer * c.layers);
    const size_t nflags = 5 * static_cast<size_t>(c.layers) + e->nch + 2;
    bad |= e->flags.alloc(nflags * 4);
    if (!bad && (cudaMemset(e->ws.p, 0, e->ws_layer * c.layers) != cudaSuccess ||
                 cudaMemset(e->flags.p, 0, nflags * 4) != cudaSuccess))
        bad = 1;
    if (!bad && c.host_staging) {
        // q_true | q_pred (q dtype) | cpu_o | cpu_ml | out_o | out_ml (f32)
        const size_t qb = c.q_dtype == SCOUT_BF16 ? 2 : 4;
        size_t per = static_cast<size_t>(c.layers) * e->UG * (2 * SCOUT_HEAD_DIM * qb + (2 * SCOUT_HEAD_DIM + 4) * 4);
        if (c.tier) per += static_cast<size_t>(c.layers) * e->U * SCOUT_HEAD_DIM * 4 * 2;  // k_new | v_new (device tier mode)
        bad |= e->stage[0].alloc(per) | e->stage[1].alloc(per);
    }
    if (bad) {
        delete e;
        set_error(SCOUT_ERR_CUDA, "scout_engine_create: device allocation failed");
        return SCOUT_ERR_CUDA;
    }
    auto* f = static_cast<unsigned*>(e->flags.p);
    e->k1_flag = f;
    e->k1_ctr = f + c.layers;
    e->recall_flag = f + 2 * c.layers;
    e->layer_done = f + 3 * c.layers;
    e->in_flag = f + 4 * c.layers;
    e->rc_ctr = f + 4 * c.layers + e->nch;
    e->k1_all_ctr = e->rc_ctr + c.layers;
    e->k1_all_flag = e->k1_all_ctr + 1;
    e->rc_token.assign(c.layers, 0u);
    e->rc_int.assign(c.layers, 0);
    for (int l = 0; l < c.layers; ++l) e->rc_int[l] = c.recall_intervals ? c.recall_intervals[l] : c.recall_interval;
    e->last_recall.assign(c.layers, 0);
    e->rc_src.resize(c.layers);
    e->rc_dst.resize(c.layers);
    e->rc_dev = std::vector<Buf>(c.layers);
    for (int l = 0; l < c.layers; ++l) {
        const scout_layer_desc& d = layers[l];
        if (d.recall_n <= 0 || !d.recall_src || !d.recall_dst) continue;
        e->rc_src[l].assign(d.recall_src, d.recall_src + d.recall_n);
        e->rc_dst[l].assign(d.recall_dst, d.recall_dst + d.recall_n);
        if (c.recall_mode == 1) {
            const size_t bytes = static_cast<size_t>(d.recall_n) * (8 + 4);
            if (e->rc_dev[l].alloc(bytes) != 0 ||
                cudaMemcpy(e->rc_dev[l].p, d.recall_src, d.recall_n * 8, cudaMemcpyHostToDevice) != cudaSuccess ||
                cudaMemcpy(static_cast<int64_t*>(e->rc_dev[l].p) + d.recall_n, d.recall_dst, d.recall_n * 4,
                           cudaMemcpyHostToDevice) != cudaSuccess) {
                delete e;
                set_error(SCOUT_ERR_CUDA, "scout_engine_create: recall plan upload failed");
                return SCOUT_ERR_CUDA;
            }
        }
    }
    for (cudaStream_t* s : {&e->k1s, &e->side, &e->h2d, &e->d2h, &e->rc_list})
        cudaStreamCreateWithFlags(s, cudaStreamNonBlocking);
    for (cudaEvent_t* ev : {&e->ev_start, &e->ev_k1_end, &e->ev_tmp, &e->ev_k2[0], &e->ev_k2[1], &e->stage_free[0],
                            &e->stage_free[1]})
        cudaEventCreateWithFlags(ev, cudaEventDisableTiming);
    if (c.tier) {
        e->tier_mode = true;
        e->tier.assign(c.tier, c.tier + c.layers);
        const size_t lu = static_cast<size_t>(c.layers) * e->U;
        if (e->plan_tab.alloc(lu * c.nb_stride * 4) || e->open_slot.alloc(lu * 4) || e->sealed_id.alloc(lu * 4) ||
            e->tier_dst.alloc(lu * c.k * 4) || e->tier_rc_ids.alloc(lu * c.k * 4) || e->tier_rc_n.alloc(lu * 4) ||
            e->rc_stats.alloc(16) || cudaMemset(e->rc_stats.p, 0, 16) != cudaSuccess ||
            cudaEventCreateWithFlags(&e->ev_side_end, cudaEventDisableTiming) ||
            cudaEventCreateWithFlags(&e->ev_kvin, cudaEventDisableTiming)) {
            delete e;
            set_error(SCOUT_ERR_CUDA, "scout_engine_create: tier-mode allocation failed");
            return SCOUT_ERR_CUDA;
        }
        e->pending.assign(c.layers, -1);
        if (c.layers > K5_MAX_LAYERS || e->tier_dev.alloc(sizeof(scout_tier_layer) * c.layers) ||
            cudaMemcpy(e->tier_dev.p, c.tier, sizeof(scout_tier_layer) * c.layers, cudaMemcpyHostToDevice) != cudaSuccess) {
            delete e;
            set_error(SCOUT_ERR_CUDA, "scout_engine_create: tier descriptors (layers <= %d)", K5_MAX_LAYERS);
            return SCOUT_ERR_CUDA;
        }
        void* hv = nullptr;
        if (cudaHostGetDevicePointer(&hv, const_cast<void*>(c.host_tier), 0) != cudaSuccess || !hv) {
            delete e;
            set_error(SCOUT_ERR_INVALID_ARGUMENT, "scout_engine_create: host_tier must be pinned, device-mapped memory");
            return SCOUT_ERR_INVALID_ARGUMENT;
        }
        e->host_dev = static_cast<uint8_t*>(hv);
    }
    cudaGetDevice(&e->device);
    if (c.tier && any_recall && c.recall_mode == 0) {
        e->rc_slot_bytes = (static_cast<size_t>(c.layers) * e->U * (2 * c.k + 1) * 4 + 255) / 256 * 256;
        if (cudaHostAlloc(reinterpret_cast<void**>(&e->rc_pinned), e->rc_slot_bytes * scout_engine::RC_SLOTS,
                          cudaHostAllocDefault) != cudaSuccess) {
            e->rc_pinned = nullptr;
            delete e;
            set_error(SCOUT_ERR_CUDA, "scout_engine_create: pinned recall lists");
            return SCOUT_ERR_CUDA;
        }
        for (auto& row : e->ev_list)
            for (auto& ev : row) cudaEventCreateWithFlags(&ev, cudaEventDisableTiming | cudaEventBlockingSync);
    }
    if (c.tier) {
        for (auto& row : e->ev_chunk)
            for (auto& ev : row) cudaEventCreateWithFlags(&ev, cudaEventDisableTiming);
        cudaEventCreateWithFlags(&e->ev_post, cudaEventDisableTiming);
        cudaEventCreateWithFlags(&e->ev_pre, cudaEventDisableTiming);
        cudaEventCreateWithFlags(&e->ev_rcg, cudaEventDisableTiming);
        cudaStreamCreateWithFlags(&e->post_s, cudaStreamNonBlocking);
    }
    if (any_recall) e->rc_thread = std::thread([e] { e->recall_loop(); });
    if (c.cpu_worker) {
        const size_t L = c.layers, U = e->U, UG = e->UG, D = SCOUT_HEAD_DIM;
        auto up = [](size_t x) { return (x + 255) / 256 * 256; };
        e->cw_off_o = up(L * U * c.k * 4 + L * U * 4);
        e->cw_off_ml = e->cw_off_o + up(L * UG * D * e->cbytes());
        e->cw_par_bytes = e->cw_off_ml + up(L * UG * 2 * 4);
        bool ok = cudaHostAlloc(reinterpret_cast<void**>(&e->cw_pinned), 2 * e->cw_par_bytes, cudaHostAllocDefault) ==
                  cudaSuccess;
        if (!ok) e->cw_pinned = nullptr;
        ok = ok && cudaStreamCreateWithFlags(&e->cw_s, cudaStreamNonBlocking) == cudaSuccess;
        for (int i = 0; i < 2 && ok; ++i)
            ok = cudaEventCreateWithFlags(&e->cw_ids_ev[i], cudaEventDisableTiming | cudaEventBlockingSync) ==
                     cudaSuccess &&
                 cudaEventCreateWithFlags(&e->cw_qt_ev[i], cudaEventDisableTiming) == cudaSuccess &&
                 cudaEventCreateWithFlags(&e->cw_copy_ev[i], cudaEventDisableTiming | cudaEventBlockingSync) ==
                     cudaSuccess;
        if (!ok) {
            delete e;
            set_error(SCOUT_ERR_CUDA, "scout_engine_create: CPU worker buffers");
            return SCOUT_ERR_CUDA;
        }
        e->cw_index.assign(L * U * c.k, 0);
        e->cw_on = true;
        e->cw_thread = std::thread([e] { e->cw_loop(); });
    }
    if (c.hidden > 0) {  // K6 inside the layer-by-layer mode
        const int n_out = c.hq * SCOUT_HEAD_DIM;
        if (c.hidden % 128 != 0 || c.batch > 256 || !c.tier) {
            delete e;
            set_error(SCOUT_ERR_INVALID_ARGUMENT,
                      "scout_engine_create: hidden %% 128, batch <= 256 and device tier mode for the q prediction");
            return SCOUT_ERR_INVALID_ARGUMENT;
        }
        e->qp_ws_bytes = std::max(scout_qpred_workspace_bytes(c.hidden, n_out, c.batch, 0),
                                  scout_qpred_workspace_bytes(c.hidden, n_out, c.batch, e->qp_ctas()));
        const size_t qb = c.q_dtype == SCOUT_BF16 ? 2 : 4;
        if (e->qp_ws.alloc(e->qp_ws_bytes) || cudaMemset(e->qp_ws.p, 0, e->qp_ws_bytes) != cudaSuccess ||
            e->qp_buf.alloc(static_cast<size_t>(c.batch) * n_out * qb)) {
            delete e;
            set_error(SCOUT_ERR_CUDA, "scout_engine_create: q prediction buffers");
            return SCOUT_ERR_CUDA;
        }
    }
    e->ev_k1.resize(c.layers);
    for (auto& ev : e->ev_k1) cudaEventCreateWithFlags(&ev, cudaEventDisableTiming);
    e->chunk_ev.resize(e->nch);
    for (auto& ev : e->chunk_ev) cudaEventCreateWithFlags(&ev, cudaEventDisableTiming);
    const cudaError_t err = cudaGetLastError();
    if (err != cudaSuccess) {
        delete e;
        set_error(SCOUT_ERR_CUDA, "scout_engine_create: %s", cudaGetErrorString(err));
        return SCOUT_ERR_CUDA;
    }
    *out = e;
    return SCOUT_OK;
}

extern "C" int scout_engine_destroy(scout_engine* eng) {
    if (eng) {
        eng->stop_worker();      // finishes the queued CPU partials (their flags) first
        eng->stop_recalls();     // drains the queued recalls first
        cudaDeviceSynchronize();  // flags / copies still reference engine memory
        if (eng->k2_prof) eng->report_k2_prof();
        if (eng->rc_prof_jobs)
            fprintf(stderr, "[recall prof] %lld layer jobs, %lld blocks, issuer %.1f ms (%.2f us per block)\n",
                    eng->rc_prof_jobs, eng->rc_prof_blocks, eng->rc_prof_ms,
                    1000.0 * eng->rc_prof_ms / static_cast<double>(eng->rc_prof_blocks ? eng->rc_prof_blocks : 1));
    }
    delete eng;
    return SCOUT_OK;
}

extern "C" int scout_engine_decode_step(scout_engine* e, int step, const void* q_true, const void* q_pred,
                                        const void* cpu_o, const float* cpu_ml, float* out_o, float* out_ml,
                                        void* stream) {
    if (!e || !q_true || !q_pred || !out_o || !out_ml || ((cpu_o == nullptr) != (cpu_ml == nullptr))) {
        scout_host::set_error(SCOUT_ERR_INVALID_ARGUMENT, "scout_engine_decode_step: null buffer");
        return SCOUT_ERR_INVALID_ARGUMENT;
    }
    if (e->cw_on) {
        scout_host::set_error(SCOUT_ERR_INVALID_ARGUMENT, "cpu_worker engine: use scout_engine_decode_step_kv_host");
        return SCOUT_ERR_INVALID_ARGUMENT;
    }
    auto st = static_cast<cudaStream_t>(stream);
    const size_t qd = static_cast<size_t>(e->UG) * SCOUT_HEAD_DIM, md = static_cast<size_t>(e->UG) * 2;
    const int L = e->cfg.layers;
    if (const int rc = e->issuer_status(); rc != SCOUT_OK) return rc;
    const unsigned token = ++e->token;
    const int par = token & 1;
    int rc;
    std::vector<const void*> q(L);
    std::vector<const void*> co(L);
    std::vector<const float*> cml(L);
    std::vector<float*> o(L), ml(L);
    for (int i = 0; i < L; ++i) {
        q[i] = e->qlayer(q_true, i);
        co[i] = cpu_o ? static_cast<const uint8_t*>(cpu_o) + i * qd * e->cbytes() : nullptr;
        cml[i] = cpu_ml ? cpu_ml + i * md : nullptr;
        o[i] = out_o + i * qd;
        ml[i] = out_ml + i * md;
    }
    // the overlapped step (scout_engine::overlap_sms: no recall plans here) on
    // the engine's own stream, as in the device tier mode
    if (const int ov = e->overlap_sms(step); ov > 0) {
        if ((rc = e->overlapped_pair(step, par, ov, q_true, q_pred, q.data(), co.data(), cml.data(), o.data(),
                                     ml.data(), nullptr, st, e->k1s, false)) != SCOUT_OK)
            return rc;
        CU(cudaStreamWaitEvent(st, e->ev_k2[par], 0));
        return e->issue_recalls(step);
    }
    // K1 for every layer in one wide launch (bandwidth-bound, the whole GPU),
    // then the persistent K2 over all layers; stream order is the dependency
    if ((rc = e->select_batch(0, L, q_true, q_pred, step, par, st)) != SCOUT_OK) return rc;
    if (e->all_res && (rc = e->resident_lists(par, 0, L, st)) != SCOUT_OK) return rc;
    if ((rc = e->launch_k2(par, q.data(), co.data(), cml.data(), o.data(), ml.data(), nullptr, false, st)) != SCOUT_OK)
        return rc;
    e->k1k2_loaded = true;
    return e->issue_recalls(step);
}

static int host_step(scout_engine* e, int step, const void* h_q_true, const void* h_q_pred, const void* h_cpu_o,
                     const float* h_cpu_ml, const float* h_k_new, const float* h_v_new, float* h_out_o, float* h_out_ml,
                     int32_t* h_cpu_ids, int32_t* h_n_cpu, void* stream);

extern "C" int scout_engine_decode_step_host(scout_engine* e, int step, const void* h_q_true, const void* h_q_pred,
                                             const void* h_cpu_o, const float* h_cpu_ml, float* h_out_o,
                                             float* h_out_ml, int32_t* h_cpu_ids, int32_t* h_n_cpu, void* stream) {
    if (e && e->tier_mode) {
        scout_host::set_error(SCOUT_ERR_INVALID_ARGUMENT,
                              "scout_engine_decode_step_host: device tier engine: use scout_engine_decode_step_kv_host");
        return SCOUT_ERR_INVALID_ARGUMENT;
    }
    return host_step(e, step, h_q_true, h_q_pred, h_cpu_o, h_cpu_ml, nullptr, nullptr, h_out_o, h_out_ml, h_cpu_ids,
                     h_n_cpu, stream);
}

extern "C" int scout_engine_decode_step_kv_host(scout_engine* e, int step, const void* h_q_true, const void* h_q_pred,
                                                const void* h_cpu_o, const float* h_cpu_ml, const float* h_k_new,
                                                const float* h_v_new, float* h_out_o, float* h_out_ml,
                                                int32_t* h_cpu_ids, int32_t* h_n_cpu, void* stream) {
    if (!e || !e->tier_mode || !h_k_new || !h_v_new) {
        scout_host::set_error(SCOUT_ERR_INVALID_ARGUMENT,
                              "scout_engine_decode_step_kv_host: needs a device tier engine and the new K/V rows");
        return SCOUT_ERR_INVALID_ARGUMENT;
    }
    return host_step(e, step, h_q_true, h_q_pred, h_cpu_o, h_cpu_ml, h_k_new, h_v_new, h_out_o, h_out_ml, h_cpu_ids,
                     h_n_cpu, stream);
}

static int host_step(scout_engine* e, int step, const void* h_q_true, const void* h_q_pred, const void* h_cpu_o,
                     const float* h_cpu_ml, const float* h_k_new, const float* h_v_new, float* h_out_o, float* h_out_ml,
                     int32_t* h_cpu_ids, int32_t* h_n_cpu, void* stream) {
    if (!e || !e->stage[0].p || !h_q_true || !h_q_pred || !h_out_o || !h_out_ml ||
        ((h_cpu_o == nullptr) != (h_cpu_ml == nullptr))) {
        scout_host::set_error(SCOUT_ERR_INVALID_ARGUMENT,
                              "scout_engine_decode_step_host: null buffer or engine created without host_staging");
        return SCOUT_ERR_INVALID_ARGUMENT;
    }
    if (e->cw_on && h_cpu_o) {
        scout_host::set_error(SCOUT_ERR_INVALID_ARGUMENT,
                              "scout_engine_decode_step_kv_host: the engine computes the CPU partials (cpu_worker): "
                              "pass h_cpu_o = h_cpu_ml = NULL");
        return SCOUT_ERR_INVALID_ARGUMENT;
    }
    if (const int rc = e->issuer_status(); rc != SCOUT_OK) return rc;
    if (e->cw_on)
        if (const int rc = e->worker_status(); rc != SCOUT_OK) return rc;
    auto st = static_cast<cudaStream_t>(stream);
    const int L = e->cfg.layers, CH = e->cfg.chunk_layers, nch = e->nch;
    const size_t qd = static_cast<size_t>(e->UG) * SCOUT_HEAD_DIM, md = static_cast<size_t>(e->UG) * 2;
    const unsigned token = ++e->token;
    const int par = token & 1;
    const size_t qb = e->qbytes();  // query element bytes
    const size_t cb = e->cbytes();
    const scout_engine::Stage g = e->stage_of(par);
    const size_t kvn = static_cast<size_t>(L) * e->U * SCOUT_HEAD_DIM * 4;
    const uint8_t* hq_t = static_cast<const uint8_t*>(h_q_true);
    const uint8_t* hq_p = static_cast<const uint8_t*>(h_q_pred);
    if (e->cw_on) {
        // the worker's pinned buffers and events of this parity belong to the
        // step two back until its job is done
        std::unique_lock<std::mutex> lk(e->cw_mu);
        e->cw_done_cv.wait(lk, [&] { return token < 3 || e->cw_done + 2 >= token; });
    }
    int rc = e->begin_step(st, par);
    if (rc != SCOUT_OK) return rc;
    // ---- inputs, in the order the device needs them: q_true of layer 0 and
    // q_pred (K1's inputs) by chunk first, each chunk releasing a K1 launch on
    // the whole GPU; then q_true / CPU partials by chunk, each publishing a
    // flag the (already running) persistent K2 polls before planning a layer.
    // The sources are host memory, so the copies only wait for this parity's
    // staging to be free (step n-2 fully done): step n's inputs stream in
    // while step n-1's K2 still runs. With the in-engine CPU worker the
    // partials come from the worker, which publishes the chunk flags.
    if (e->stage_recorded[par]) CU(cudaStreamWaitEvent(e->h2d, e->stage_free[par], 0));
    CU(cudaMemcpyAsync(g.qt, hq_t, qd * qb, cudaMemcpyHostToDevice, e->h2d));
    CU(cudaMemcpyAsync(g.qp + qd * qb, hq_p + qd * qb, (L - 1) * qd * qb, cudaMemcpyHostToDevice, e->h2d));
    CU(cudaEventRecord(e->chunk_ev[0], e->h2d));
    for (int c = 0; c < nch; ++c) {
        const int lo = c * CH, n = (c + 1) * CH > L ? L - lo : CH;
        const int lq = c == 0 ? 1 : lo;  // layer 0's q_true went first
        CU(cudaMemcpyAsync(g.qt + lq * qd * qb, hq_t + lq * qd * qb, (lo + n - lq) * qd * qb, cudaMemcpyHostToDevice,
                           e->h2d));
        if (h_cpu_o) {
            CU(cudaMemcpyAsync(g.co + lo * qd * cb, static_cast<const uint8_t*>(h_cpu_o) + lo * qd * cb, n * qd * cb,
                               cudaMemcpyHostToDevice, e->h2d));
            CU(cudaMemcpyAsync(g.cm + lo * md, h_cpu_ml + lo * md, n * md * 4, cudaMemcpyHostToDevice, e->h2d));
        }
        if (!e->cw_on && (rc = write_value(e->h2d, e->in_flag + c, token)) != SCOUT_OK) return rc;
    }
    if (e->cw_on) {  // the worker's flags follow every q_true copy of the step
        CU(cudaEventRecord(e->cw_qt_ev[par], e->h2d));
        CU(cudaStreamWaitEvent(e->cw_s, e->cw_qt_ev[par], 0));
    }
    if (e->tier_mode) {  // the token's K/V, needed after the attention
        CU(cudaMemcpyAsync(g.kn, h_k_new, kvn, cudaMemcpyHostToDevice, e->h2d));
        CU(cudaMemcpyAsync(g.vn, h_v_new, kvn, cudaMemcpyHostToDevice, e->h2d));
        CU(cudaEventRecord(e->ev_kvin, e->h2d));
    }
    // ---- K1 for every layer in one launch once q_pred landed (in steady state
    // it was copied while the previous step's K2 ran); the CPU-side ids then
    // go out to the host worker. Device tier mode: planning view + K1 + ticket
    // application (the previous step's bookkeeping is ordered by ev_start)
    CU(cudaStreamWaitEvent(e->k1s, e->chunk_ev[0], 0));
    const bool have_cpu = h_cpu_o != nullptr || e->cw_on;
    std::vector<const void*> q(L);
    std::vector<const void*> co(L);
    std::vector<const float*> cml(L);
    std::vector<float*> o(L), ml(L);
    std::vector<const unsigned*> inflag(L);
    for (int i = 0; i < L; ++i) {
        q[i] = g.qt + i * qd * qb;
        co[i] = have_cpu ? g.co + i * qd * cb : nullptr;
        cml[i] = have_cpu ? g.cm + i * md : nullptr;
        o[i] = g.o + i * qd;
        ml[i] = g.oml + i * md;
        inflag[i] = e->in_flag + i / CH;
    }
    const size_t id_bytes = static_cast<size_t>(L) * e->U * e->cfg.k * 4, n_bytes = static_cast<size_t>(L) * e->U * 4;
    // the overlapped step (scout_engine::overlap_sms; not with the in-engine
    // worker, which takes K1's CPU-side ids while K2 runs)
    const int ov = e->cw_on ? 0 : e->overlap_sms(step);
    if (ov > 0) {
        if ((rc = e->overlapped_pair(step, par, ov, g.qt, g.qp, q.data(), co.data(), cml.data(), o.data(), ml.data(),
                                     inflag.data(), e->k1s, e->k1s, h_cpu_ids != nullptr)) != SCOUT_OK)
            return rc;
        if (h_cpu_ids) {  // K1's CPU-side ids once every layer published (K2 may still run)
            if ((rc = wait_value(e->d2h, e->k1_all_flag, token)) != SCOUT_OK) return rc;
            CU(cudaMemcpyAsync(h_cpu_ids, e->I(e->cpu_ids[par]), id_bytes, cudaMemcpyDeviceToHost, e->d2h));
            if (h_n_cpu) CU(cudaMemcpyAsync(h_n_cpu, e->I(e->n_cpu[par]), n_bytes, cudaMemcpyDeviceToHost, e->d2h));
        }
        CU(cudaStreamWaitEvent(st, e->ev_k2[par], 0));
    } else {
    // ---- K1 for every layer in one launch once q_pred landed (in steady state
    // it was copied while the previous step's K2 ran); the CPU-side ids then
    // go out to the host worker. Device tier mode: planning view + K1 + ticket
    // application (the previous step's bookkeeping is ordered by ev_start)
    if (e->tier_mode) {
        rc = e->tier_pre(step, par, g.qt, g.qp, e->k1s);
        if (rc == SCOUT_OK && cudaEventRecord(e->ev_pre, e->k1s) != cudaSuccess) rc = SCOUT_ERR_CUDA;
    } else {
        rc = e->select_batch(0, L, g.qt, g.qp, step, par, e->k1s);
        if (rc == SCOUT_OK && e->all_res) rc = e->resident_lists(par, 0, L, e->k1s);
    }
    if (rc != SCOUT_OK) return rc;
    if (h_cpu_ids || e->cw_on) {
        CU(cudaEventRecord(e->ev_k1[0], e->k1s));
        CU(cudaStreamWaitEvent(e->d2h, e->ev_k1[0], 0));
    }
    if (e->cw_on) {  // the worker's input: this step's CPU-side ids, then the job
        CU(cudaMemcpyAsync(e->cw_ids(par), e->I(e->cpu_ids[par]), id_bytes, cudaMemcpyDeviceToHost, e->d2h));
        CU(cudaMemcpyAsync(e->cw_n(par), e->I(e->n_cpu[par]), n_bytes, cudaMemcpyDeviceToHost, e->d2h));
        CU(cudaEventRecord(e->cw_ids_ev[par], e->d2h));
        {
            std::lock_guard<std::mutex> lk(e->cw_mu);
            e->cw_jobs.push_back(scout_engine::CwJob{token, par, h_q_pred});
        }
        e->cw_cv.notify_one();
    }
    if (h_cpu_ids) {
        CU(cudaMemcpyAsync(h_cpu_ids, e->I(e->cpu_ids[par]), id_bytes, cudaMemcpyDeviceToHost, e->d2h));
        if (h_n_cpu) CU(cudaMemcpyAsync(h_n_cpu, e->I(e->n_cpu[par]), n_bytes, cudaMemcpyDeviceToHost, e->d2h));
    }
    CU(cudaEventRecord(e->ev_k1_end, e->k1s));
    CU(cudaStreamWaitEvent(st, e->ev_k1_end, 0));
    // ---- K2: one launch; layer i waits for its input chunk's flag on the device
    if ((rc = e->launch_k2(par, q.data(), co.data(), cml.data(), o.data(), ml.data(), inflag.data(), false, st)) !=
        SCOUT_OK)
        return rc;
    e->k1k2_loaded = true;
    }
    if (e->tier_mode) {
        CU(cudaStreamWaitEvent(e->post_s, e->ev_kvin, 0));  // the token's K/V landed
        if ((rc = e->tier_post(step, par, token, g.kn, g.vn, e->ev_pre, st)) != SCOUT_OK) return rc;
    } else if ((rc = e->issue_recalls(step)) != SCOUT_OK) {
        return rc;
    }
    // ---- outputs: OUT_CH layers at a time, each group leaving once every CTA
    // finished its last layer; the last OUT_CH layers one at a time, so the
    // tail after K2 ends is one layer's copy
    constexpr int OUT_CH = 4;
    for (int lo = 0, n = 0; lo < L; lo += n) {
        n = lo + 2 * OUT_CH <= L ? OUT_CH : 1;
        if ((rc = wait_value(e->d2h, e->layer_done + lo + n - 1, token * static_cast<unsigned>(e->grid))) != SCOUT_OK)
            return rc;
        CU(cudaMemcpyAsync(h_out_o + lo * qd, g.o + lo * qd, n * qd * 4, cudaMemcpyDeviceToHost, e->d2h));
        CU(cudaMemcpyAsync(h_out_ml + lo * md, g.oml + lo * md, n * md * 4, cudaMemcpyDeviceToHost, e->d2h));
    }
    CU(cudaEventRecord(e->ev_tmp, e->d2h));
    CU(cudaStreamWaitEvent(st, e->ev_tmp, 0));
    if ((rc = e->end_step(st)) != SCOUT_OK) return rc;
    CU(cudaEventRecord(e->stage_free[par], st));
    e->stage_recorded[par] = true;
    return SCOUT_OK;
}

extern "C" int scout_engine_decode_step_kv(scout_engine* e, int step, const void* q_true, const void* q_pred,
                                           const void* cpu_o, const float* cpu_ml, const float* k_new,
                                           const float* v_new, float* out_o, float* out_ml, void* stream) {
    using scout_host::set_error;
    if (!e || !e->tier_mode || !q_true || !q_pred || !k_new || !v_new || !out_o || !out_ml ||
        ((cpu_o == nullptr) != (cpu_ml == nullptr))) {
        set_error(SCOUT_ERR_INVALID_ARGUMENT, "scout_engine_decode_step_kv: null buffer or engine without tier state");
        return SCOUT_ERR_INVALID_ARGUMENT;
    }
    if (e->cw_on) {
        set_error(SCOUT_ERR_INVALID_ARGUMENT, "cpu_worker engine: use scout_engine_decode_step_kv_host");
        return SCOUT_ERR_INVALID_ARGUMENT;
    }
    if (const int rc = e->issuer_status(); rc != SCOUT_OK) return rc;
    auto st = static_cast<cudaStream_t>(stream);
    const int L = e->cfg.layers;
    const size_t qd = static_cast<size_t>(e->UG) * SCOUT_HEAD_DIM, md = static_cast<size_t>(e->UG) * 2;
    const unsigned token = ++e->token;
    const int par = token & 1;
    int rc;
    // debug: SCOUT_ENGINE_PHASES=1 prints per-phase device times (synchronises)
    static const bool phases = getenv("SCOUT_ENGINE_PHASES") != nullptr;
    cudaEvent_t pe[4] = {};
    if (phases) {
        for (auto& ev : pe) cudaEventCreate(&ev);
        for (auto& ev : e->ph_ev)
            if (!ev) cudaEventCreate(&ev);
    }
    if (phases) cudaEventRecord(pe[0], st);
    std::vector<const void*> q(L);
    std::vector<const void*> co(L);
    std::vector<const float*> cml(L);
    std::vector<float*> o(L), ml(L);
    for (int i = 0; i < L; ++i) {
        q[i] = e->qlayer(q_true, i);
        co[i] = cpu_o ? static_cast<const uint8_t*>(cpu_o) + i * qd * e->cbytes() : nullptr;
        cml[i] = cpu_ml ? cpu_ml + i * md : nullptr;
        o[i] = out_o + i * qd;
        ml[i] = out_ml + i * md;
    }
    // the overlapped step (scout_engine::overlap_sms) on the engine's own
    // stream: a programmatic launch needs its primary in the same stream, and
    // the caller's stream may carry other work between them
    const int ov = phases ? 0 : e->overlap_sms(step);
    if (ov > 0) {
        if ((rc = e->overlapped_pair(step, par, ov, q_true, q_pred, q.data(), co.data(), cml.data(), o.data(),
                                     ml.data(), nullptr, st, e->k1s, false)) != SCOUT_OK)
            return rc;
        CU(cudaStreamWaitEvent(st, e->ev_k2[par], 0));
    } else {
        // 1-3. planning view, select + split + mark, begin_layer's ticket application
        if ((rc = e->tier_pre(step, par, q_true, q_pred, st)) != SCOUT_OK) return rc;
        CU(cudaEventRecord(e->ev_pre, st));
        if (phases) cudaEventRecord(pe[1], st);
        // 4. attention + merge over all layers (one persistent launch)
        if ((rc = e->launch_k2(par, q.data(), co.data(), cml.data(), o.data(), ml.data(), nullptr, false, st)) !=
            SCOUT_OK)
            return rc;
        e->k1k2_loaded = true;
    }
    if (phases) cudaEventRecord(pe[2], st);
    // 5-6. append + write-through + recall scheduling, then the recall copies
    if ((rc = e->tier_post(step, par, token, k_new, v_new, e->ev_pre, st)) != SCOUT_OK) return rc;
    if (phases) {
        cudaEventRecord(pe[3], st);
        cudaEventSynchronize(pe[3]);
        float t[3], tp = 0.f, tk = 0.f;
        for (int i = 0; i < 3; ++i) cudaEventElapsedTime(&t[i], pe[i], pe[i + 1]);
        cudaEventElapsedTime(&tp, pe[0], e->ph_ev[0]);
        cudaEventElapsedTime(&tk, e->ph_ev[0], e->ph_ev[1]);
        fprintf(stderr, "step %d: plan %.3f K1 %.3f apply %.3f K2 %.3f post tail %.3f ms\n", step, tp, tk,
                t[0] - tp - tk, t[1], t[2]);
        for (auto& ev : pe) cudaEventDestroy(ev);
    }
    return SCOUT_OK;
}

// Layer-by-layer mode (device tier mode): the calls a decoder makes inside its
// layer loop, in the order of ScoutEngine::decode_step's body for layer i
// (engine.hpp:219-307): begin_layer's tickets for layer i; K1 for layer i+1
// with the predicted query (layer 0 also selects itself with the true query,
// :227-233); K2+K3 for layer i over the share K1 chose one call earlier; the
// append + seal/evict + recall scheduling of layer i after its attention.
// Layer i's inputs need only exist when the call is made -- q_true[i] and
// q_pred[i+1] come from layer i-1's output in a real decoder -- and K1(i+1)
// may run beside K2(i), on the engine's K1 stream.
static int decode_layer_impl(scout_engine* e, int step, int layer, const void* q_true, const void* q_pred_next,
                             const float* x_next, const void* wq_next, const void* cpu_o, const float* cpu_ml,
                             const float* k_new, const float* v_new, float* out_o, float* out_ml, void* stream);

extern "C" int scout_engine_decode_layer(scout_engine* e, int step, int layer, const void* q_true,
                                         const void* q_pred_next, const void* cpu_o, const float* cpu_ml,
                                         const float* k_new, const float* v_new, float* out_o, float* out_ml,
                                         void* stream) {
    if (!e || (e->tier_mode && layer >= 0 && layer + 1 < e->cfg.layers && !q_pred_next)) {
        scout_host::set_error(SCOUT_ERR_INVALID_ARGUMENT, "scout_engine_decode_layer: bad arguments (device tier "
                                                          "engine, q_pred of the next layer unless this is the last)");
        return SCOUT_ERR_INVALID_ARGUMENT;
    }
    return decode_layer_impl(e, step, layer, q_true, q_pred_next, nullptr, nullptr, cpu_o, cpu_ml, k_new, v_new, out_o,
                             out_ml, stream);
}

extern "C" int scout_engine_decode_layer_x(scout_engine* e, int step, int layer, const void* q_true,
                                           const float* x_next, const void* wq_next_packed, const void* cpu_o,
                                           const float* cpu_ml, const float* k_new, const float* v_new, float* out_o,
                                           float* out_ml, void* stream) {
    if (!e || e->cfg.hidden <= 0 ||
        (layer >= 0 && layer + 1 < e->cfg.layers && (!x_next || !wq_next_packed))) {
        scout_host::set_error(SCOUT_ERR_INVALID_ARGUMENT,
                              "scout_engine_decode_layer_x: needs cfg.hidden > 0, and x_next / wq_next_packed unless "
                              "this is the last layer");
        return SCOUT_ERR_INVALID_ARGUMENT;
    }
    return decode_layer_impl(e, step, layer, q_true, nullptr, x_next, wq_next_packed, cpu_o, cpu_ml, k_new, v_new,
                             out_o, out_ml, stream);
}

static int decode_layer_impl(scout_engine* e, int step, int layer, const void* q_true, const void* q_pred_next,
                             const float* x_next, const void* wq_next, const void* cpu_o, const float* cpu_ml,
                             const float* k_new, const float* v_new, float* out_o, float* out_ml, void* stream) {
    using scout_host::set_error;
    if (!e || !e->tier_mode || e->cw_on || !q_true || !k_new || !v_new || !out_o || !out_ml ||
        ((cpu_o == nullptr) != (cpu_ml == nullptr)) || layer < 0 || layer >= e->cfg.layers) {
        set_error(SCOUT_ERR_INVALID_ARGUMENT, "scout_engine_decode_layer: bad arguments (device tier engine, "
                                              "q_pred of the next layer unless this is the last)");
        return SCOUT_ERR_INVALID_ARGUMENT;
    }
    if (layer != e->lw_next || (layer > 0 && step != e->lw_step)) {
        set_error(SCOUT_ERR_LOGIC, "scout_engine_decode_layer: expected layer %d of step %d, got layer %d of step %d",
                  e->lw_next, layer > 0 ? e->lw_step : step, layer, step);
        return SCOUT_ERR_LOGIC;
    }
    if (const int rc = e->issuer_status(); rc != SCOUT_OK) return rc;
    auto st = static_cast<cudaStream_t>(stream);
    const int L = e->cfg.layers;
    int rc;
    static const bool hprof = getenv("SCOUT_LW_HOSTPROF") != nullptr;
    using hclock = std::chrono::steady_clock;
    hclock::time_point ht[6];
    if (hprof) ht[0] = hclock::now();
    auto hmark = [&](int i) {
        if (!hprof) return;
        ht[i] = hclock::now();
        e->lw_host[i - 1] += std::chrono::duration<double, std::micro>(ht[i] - ht[i - 1]).count();
    };
    if (layer == 0) {
        e->token += 1;
        e->lw_step = step;
        const int par = e->token & 1;
        // the previous step's bookkeeping, and the K2 that read this parity's lists
        if (e->post_recorded) CU(cudaStreamWaitEvent(e->k1s, e->ev_post, 0));
        if (e->k2_recorded[par]) CU(cudaStreamWaitEvent(e->k1s, e->ev_k2[par], 0));
        if (e->planned_step != step) {
            ++e->launches;
            if ((rc = scout_tier_plan_layers(static_cast<const scout_tier_layer*>(e->tier_dev.p), L, e->U,
                                             e->cfg.nb_stride, e->cfg.n_tokens, step, e->I(e->plan_tab), e->k1s)) !=
                SCOUT_OK)
                return rc;
        }
        if ((rc = e->post_begin(step, par, e->token, k_new, v_new)) != SCOUT_OK) return rc;
    }
    const unsigned token = e->token;
    const int par = token & 1;
    // this call's inputs exist on the caller's stream from here on
    CU(cudaEventRecord(e->ev_tmp, st));
    CU(cudaStreamWaitEvent(e->k1s, e->ev_tmp, 0));
    hmark(1);
    // begin_layer(step, layer): the layer's due tickets, after K1's marks of it (one call back)
    if (e->pending[layer] >= 0 && e->pending[layer] <= e->tick(step, layer)) {
        TierApplyArgs ap{};
        ap.layers = static_cast<const scout_tier_layer*>(e->tier_dev.p);
        ap.nbs = e->cfg.nb_stride;
        ap.n_tokens = e->cfg.n_tokens;
        ap.layer[0] = layer;
        ap.due_tick[0] = e->tick(step, layer);
        ap.n = 1;
        e->pending[layer] = -1;
        ++e->launches;
        if ((rc = scout_tier_apply_layers(ap, e->U, e->k1s)) != SCOUT_OK) return rc;
    }
    // K1: layer 0 selects itself (true query), then layer + 1 (predicted query)
    if (layer == 0) {
        if ((rc = e->select_batch(0, 1, q_true, nullptr, step, par, e->k1s)) != SCOUT_OK) return rc;
        CU(cudaEventRecord(e->ev_k1[0], e->k1s));
    }
    if (e->all_res && (rc = e->resident_lists(par, layer, 1, e->k1s)) != SCOUT_OK) return rc;
    CU(cudaEventRecord(e->ev_pre, e->k1s));  // this layer's tier state is final until its post
    hmark(2);
    // K2 + K3 for this layer, once its lists exist. Queued before K1 of the
    // next layer: K2's persistent CTAs (one per SM, most of its shared memory)
    // take their SMs first, and K1(i+1) runs beside them on the SMs K2 leaves
    // free (cfg.layer_ctas) instead of holding SMs K2 then waits for
    CU(cudaStreamWaitEvent(st, e->ev_k1[layer], 0));
    if (e->all_res) CU(cudaStreamWaitEvent(st, e->ev_pre, 0));  // the layer's fast tier after its tickets
    const void* q[1] = {q_true};
    const void* co[1] = {cpu_o};
    const float* cml[1] = {cpu_ml};
    float* o[1] = {out_o};
    float* ml[1] = {out_ml};
    if ((rc = e->launch_k2(par, q, co, cml, o, ml, nullptr, false, st, layer, 1, e->layer_ctas())) != SCOUT_OK)
        return rc;
    hmark(3);
    if (layer + 1 < L) {
        if (x_next) {  // engine.hpp:237: q_pred of layer + 1 from the model's hidden state (K6, tcgen05)
            const bool bf = e->cfg.q_dtype == SCOUT_BF16;
            ++e->launches;
            if ((rc = scout_predict_query(x_next, e->cfg.batch, e->cfg.hidden, wq_next, e->cfg.hq * SCOUT_HEAD_DIM,
                                          bf ? nullptr : static_cast<float*>(e->qp_buf.p), bf ? e->qp_buf.p : nullptr,
                                          e->qp_ws.p, e->qp_ws_bytes, e->qp_ctas(), e->k1s)) != SCOUT_OK)
                return rc;
            q_pred_next = e->qp_buf.p;
        }
        std::vector<scout_topk_args> v{e->k1_args(layer + 1, q_pred_next, step, par)};
        ++e->launches;
        if ((rc = scout_k1_launch_batch(v.data(), 1, e->k1s)) != SCOUT_OK) return rc;
        CU(cudaEventRecord(e->ev_k1[layer + 1], e->k1s));
    }
    hmark(4);
    // post-attention bookkeeping of this layer (append with this call's K/V row)
    const size_t row = static_cast<size_t>(layer) * e->U * SCOUT_HEAD_DIM;
    e->pa_step.k_new = k_new - row;  // the post kernel indexes [layer][unit][128]
    e->pa_step.v_new = v_new - row;
    CU(cudaStreamWaitEvent(e->post_s, e->ev_pre, 0));
    if ((rc = e->post_chunk(step, token, layer, layer, 1)) != SCOUT_OK) return rc;
    hmark(5);
    if (hprof) {
        e->lw_host[5] += std::chrono::duration<double, std::micro>(ht[5] - ht[0]).count();
        ++e->lw_calls;
    }
    e->lw_next = layer + 1 == L ? 0 : layer + 1;
    if (layer + 1 == L) return e->post_end(step, st);
    return SCOUT_OK;
}

extern "C" int scout_engine_sync(scout_engine* e, void* stream) {
    if (!e) return SCOUT_ERR_INVALID_ARGUMENT;
    auto st = static_cast<cudaStream_t>(stream);
    if (e->cw_on) {  // every queued CPU share computed and its copies enqueued
        std::unique_lock<std::mutex> lk(e->cw_mu);
        e->cw_done_cv.wait(lk, [&] { return e->cw_jobs.empty() && e->cw_done == e->token; });
    }
    e->drain_recalls();
    CU(cudaEventRecord(e->ev_tmp, e->side));
    CU(cudaStreamWaitEvent(st, e->ev_tmp, 0));
    if (e->cw_on) {
        CU(cudaEventRecord(e->ev_tmp, e->cw_s));
        CU(cudaStreamWaitEvent(st, e->ev_tmp, 0));
        if (const int rc = e->worker_status(); rc != SCOUT_OK) return rc;
    }
    return e->issuer_status();
}

extern "C" int scout_engine_tier_changed(scout_engine* e) {
    if (!e) return SCOUT_ERR_INVALID_ARGUMENT;
    e->planned_step = -1;
    return SCOUT_OK;
}

extern "C" int scout_engine_set_timing(scout_engine* e, int enable) {
    if (!e) return SCOUT_ERR_INVALID_ARGUMENT;
    e->timing = enable != 0;
    e->tev_used = 0;
    return SCOUT_OK;
}

extern "C" int scout_engine_k2_times(scout_engine* e, float* ms, int max_n, int* n) {
    if (!e || (max_n > 0 && !ms)) return SCOUT_ERR_INVALID_ARGUMENT;
    int k = 0;
    for (size_t i = 0; i + 1 < e->tev_used; i += 2, ++k) {
        if (k >= max_n) continue;
        CU(cudaEventSynchronize(e->tev[i + 1]));
        CU(cudaEventElapsedTime(ms + k, e->tev[i], e->tev[i + 1]));
    }
    if (n) *n = k;
    return SCOUT_OK;
}

extern "C" int scout_engine_recall_stats(scout_engine* e, long long* warm_blocks, long long* copied_blocks, int reset) {
    if (!e) return SCOUT_ERR_INVALID_ARGUMENT;
    unsigned long long h[2] = {0, 0};
    if (e->rc_stats.p) {
        CU(cudaDeviceSynchronize());
        CU(cudaMemcpy(h, e->rc_stats.p, 16, cudaMemcpyDeviceToHost));
        if (reset) CU(cudaMemset(e->rc_stats.p, 0, 16));
    }
    if (warm_blocks) *warm_blocks = static_cast<long long>(h[0]);
    if (copied_blocks) *copied_blocks = static_cast<long long>(h[1]);
    return SCOUT_OK;
}

// ScoutEngine::prefill + place_after_prefill (engine.hpp:192-201) on the
// engine's device tier state: every layer's fresh state filled from the
// model's rows in one pass (scout_tier_prefill: the state of the token-by-token
// appends, the rows, the digests, the write-through), then for every unpinned
// layer the top-capacity sealed blocks by the layer's last prefill query kept
// fast (K1 over the sealed blocks + scout_tier_place). Not a hot call: it
// allocates scratch and synchronises.
extern "C" int scout_engine_prefill(scout_engine* e, const float* k_rows, const float* v_rows, const int32_t* n_tokens,
                                    int max_tokens, const void* q_place, void* stream) {
    using scout_host::set_error;
    if (!e || !e->tier_mode || !k_rows || !v_rows || !n_tokens || max_tokens <= 0) {
        set_error(SCOUT_ERR_INVALID_ARGUMENT, "scout_engine_prefill: needs a device tier engine, rows and counts");
        return SCOUT_ERR_INVALID_ARGUMENT;
    }
    if (e->prefilled) {  // engine.hpp:194
        set_error(SCOUT_ERR_LOGIC, "scout_engine_prefill: prefill already done");
        return SCOUT_ERR_LOGIC;
    }
    auto st = static_cast<cudaStream_t>(stream);
    const int L = e->cfg.layers, U = e->U, nbs = e->cfg.nb_stride;
    int kmax = 1;
    for (int l = 0; l < L; ++l) kmax = std::max(kmax, e->tier[l].capacity);
    if (kmax > SCOUT_MAX_K) {
        set_error(SCOUT_ERR_INVALID_ARGUMENT, "scout_engine_prefill: capacity %d > %d", kmax, SCOUT_MAX_K);
        return SCOUT_ERR_INVALID_ARGUMENT;
    }
    if (q_place && !e->cfg.host_tier) {
        set_error(SCOUT_ERR_INVALID_ARGUMENT, "scout_engine_prefill: placement fills from the host tier");
        return SCOUT_ERR_INVALID_ARGUMENT;
    }
    Buf blk, sealed, keep, nkeep, fill;
    if (blk.alloc(static_cast<size_t>(U) * nbs * 4) || sealed.alloc(static_cast<size_t>(U) * 4) ||
        keep.alloc(static_cast<size_t>(U) * kmax * 4) || nkeep.alloc(static_cast<size_t>(U) * 4) ||
        fill.alloc(static_cast<size_t>(U) * kmax * 4)) {
        set_error(SCOUT_ERR_CUDA, "scout_engine_prefill: scratch");
        return SCOUT_ERR_CUDA;
    }
    int32_t* ntok = const_cast<int32_t*>(e->cfg.n_tokens);
    CU(cudaMemcpyAsync(ntok, n_tokens, static_cast<size_t>(U) * 4, cudaMemcpyDeviceToDevice, st));
    const size_t layer_rows = static_cast<size_t>(U) * max_tokens * SCOUT_HEAD_DIM;
    int rc;
    for (int l = 0; l < L; ++l) {
        ++e->launches;
        if ((rc = scout_tier_prefill(&e->tier[l], U, nbs, ntok, 0, k_rows + l * layer_rows, v_rows + l * layer_rows,
                                     max_tokens, e->cfg.kv_pool, e->cfg.kv_dtype, const_cast<void*>(e->layers[l].digests),
                                     const_cast<void*>(e->cfg.host_tier), e->host_row(l, 0), e->cfg.host_blocks,
                                     e->I(blk), st)) != SCOUT_OK)
            return rc;
    }
    if (q_place) {
        std::vector<int32_t> h(U);
        CU(cudaMemcpyAsync(h.data(), ntok, static_cast<size_t>(U) * 4, cudaMemcpyDeviceToHost, st));
        CU(cudaStreamSynchronize(st));
        for (auto& t : h) t = t / SCOUT_BLOCK_SIZE * SCOUT_BLOCK_SIZE;  // the sealed blocks (kv_store.hpp:273-276)
        CU(cudaMemcpyAsync(sealed.p, h.data(), static_cast<size_t>(U) * 4, cudaMemcpyHostToDevice, st));
        for (int l = 0; l < L; ++l) {
            const int cap = e->tier[l].capacity;
            if (cap <= 0) continue;  // pinned
            scout_topk_args a{};
            a.n_units = U;
            a.group = e->G;
            a.digest_dtype = e->cfg.kv_dtype;
            a.method = SCOUT_DIGEST_MINMAX;
            a.k = cap;
            a.k_stride = cap;
            a.nb_stride = nbs;
            a.q = e->qlayer(q_place, l);
            a.digests = e->layers[l].digests;
            a.n_tokens = e->I(sealed);
            a.sel_ids = e->I(keep);
            a.n_sel = e->I(nkeep);
            a.q_dtype = e->cfg.q_dtype;
            e->launches += 3;
            if ((rc = scout_score_topk_split(&a, st)) != SCOUT_OK) return rc;
            if ((rc = scout_tier_place(&e->tier[l], U, nbs, ntok, e->I(keep), e->I(nkeep), cap, e->I(fill), st)) !=
                SCOUT_OK)
                return rc;
            // the promoted blocks' images: warm slots (fill <= -2) already hold
            // them, the others come from their written-through host images
            if ((rc = scout_recall_gather_ids(e->cfg.kv_pool, e->cfg.kv_dtype, e->cfg.host_tier, e->host_row(l, 0), nbs,
                                              e->cfg.host_blocks, U, e->I(keep), e->I(nkeep), e->I(fill), cap, 0,
                                              st)) != SCOUT_OK)
                return rc;
        }
    }
    CU(cudaStreamSynchronize(st));
    e->prefilled = true;
    e->planned_step = -1;  // the next step plans from the new state
    std::vector<int32_t> err(U);
    for (int l = 0; l < L; ++l) {
        CU(cudaMemcpy(err.data(), e->tier[l].err, static_cast<size_t>(U) * 4, cudaMemcpyDeviceToHost));
        for (int u = 0; u < U; ++u)
            if (err[u]) {
                set_error(err[u] == SCOUT_ERR_INVALID_ARGUMENT ? SCOUT_ERR_INVALID_ARGUMENT : SCOUT_ERR_LOGIC,
                          "scout_engine_prefill: layer %d unit %d: tier error %d (a layer that was not fresh, or too "
                          "few slots)", l, u, err[u]);
                return err[u] == SCOUT_ERR_INVALID_ARGUMENT ? SCOUT_ERR_INVALID_ARGUMENT : SCOUT_ERR_LOGIC;
            }
    }
    return SCOUT_OK;
}

extern "C" int scout_engine_cpu_tokens(scout_engine* e, int64_t* cpu_tokens, int64_t* budget_tokens) {
    if (!e || !cpu_tokens || e->token == 0) {
        scout_host::set_error(SCOUT_ERR_INVALID_ARGUMENT, "scout_engine_cpu_tokens: no step yet");
        return SCOUT_ERR_INVALID_ARGUMENT;
    }
    const int L = e->cfg.layers, par = e->token & 1;
    std::vector<int32_t> h(static_cast<size_t>(L) * e->U);
    CU(cudaDeviceSynchronize());
    CU(cudaMemcpy(h.data(), e->I(e->cpu_tok[par]), h.size() * 4, cudaMemcpyDeviceToHost));
    for (int l = 0; l < L; ++l) {
        int64_t t = 0;
        for (int u = 0; u < e->U; ++u) t += h[static_cast<size_t>(l) * e->U + u];
        cpu_tokens[l] = t;
        if (budget_tokens) budget_tokens[l] = static_cast<int64_t>(e->U) * e->cfg.k * SCOUT_BLOCK_SIZE;
    }
    return SCOUT_OK;
}

extern "C" int scout_engine_stats(scout_engine* e, double* k2_ms_total, int* k2_count, long long* launches) {
    if (!e) return SCOUT_ERR_INVALID_ARGUMENT;
    double tot = 0.0;
    for (size_t i = 0; i + 1 < e->tev_used; i += 2) {
        CU(cudaEventSynchronize(e->tev[i + 1]));
        float ms = 0.f;
        CU(cudaEventElapsedTime(&ms, e->tev[i], e->tev[i + 1]));
        tot += ms;
    }
    if (k2_ms_total) *k2_ms_total = tot;
    if (k2_count) *k2_count = static_cast<int>(e->tev_used / 2);
    if (launches) *launches = e->launches;
    e->tev_used = 0;
    e->launches = 0;
    return SCOUT_OK;
}

extern "C" int scout_engine_set_overlap(scout_engine* e, int k1_sms) {
    if (!e || k1_sms < -1) return SCOUT_ERR_INVALID_ARGUMENT;
    e->ov_setting = k1_sms;
    return SCOUT_OK;
}

extern "C" int scout_engine_overlap_stats(scout_engine* e, long long* steps, int* k1_sms, int reset) {
    if (!e) return SCOUT_ERR_INVALID_ARGUMENT;
    if (steps) *steps = e->ov_steps;
    if (k1_sms) *k1_sms = e->ov_last_sms;
    if (reset) e->ov_steps = 0;
    return SCOUT_OK;
}

extern "C" int scout_engine_check_state(scout_engine* e) {
    if (!e) return SCOUT_ERR_INVALID_ARGUMENT;
    if (!e->tier_mode) return SCOUT_OK;
    CU(cudaDeviceSynchronize());
    std::vector<int32_t> err(static_cast<size_t>(e->U));
    for (int l = 0; l < e->cfg.layers; ++l) {
        CU(cudaMemcpy(err.data(), e->tier[l].err, err.size() * 4, cudaMemcpyDeviceToHost));
        for (int u = 0; u < e->U; ++u) {
            if (err[u] == 0) continue;
            const char* what = err[u] == SCOUT_ERR_INVALID_ARGUMENT ? "recall ticket rejected (schedule_recall)"
                               : err[u] == SCOUT_TIER_ERR_SPLIT   ? "split broke check_split (engine.hpp:317-329)"
                                                                  : "out of pool slots";
            const int code = err[u] == SCOUT_ERR_INVALID_ARGUMENT ? SCOUT_ERR_INVALID_ARGUMENT : SCOUT_ERR_LOGIC;
            scout_host::set_error(code, "tier state: layer %d unit %d: %s", l, u, what);
            return code;
        }
    }
    return SCOUT_OK;
}

extern "C" int scout_engine_worker_stats(scout_engine* e, double* cpu_ms_total, int* steps) {
    if (!e) return SCOUT_ERR_INVALID_ARGUMENT;
    std::lock_guard<std::mutex> lk(e->cw_mu);
    if (cpu_ms_total) *cpu_ms_total = e->cw_ms;
    if (steps) *steps = e->cw_steps;
    e->cw_ms = 0.0;
    e->cw_steps = 0;
    return SCOUT_OK;
}

extern "C" int scout_engine_k1_outputs(scout_engine* e, int32_t** res_slots, int32_t** res_ids, int32_t** n_res,
                                       int32_t** cpu_ids, int32_t** n_cpu, int32_t** res_tokens,
                                       int32_t** cpu_tokens) {
    if (!e) return SCOUT_ERR_INVALID_ARGUMENT;
    const int par = e->token & 1;  // the lists of the last step launched
    if (res_slots) *res_slots = e->I(e->res_slots[par]);
    if (res_ids) *res_ids = e->I(e->res_ids[par]);
    if (n_res) *n_res = e->I(e->n_res[par]);
    if (cpu_ids) *cpu_ids = e->I(e->cpu_ids[par]);
    if (n_cpu) *n_cpu = e->I(e->n_cpu[par]);
    if (res_tokens) *res_tokens = e->I(e->res_tok[par]);
    if (cpu_tokens) *cpu_tokens = e->I(e->cpu_tok[par]);
    return SCOUT_OK;
}
