// Host-side decode-step orchestration in C++ (the GPU side of
// ScoutEngine::decode_step, reference proj/include/scout/engine.hpp:205-314).
//
// The engine owns only launch plumbing: per-layer K1 output buffers, the K2
// workspace, a side stream + per-layer events for K4 recalls, copy streams and
// double-buffered device staging for the host-buffer path, and an event pool
// for K2 timing. Kernel launches go through the C ABI entry points; nothing
// here allocates or synchronises inside a step.
#include <cuda_runtime.h>

#include <cmath>
#include <cstring>
#include <new>
#include <vector>

#include "../../include/scout_b200.h"

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

}  // namespace

struct scout_engine {
    scout_engine_config cfg{};
    std::vector<scout_layer_desc> layers;
    int U = 0, G = 0, UG = 0;
    // per-layer K1 outputs
    Buf sel_ids, n_sel, res_slots, res_ids, n_res, cpu_ids, n_cpu, res_tok, cpu_tok;
    Buf ws;
    size_t ws_bytes = 0;
    // recall plumbing (plans copied at create: host arrays for the copy
    // engines, device arrays for the SM gather kernel)
    std::vector<std::vector<int64_t>> rc_src;
    std::vector<std::vector<int32_t>> rc_dst;
    std::vector<Buf> rc_dev;
    cudaStream_t side = nullptr;
    std::vector<cudaEvent_t> recall_ev;
    std::vector<char> recall_pending;
    cudaEvent_t ev_main = nullptr;
    // host path
    cudaStream_t h2d = nullptr, d2h = nullptr;
    Buf stage[2];  // q_true | q_pred | cpu_o | cpu_ml | out_o | out_ml, per step parity
    cudaEvent_t stage_free[2] = {nullptr, nullptr};
    std::vector<cudaEvent_t> chunk_ev;   // h2d chunk ready
    std::vector<cudaEvent_t> done_ev;    // compute chunk done
    cudaEvent_t k1_ev = nullptr;
    bool pdl = false;  // programmatic dependent launch (off: K1 runs on its own stream)
    // K1 runs one layer ahead on its own stream, co-resident with the
    // persistent K2 CTAs (K1 fits in the shared memory K2 leaves free)
    cudaStream_t k1s = nullptr;
    std::vector<cudaEvent_t> ev_k1;     // K1(i) done  -> K2(i) may read its lists
    std::vector<cudaEvent_t> ev_k2;     // K2(i) done  -> next step's K1(i) may overwrite them
    std::vector<char> k2_recorded;
    cudaEvent_t ev_start = nullptr;
    // timing
    bool timing = false;
    std::vector<cudaEvent_t> tev;
    size_t tev_used = 0;
    long long launches = 0;

    size_t lk(int layer) const { return static_cast<size_t>(layer) * U * cfg.k; }
    size_t lu(int layer) const { return static_cast<size_t>(layer) * U; }
    int32_t* I(Buf& b) const { return static_cast<int32_t*>(b.p); }

    ~scout_engine() {
        if (k1s) cudaStreamDestroy(k1s);
        for (auto e : ev_k1) cudaEventDestroy(e);
        for (auto e : ev_k2) cudaEventDestroy(e);
        if (ev_start) cudaEventDestroy(ev_start);
        if (side) cudaStreamDestroy(side);
        if (h2d) cudaStreamDestroy(h2d);
        if (d2h) cudaStreamDestroy(d2h);
        for (auto e : recall_ev) cudaEventDestroy(e);
        for (auto e : chunk_ev) cudaEventDestroy(e);
        for (auto e : done_ev) cudaEventDestroy(e);
        for (auto e : tev) cudaEventDestroy(e);
        for (auto e : stage_free)
            if (e) cudaEventDestroy(e);
        if (ev_main) cudaEventDestroy(ev_main);
        if (k1_ev) cudaEventDestroy(k1_ev);
    }

    // ---------------------------------------------------------------- K1
    int select(int layer, const float* q, int step, cudaStream_t st) {
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
        a.block_table = layers[layer].block_table;
        a.sel_ids = I(sel_ids) + lk(layer);
        a.n_sel = I(n_sel) + lu(layer);
        a.res_slots = I(res_slots) + lk(layer);
        a.res_ids = I(res_ids) + lk(layer);
        a.n_res = I(n_res) + lu(layer);
        a.cpu_ids = I(cpu_ids) + lk(layer);
        a.n_cpu = I(n_cpu) + lu(layer);
        a.res_tokens = I(res_tok) + lu(layer);
        a.cpu_tokens = I(cpu_tok) + lu(layer);
        a.flags = pdl ? SCOUT_LAUNCH_PDL : 0;
        ++launches;
        return scout_score_topk_split(&a, st);
    }

    // ------------------------------------------------------------- K2+K3
    int attend(int layer, const float* q, const float* co, const float* cml, float* o, float* ml, cudaStream_t st) {
        if (recall_pending[layer]) {
            CU(cudaStreamWaitEvent(st, recall_ev[layer], 0));
            recall_pending[layer] = 0;
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
        scout_decode_args a{};
        a.n_units = U;
        a.group = G;
        a.kv_dtype = cfg.kv_dtype;
        a.k_stride = cfg.k;
        a.scale = cfg.scale;
        a.q = q;
        a.kv_pool = cfg.kv_pool;
        a.res_slots = I(res_slots) + lk(layer);
        a.res_ids = I(res_ids) + lk(layer);
        a.n_res = I(n_res) + lu(layer);
        a.n_tokens = cfg.n_tokens;
        a.cpu_o = co;
        a.cpu_ml = cml;
        a.o = o;
        a.ml = ml;
        a.workspace = ws.p;
        a.workspace_bytes = ws_bytes;
        a.max_ctas = cfg.max_ctas;
        a.flags = pdl ? SCOUT_LAUNCH_PDL : 0;
        ++launches;
        const int rc = scout_sparse_decode(&a, st);
        if (rc != SCOUT_OK) return rc;
        if (timing) CU(cudaEventRecord(e1, st));
        return SCOUT_OK;
    }

    // ---------------------------------------------------------------- K4
    int maybe_recall(int layer, int step, cudaStream_t st) {
        const scout_layer_desc& L = layers[layer];
        if (cfg.recall_interval <= 0 || L.recall_n <= 0 || !L.recall_src || !L.recall_dst) return SCOUT_OK;
        if ((step + layer) % cfg.recall_interval != 0) return SCOUT_OK;
        CU(cudaEventRecord(ev_main, st));  // issued after the layer's attention
        CU(cudaStreamWaitEvent(side, ev_main, 0));
        int rc;
        if (cfg.recall_mode == 1) {
            ++launches;
            const int64_t* src = static_cast<const int64_t*>(rc_dev[layer].p);
            const int32_t* dst = reinterpret_cast<const int32_t*>(src + L.recall_n);
            rc = scout_recall_gather(cfg.kv_pool, cfg.kv_dtype, cfg.host_tier, src, dst, L.recall_n, side);
        } else {
            rc = scout_recall_copy(cfg.kv_pool, cfg.kv_dtype, cfg.host_tier, rc_src[layer].data(),
                                   rc_dst[layer].data(), L.recall_n, side);
        }
        if (rc != SCOUT_OK) return rc;
        CU(cudaEventRecord(recall_ev[layer], side));
        recall_pending[layer] = 1;
        return SCOUT_OK;
    }

    // K1(i) on the K1 stream (after the previous step's K2(i) released layer
    // i's lists), K2(i) on the caller's stream after K1(i).
    int k1_layer(int i, const float* q, int step) {
        if (k2_recorded[i]) CU(cudaStreamWaitEvent(k1s, ev_k2[i], 0));
        const int rc = select(i, q, step, k1s);
        if (rc != SCOUT_OK) return rc;
        CU(cudaEventRecord(ev_k1[i], k1s));
        return SCOUT_OK;
    }
    int k2_layer(int i, int step, const float* qt, const float* co, const float* cml, float* o, float* ml,
                 cudaStream_t st) {
        CU(cudaStreamWaitEvent(st, ev_k1[i], 0));
        int rc = attend(i, qt, co, cml, o, ml, st);
        if (rc != SCOUT_OK) return rc;
        CU(cudaEventRecord(ev_k2[i], st));
        k2_recorded[i] = 1;
        return maybe_recall(i, step, st);
    }
    // inputs written to `st` before the step are visible to the K1 stream
    int begin_step(cudaStream_t st) {
        CU(cudaEventRecord(ev_start, st));
        CU(cudaStreamWaitEvent(k1s, ev_start, 0));
        return SCOUT_OK;
    }
    int end_step(cudaStream_t st) {
        CU(cudaEventRecord(ev_start, k1s));
        CU(cudaStreamWaitEvent(st, ev_start, 0));
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
    if (c.layers <= 0 || c.batch <= 0 || c.hkv <= 0 || c.hq % c.hkv != 0 || c.k <= 0 || c.nb_stride <= 0 ||
        !c.kv_pool || !c.n_tokens || !(c.scale > 0.f)) {
        set_error(SCOUT_ERR_INVALID_ARGUMENT, "scout_engine_create: bad config");
        return SCOUT_ERR_INVALID_ARGUMENT;
    }
    if (c.recall_interval > 0 && !c.host_tier) {
        set_error(SCOUT_ERR_INVALID_ARGUMENT, "scout_engine_create: recall needs a host tier");
        return SCOUT_ERR_INVALID_ARGUMENT;
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
    const size_t lk = static_cast<size_t>(c.layers) * e->U * c.k * 4, lu = static_cast<size_t>(c.layers) * e->U * 4;
    int bad = e->sel_ids.alloc(lk) | e->res_slots.alloc(lk) | e->res_ids.alloc(lk) | e->cpu_ids.alloc(lk) |
              e->n_sel.alloc(lu) | e->n_res.alloc(lu) | e->n_cpu.alloc(lu) | e->res_tok.alloc(lu) |
              e->cpu_tok.alloc(lu);
    e->ws_bytes = scout_sparse_decode_workspace_bytes(e->U, e->G, c.max_ctas);
    bad |= e->ws.alloc(e->ws_bytes);
    if (!bad && cudaMemset(e->ws.p, 0, e->ws_bytes) != cudaSuccess) bad = 1;
    if (!bad && c.host_staging) {
        // q_true | q_pred | cpu_o | cpu_ml | out_o | out_ml, per step parity
        const size_t per = static_cast<size_t>(c.layers) * e->UG * (4 * SCOUT_HEAD_DIM + 4) * 4;
        bad |= e->stage[0].alloc(per) | e->stage[1].alloc(per);
    }
    if (bad) {
        delete e;
        set_error(SCOUT_ERR_CUDA, "scout_engine_create: device allocation failed");
        return SCOUT_ERR_CUDA;
    }
    cudaStreamCreateWithFlags(&e->side, cudaStreamNonBlocking);
    cudaStreamCreateWithFlags(&e->k1s, cudaStreamNonBlocking);
    cudaEventCreateWithFlags(&e->ev_start, cudaEventDisableTiming);
    e->ev_k1.resize(c.layers);
    e->ev_k2.resize(c.layers);
    for (auto& ev : e->ev_k1) cudaEventCreateWithFlags(&ev, cudaEventDisableTiming);
    for (auto& ev : e->ev_k2) cudaEventCreateWithFlags(&ev, cudaEventDisableTiming);
    e->k2_recorded.assign(c.layers, 0);
    cudaStreamCreateWithFlags(&e->h2d, cudaStreamNonBlocking);
    cudaStreamCreateWithFlags(&e->d2h, cudaStreamNonBlocking);
    cudaEventCreateWithFlags(&e->ev_main, cudaEventDisableTiming);
    cudaEventCreateWithFlags(&e->k1_ev, cudaEventDisableTiming);
    for (int i = 0; i < 2; ++i) cudaEventCreateWithFlags(&e->stage_free[i], cudaEventDisableTiming);
    e->recall_ev.resize(c.layers);
    for (auto& ev : e->recall_ev) cudaEventCreateWithFlags(&ev, cudaEventDisableTiming);
    e->recall_pending.assign(c.layers, 0);
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
    const int nch = (c.layers + e->cfg.chunk_layers - 1) / e->cfg.chunk_layers;
    e->chunk_ev.resize(nch);
    e->done_ev.resize(nch);
    for (auto& ev : e->chunk_ev) cudaEventCreateWithFlags(&ev, cudaEventDisableTiming);
    for (auto& ev : e->done_ev) cudaEventCreateWithFlags(&ev, cudaEventDisableTiming);
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
    delete eng;
    return SCOUT_OK;
}

extern "C" int scout_engine_decode_step(scout_engine* e, int step, const float* q_true, const float* q_pred,
                                        const float* cpu_o, const float* cpu_ml, float* out_o, float* out_ml,
                                        void* stream) {
    if (!e || !q_true || !q_pred || !out_o || !out_ml || ((cpu_o == nullptr) != (cpu_ml == nullptr))) {
        scout_host::set_error(SCOUT_ERR_INVALID_ARGUMENT, "scout_engine_decode_step: null buffer");
        return SCOUT_ERR_INVALID_ARGUMENT;
    }
    auto st = static_cast<cudaStream_t>(stream);
    const size_t qd = static_cast<size_t>(e->UG) * SCOUT_HEAD_DIM, md = static_cast<size_t>(e->UG) * 2;
    const int L = e->cfg.layers;
    int rc = e->begin_step(st);
    // K1 runs ahead: layer 0 with the true query, layer i+1 with the predicted one
    for (int i = 0; i < L && rc == SCOUT_OK; ++i) {
        rc = e->k1_layer(i, i == 0 ? q_true : q_pred + i * qd, step);
        if (rc == SCOUT_OK) rc = e->k2_layer(i, step, q_true + i * qd, cpu_o ? cpu_o + i * qd : nullptr,
                                             cpu_ml ? cpu_ml + i * md : nullptr, out_o + i * qd, out_ml + i * md, st);
    }
    if (rc != SCOUT_OK) return rc;
    return e->end_step(st);
}

extern "C" int scout_engine_decode_step_host(scout_engine* e, int step, const float* h_q_true, const float* h_q_pred,
                                             const float* h_cpu_o, const float* h_cpu_ml, float* h_out_o,
                                             float* h_out_ml, int32_t* h_cpu_ids, int32_t* h_n_cpu, void* stream) {
    if (!e || !e->stage[0].p || !h_q_true || !h_q_pred || !h_out_o || !h_out_ml ||
        ((h_cpu_o == nullptr) != (h_cpu_ml == nullptr))) {
        scout_host::set_error(SCOUT_ERR_INVALID_ARGUMENT,
                              "scout_engine_decode_step_host: null buffer or engine created without host_staging");
        return SCOUT_ERR_INVALID_ARGUMENT;
    }
    auto st = static_cast<cudaStream_t>(stream);
    const int L = e->cfg.layers, CH = e->cfg.chunk_layers;
    const int nch = (L + CH - 1) / CH;
    const size_t qd = static_cast<size_t>(e->UG) * SCOUT_HEAD_DIM, md = static_cast<size_t>(e->UG) * 2;
    const int par = step & 1;
    float* base = static_cast<float*>(e->stage[par].p);
    float* d_qt = base;
    float* d_qp = d_qt + L * qd;
    float* d_co = d_qp + L * qd;
    float* d_cm = d_co + L * qd;
    // staging of this parity is free once the step two steps back finished
    CU(cudaStreamWaitEvent(e->h2d, e->stage_free[par], 0));
    for (int c = 0; c < nch; ++c) {
        const int lo = c * CH, n = (c + 1) * CH > L ? L - lo : CH;
        CU(cudaMemcpyAsync(d_qt + lo * qd, h_q_true + lo * qd, n * qd * 4, cudaMemcpyHostToDevice, e->h2d));
        CU(cudaMemcpyAsync(d_qp + lo * qd, h_q_pred + lo * qd, n * qd * 4, cudaMemcpyHostToDevice, e->h2d));
        if (h_cpu_o) {
            CU(cudaMemcpyAsync(d_co + lo * qd, h_cpu_o + lo * qd, n * qd * 4, cudaMemcpyHostToDevice, e->h2d));
            CU(cudaMemcpyAsync(d_cm + lo * md, h_cpu_ml + lo * md, n * md * 4, cudaMemcpyHostToDevice, e->h2d));
        }
        CU(cudaEventRecord(e->chunk_ev[c], e->h2d));
    }
    float* d_o = d_cm + L * md;   // outputs: [L][UG][128] then [L][UG][2]
    float* d_oml = d_o + L * qd;
    // K1 stream: waits for each input chunk, runs one layer ahead of K2
    int rc = e->begin_step(st);
    if (rc != SCOUT_OK) return rc;
    for (int i = 0; i < L; ++i) {
        if (i % CH == 0) {
            CU(cudaStreamWaitEvent(st, e->chunk_ev[i / CH], 0));
            CU(cudaStreamWaitEvent(e->k1s, e->chunk_ev[i / CH], 0));
        }
        rc = e->k1_layer(i, i == 0 ? d_qt : d_qp + i * qd, step);
        if (rc != SCOUT_OK) return rc;
        if (h_cpu_ids && i > 0) {
            // the host co-attention worker needs layer i's CPU-side ids as soon as K1(i) is done
            CU(cudaStreamWaitEvent(e->d2h, e->ev_k1[i], 0));
            CU(cudaMemcpyAsync(h_cpu_ids + e->lk(i), e->I(e->cpu_ids) + e->lk(i),
                               static_cast<size_t>(e->U) * e->cfg.k * 4, cudaMemcpyDeviceToHost, e->d2h));
            if (h_n_cpu)
                CU(cudaMemcpyAsync(h_n_cpu + e->lu(i), e->I(e->n_cpu) + e->lu(i), static_cast<size_t>(e->U) * 4,
                                   cudaMemcpyDeviceToHost, e->d2h));
        }
        rc = e->k2_layer(i, step, d_qt + i * qd, h_cpu_o ? d_co + i * qd : nullptr, h_cpu_ml ? d_cm + i * md : nullptr,
                         d_o + i * qd, d_oml + i * md, st);
        if (rc != SCOUT_OK) return rc;
        if (i % CH == CH - 1 || i == L - 1) {
            const int c = i / CH, lo = c * CH, n = i + 1 - lo;
            CU(cudaEventRecord(e->done_ev[c], st));
            CU(cudaStreamWaitEvent(e->d2h, e->done_ev[c], 0));
            CU(cudaMemcpyAsync(h_out_o + lo * qd, d_o + lo * qd, n * qd * 4, cudaMemcpyDeviceToHost, e->d2h));
            CU(cudaMemcpyAsync(h_out_ml + lo * md, d_oml + lo * md, n * md * 4, cudaMemcpyDeviceToHost, e->d2h));
        }
    }
    if ((rc = e->end_step(st)) != SCOUT_OK) return rc;
    if (h_cpu_ids) {  // layer 0's ids (selected on the true query; layer 0 is pinned so none)
        CU(cudaMemcpyAsync(h_cpu_ids, e->I(e->cpu_ids), static_cast<size_t>(e->U) * e->cfg.k * 4,
                           cudaMemcpyDeviceToHost, e->d2h));
        if (h_n_cpu)
            CU(cudaMemcpyAsync(h_n_cpu, e->I(e->n_cpu), static_cast<size_t>(e->U) * 4, cudaMemcpyDeviceToHost, e->d2h));
    }
    CU(cudaEventRecord(e->ev_main, e->d2h));
    CU(cudaStreamWaitEvent(st, e->ev_main, 0));
    CU(cudaEventRecord(e->stage_free[par], st));
    return SCOUT_OK;
}

extern "C" int scout_engine_sync(scout_engine* e, void* stream) {
    if (!e) return SCOUT_ERR_INVALID_ARGUMENT;
    auto st = static_cast<cudaStream_t>(stream);
    CU(cudaEventRecord(e->ev_main, e->side));
    CU(cudaStreamWaitEvent(st, e->ev_main, 0));
    std::fill(e->recall_pending.begin(), e->recall_pending.end(), 0);
    return SCOUT_OK;
}

extern "C" int scout_engine_set_timing(scout_engine* e, int enable) {
    if (!e) return SCOUT_ERR_INVALID_ARGUMENT;
    e->timing = enable != 0;
    e->tev_used = 0;
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

extern "C" int scout_engine_k1_outputs(scout_engine* e, int32_t** res_slots, int32_t** res_ids, int32_t** n_res,
                                       int32_t** cpu_ids, int32_t** n_cpu, int32_t** res_tokens,
                                       int32_t** cpu_tokens) {
    if (!e) return SCOUT_ERR_INVALID_ARGUMENT;
    if (res_slots) *res_slots = e->I(e->res_slots);
    if (res_ids) *res_ids = e->I(e->res_ids);
    if (n_res) *n_res = e->I(e->n_res);
    if (cpu_ids) *cpu_ids = e->I(e->cpu_ids);
    if (n_cpu) *n_cpu = e->I(e->n_cpu);
    if (res_tokens) *res_tokens = e->I(e->res_tok);
    if (cpu_tokens) *cpu_tokens = e->I(e->cpu_tok);
    return SCOUT_OK;
}
