// ref_shim.cpp — C entry points over the UNMODIFIED reference headers.
//
// TEST / BASELINE INFRASTRUCTURE ONLY. Built by oracle/Makefile with
// -I /root/reference/proj/include into oracle/_ref/libscout_ref.so (git-ignored,
// travels to the GPU box). It is (1) the generator of the golden vectors under
// tests/golden/ (script tests/golden/make_golden.py), (2) a second oracle for
// the restatement oracle/scout_oracle.c, and (3) the CPU baseline that
// bench.py times ("kind": "reference"): the reference's own select_topk /
// partial_attention / merge / finalize on the same workload shape.
#include <atomic>
#include <chrono>
#include <cstdint>
#include <cstring>
#include <span>
#include <stdexcept>
#include <thread>
#include <vector>

#include "scout/attention.hpp"
#include "scout/digest.hpp"
#include "scout/kv_store.hpp"
#include "scout/model.hpp"
#include "scout/recall.hpp"
#ifdef SCOUT_REF_HARNESS
#include "scout/harness.hpp"  // recompute_layer_attention (needs nlohmann json.hpp on the include path)
#endif

using scout::BlockDigest;
using scout::BlockIdSet;
using scout::KvBlock;
using scout::Mat;
using scout::PartialAttention;
using scout::Vec;

namespace {

Mat mat_from(const double* p, int rows, int cols) {
    Mat m(rows, cols);
    std::memcpy(m.data.data(), p, sizeof(double) * static_cast<size_t>(rows) * cols);
    return m;
}

// Stacked GQA digest for block b of one unit: q_s[c*G+g], lo/hi tiled G times.
BlockDigest stacked_digest(const double* dig, int G, int d, int nb_stride, int b, int method) {
    BlockDigest bd;
    bd.block_id = static_cast<size_t>(b);
    if (method == 0) {
        bd.method = scout::DigestMethod::minmax;
        bd.lo.resize(static_cast<size_t>(G) * d);
        bd.hi.resize(static_cast<size_t>(G) * d);
        for (int c = 0; c < d; ++c)
            for (int g = 0; g < G; ++g) {
                bd.lo[c * G + g] = dig[static_cast<size_t>(c) * nb_stride + b];
                bd.hi[c * G + g] = dig[static_cast<size_t>(d + c) * nb_stride + b];
            }
    } else {
        bd.method = scout::DigestMethod::mean;
        bd.mean.resize(static_cast<size_t>(G) * d);
        for (int c = 0; c < d; ++c)
            for (int g = 0; g < G; ++g) bd.mean[c * G + g] = dig[static_cast<size_t>(c) * nb_stride + b];
    }
    return bd;
}

Vec stacked_query(const double* q, int G, int d) {
    Vec qs(static_cast<size_t>(G) * d);
    for (int c = 0; c < d; ++c)
        for (int g = 0; g < G; ++g) qs[c * G + g] = q[static_cast<size_t>(g) * d + c];
    return qs;
}

}  // namespace

extern "C" {

// build_digest (digest.hpp:34) — method 0 minmax (lo, hi), 1 mean (lo = mean).
int ref_build_digest(const double* keys, int rows, int d, int method, double* lo, double* hi) {
    try {
        const BlockDigest bd = scout::build_digest(mat_from(keys, rows, d),
                                                   method == 0 ? scout::DigestMethod::minmax : scout::DigestMethod::mean);
        if (method == 0) {
            std::memcpy(lo, bd.lo.data(), sizeof(double) * d);
            std::memcpy(hi, bd.hi.data(), sizeof(double) * d);
        } else {
            std::memcpy(lo, bd.mean.data(), sizeof(double) * d);
        }
        return 0;
    } catch (const std::invalid_argument&) {
        return -1;
    }
}

// digest_score (digest.hpp:62) on an n-vector.
double ref_digest_score(const double* q, const double* lo, const double* hi, int n, int method) {
    BlockDigest bd;
    if (method == 0) {
        bd.method = scout::DigestMethod::minmax;
        bd.lo.assign(lo, lo + n);
        bd.hi.assign(hi, hi + n);
    } else {
        bd.method = scout::DigestMethod::mean;
        bd.mean.assign(lo, lo + n);
    }
    return scout::digest_score(Vec(q, q + n), bd);
}

// select_topk (digest.hpp:101) for one unit under the stacked-GQA rule.
// digests: [2][d][nb_stride] (minmax) or [d][nb_stride] (mean). Returns the
// number of ids written ascending to out, -1 on std::invalid_argument.
int ref_unit_topk(const double* q, int G, int d, const double* dig, int nb_stride, int nb, int k, int method,
                  int32_t* out, double* scores) {
    std::vector<BlockDigest> ds;
    ds.reserve(static_cast<size_t>(nb));
    for (int b = 0; b < nb; ++b) ds.push_back(stacked_digest(dig, G, d, nb_stride, b, method));
    const Vec qs = stacked_query(q, G, d);
    try {
        if (scores)
            for (int b = 0; b < nb; ++b) scores[b] = scout::digest_score(qs, ds[b]);
        const BlockIdSet ids = scout::select_topk(qs, ds, static_cast<size_t>(k));
        for (size_t i = 0; i < ids.size(); ++i) out[i] = static_cast<int32_t>(ids[i]);
        return static_cast<int>(ids.size());
    } catch (const std::invalid_argument&) {
        return -1;
    }
}

// Generic select_topk over single-head digests given as [n][dim] arrays.
int ref_select_topk(const double* q, int dim, const double* lo, const double* hi, int n, int k, int method,
                    int32_t* out) {
    std::vector<BlockDigest> ds(static_cast<size_t>(n));
    for (int i = 0; i < n; ++i) {
        ds[i].block_id = static_cast<size_t>(i);
        if (method == 0) {
            ds[i].method = scout::DigestMethod::minmax;
            ds[i].lo.assign(lo + static_cast<size_t>(i) * dim, lo + static_cast<size_t>(i + 1) * dim);
            ds[i].hi.assign(hi + static_cast<size_t>(i) * dim, hi + static_cast<size_t>(i + 1) * dim);
        } else {
            ds[i].method = scout::DigestMethod::mean;
            ds[i].mean.assign(lo + static_cast<size_t>(i) * dim, lo + static_cast<size_t>(i + 1) * dim);
        }
    }
    try {
        const BlockIdSet ids = scout::select_topk(Vec(q, q + dim), ds, static_cast<size_t>(k));
        for (size_t i = 0; i < ids.size(); ++i) out[i] = static_cast<int32_t>(ids[i]);
        return static_cast<int>(ids.size());
    } catch (const std::invalid_argument&) {
        return -1;
    }
}

// partial_attention (attention.hpp:73) over nblk blocks; block i has rows[i]
// rows starting at row offset sum(rows[:i]) of keys/values [total][d].
int ref_partial_attention(const double* q, int d, const double* keys, const double* values, const int32_t* rows,
                          int nblk, double scale, double* o_acc, double* max_logit, double* denom, int64_t* count) {
    std::vector<KvBlock> blocks(static_cast<size_t>(nblk));
    size_t off = 0;
    for (int i = 0; i < nblk; ++i) {
        blocks[i].block_id = static_cast<size_t>(i);
        blocks[i].keys = mat_from(keys + off * d, rows[i], d);
        blocks[i].values = mat_from(values + off * d, rows[i], d);
        blocks[i].sealed = true;
        off += static_cast<size_t>(rows[i]);
    }
    std::vector<const KvBlock*> ptrs;
    for (const KvBlock& b : blocks) ptrs.push_back(&b);
    try {
        const PartialAttention p = scout::partial_attention(Vec(q, q + d), ptrs, scale);
        std::memcpy(o_acc, p.o_acc.data(), sizeof(double) * d);
        *max_logit = p.max_logit;
        *denom = p.denom;
        *count = static_cast<int64_t>(p.token_count);
        return 0;
    } catch (const std::invalid_argument&) {
        return -1;
    }
}

// merge (attention.hpp:100) of two partials.
int ref_merge(int d, const double* oa, double ma, double la, int64_t na, const double* ob, double mb, double lb,
              int64_t nb, double* o, double* m, double* l, int64_t* n) {
    PartialAttention a, b;
    a.o_acc.assign(oa, oa + d); a.max_logit = ma; a.denom = la; a.token_count = static_cast<size_t>(na);
    b.o_acc.assign(ob, ob + d); b.max_logit = mb; b.denom = lb; b.token_count = static_cast<size_t>(nb);
    try {
        const PartialAttention r = scout::merge(a, b);
        std::memcpy(o, r.o_acc.data(), sizeof(double) * d);
        *m = r.max_logit; *l = r.denom; *n = static_cast<int64_t>(r.token_count);
        return 0;
    } catch (const std::invalid_argument&) {
        return -1;
    }
}

// finalize (attention.hpp:117); -1 for an empty partial.
int ref_finalize(int d, const double* o_acc, double denom, int64_t count, double* out) {
    PartialAttention p;
    p.o_acc.assign(o_acc, o_acc + d); p.denom = denom; p.token_count = static_cast<size_t>(count);
    try {
        const Vec v = scout::finalize(p);
        std::memcpy(out, v.data(), sizeof(double) * d);
        return 0;
    } catch (const std::invalid_argument&) {
        return -1;
    }
}

// ------------------------------------------------------------------ baseline
// The reference's per-(request, layer) decode work, as the GPU arm does it:
// for each of hkv units: select_topk (stacked) over nb digests, split against
// the resident set (set_intersection, engine.hpp:240), partial_attention per
// query head over the resident blocks, merge with a pre-staged CPU partial,
// finalize. `samples` distinct (request, layer) inputs are cycled through
// `units_total` times by `threads` std::threads. Returns seconds.
struct RefSample {
    std::vector<std::vector<BlockDigest>> digests;  // [hkv][nb]
    std::vector<BlockIdSet> residency;              // [hkv]
    std::vector<std::vector<KvBlock>> blocks;       // [hkv][nb] (only resident ones filled)
    std::vector<Vec> q;                             // [hq] (true query, widened f32)
    std::vector<Vec> qs;                            // [hkv] stacked predicted query
    std::vector<PartialAttention> cpu;              // [hq]
};

double ref_cpu_baseline(int samples, int hq, int hkv, int d, int nb, int k, const double* q /*[s][hq][d]*/,
                        const double* digests /*[s][hkv][2][d][nb]*/, const int32_t* resident /*[s][hkv][nb] 0/1*/,
                        const double* kv /*[s][hkv][nb_res_max][2][64][d]*/, const int32_t* res_index /*[s][hkv][nb]*/,
                        int nb_res_max, int units_total, int threads, double* checksum) {
    const int G = hq / hkv;
    const double scale = 1.0 / std::sqrt(static_cast<double>(d));
    std::vector<RefSample> S(static_cast<size_t>(samples));
    for (int s = 0; s < samples; ++s) {
        RefSample& rs = S[s];
        rs.digests.resize(hkv);
        rs.residency.resize(hkv);
        rs.blocks.resize(hkv);
        rs.qs.resize(hkv);
        for (int h = 0; h < hq; ++h) {
            const double* qp = q + (static_cast<size_t>(s) * hq + h) * d;
            rs.q.emplace_back(qp, qp + d);
            PartialAttention cp = PartialAttention::empty(static_cast<size_t>(d));
            for (int c = 0; c < d; ++c) cp.o_acc[c] = qp[c] * 0.01;  // synthetic pre-staged CPU partial
            cp.max_logit = 0.5; cp.denom = 3.0; cp.token_count = 64;
            rs.cpu.push_back(cp);
        }
        for (int u = 0; u < hkv; ++u) {
            const double* dig = digests + (static_cast<size_t>(s) * hkv + u) * 2 * d * nb;
            for (int b = 0; b < nb; ++b) rs.digests[u].push_back(stacked_digest(dig, G, d, nb, b, 0));
            rs.qs[u] = stacked_query(q + (static_cast<size_t>(s) * hq + u * G) * d, G, d);
            rs.blocks[u].resize(static_cast<size_t>(nb));
            for (int b = 0; b < nb; ++b) {
                if (!resident[(static_cast<size_t>(s) * hkv + u) * nb + b]) continue;
                rs.residency[u].push_back(static_cast<size_t>(b));
                const int ri = res_index[(static_cast<size_t>(s) * hkv + u) * nb + b];
                const double* kb = kv + ((static_cast<size_t>(s) * hkv + u) * nb_res_max + ri) * 2 * 64 * d;
                KvBlock& blk = rs.blocks[u][b];
                blk.block_id = static_cast<size_t>(b);
                blk.keys = mat_from(kb, 64, d);
                blk.values = mat_from(kb + 64 * d, 64, d);
                blk.sealed = true;
            }
        }
    }
    std::atomic<int> next{0};
    std::vector<double> sums(static_cast<size_t>(threads), 0.0);
    auto worker = [&](int tix) {
        double acc = 0.0;
        for (;;) {
            const int i = next.fetch_add(1);
            if (i >= units_total) break;
            const RefSample& rs = S[i % samples];
            for (int u = 0; u < hkv; ++u) {
                const BlockIdSet pred = scout::select_topk(rs.qs[u], rs.digests[u], static_cast<size_t>(k));
                const BlockIdSet res = scout::set_intersection(pred, rs.residency[u]);
                std::vector<const KvBlock*> ptrs;
                ptrs.reserve(res.size());
                for (size_t id : res) ptrs.push_back(&rs.blocks[u][id]);
                for (int g = 0; g < G; ++g) {
                    const int h = u * G + g;
                    const PartialAttention gp = scout::partial_attention(rs.q[h], ptrs, scale);
                    const PartialAttention m = scout::merge(gp, rs.cpu[h]);
                    const Vec o = m.is_empty() ? Vec(static_cast<size_t>(d), 0.0) : scout::finalize(m);
                    acc += o[0];
                }
            }
        }
        sums[tix] = acc;
    };
    const auto t0 = std::chrono::steady_clock::now();
    std::vector<std::thread> pool;
    for (int t = 0; t < threads; ++t) pool.emplace_back(worker, t);
    for (auto& th : pool) th.join();
    const double secs = std::chrono::duration<double>(std::chrono::steady_clock::now() - t0).count();
    if (checksum) {
        double s = 0.0;
        for (double v : sums) s += v;
        *checksum = s;
    }
    return secs;
}

// ---- TieredKvCache (kv_store.hpp) driven through a handle: the oracle of the
// device tier bookkeeping (K5). Values of K/V rows do not matter for the tier
// state except through place_after_prefill, which scores the digests.
void* ref_cache_new(int layers, int block_size, int head_dim, int method, long long capacity) {
    try {
        return new scout::TieredKvCache(static_cast<size_t>(layers), static_cast<size_t>(block_size),
                                        static_cast<size_t>(head_dim),
                                        method == 0 ? scout::DigestMethod::minmax : scout::DigestMethod::mean,
                                        static_cast<size_t>(capacity));
    } catch (const std::invalid_argument&) {
        return nullptr;
    }
}
void ref_cache_free(void* c) { delete static_cast<scout::TieredKvCache*>(c); }
void ref_cache_pin(void* c, int layer) { static_cast<scout::TieredKvCache*>(c)->pin_layer(static_cast<size_t>(layer)); }
// returns the sealed block id, -1 if the append sealed nothing, -2 on invalid_argument
long long ref_cache_append(void* c, int layer, const double* k, const double* v, int d) {
    try {
        const auto r = static_cast<scout::TieredKvCache*>(c)->append_token(static_cast<size_t>(layer), Vec(k, k + d),
                                                                            Vec(v, v + d));
        return r ? static_cast<long long>(*r) : -1;
    } catch (const std::invalid_argument&) {
        return -2;
    }
}
// number of tickets applied
int ref_cache_begin_layer(void* c, long long step, int layer) {
    return static_cast<int>(
        static_cast<scout::TieredKvCache*>(c)->begin_layer(static_cast<size_t>(step), static_cast<size_t>(layer)).size());
}
int ref_cache_schedule_recall(void* c, int layer, const int32_t* ids, int n, long long issue_step, int issue_layer) {
    try {
        BlockIdSet s(ids, ids + n);
        static_cast<scout::TieredKvCache*>(c)->schedule_recall(static_cast<size_t>(layer), s,
                                                               static_cast<size_t>(issue_step),
                                                               static_cast<size_t>(issue_layer));
        return 0;
    } catch (const std::invalid_argument&) {
        return -1;
    }
}
int ref_cache_mark_selected(void* c, int layer, const int32_t* ids, int n, long long step) {
    try {
        BlockIdSet s(ids, ids + n);
        static_cast<scout::TieredKvCache*>(c)->mark_selected(static_cast<size_t>(layer), s, static_cast<size_t>(step));
        return 0;
    } catch (const std::invalid_argument&) {
        return -1;
    }
}
int ref_cache_residency(void* c, int layer, int32_t* out) {
    const BlockIdSet r = static_cast<scout::TieredKvCache*>(c)->residency_set(static_cast<size_t>(layer));
    for (size_t i = 0; i < r.size(); ++i) out[i] = static_cast<int32_t>(r[i]);
    return static_cast<int>(r.size());
}
// per block: tier (1 fast), last_selected, in flight (1/0); returns the block count
int ref_cache_state(void* c, int layer, int32_t* tier, int64_t* last_sel, int32_t* in_flight) {
    const auto* kc = static_cast<scout::TieredKvCache*>(c);
    const size_t L = static_cast<size_t>(layer);
    const size_t n = kc->block_count(L);
    for (size_t id = 0; id < n; ++id) {
        tier[id] = kc->tier_of(L, id) == scout::Tier::fast ? 1 : 0;
        last_sel[id] = static_cast<int64_t>(kc->last_selected(L, id));
        in_flight[id] = kc->is_in_flight(L, id) ? 1 : 0;
    }
    return static_cast<int>(n);
}
int ref_cache_place(void* c, int layer, const double* q, int d) {
    try {
        static_cast<scout::TieredKvCache*>(c)->place_after_prefill(static_cast<size_t>(layer), Vec(q, q + d));
        return 0;
    } catch (const std::invalid_argument&) {
        return -1;
    }
}
// the layer's digests as [2][d][nb_stride] (minmax) for the GPU side of a place test
int ref_cache_digests(void* c, int layer, int d, int nb_stride, double* out) {
    const auto& ds = static_cast<scout::TieredKvCache*>(c)->digests(static_cast<size_t>(layer));
    for (size_t b = 0; b < ds.size(); ++b)
        for (int ch = 0; ch < d; ++ch) {
            out[static_cast<size_t>(ch) * nb_stride + b] = ds[b].lo[ch];
            out[static_cast<size_t>(d + ch) * nb_stride + b] = ds[b].hi[ch];
        }
    return static_cast<int>(ds.size());
}

// predict_next_query(rms_normalize(x), W) (model.hpp:215-217, numerics.hpp:99-123):
// the oracle of K6. W [hidden][n_out] row-major.
int ref_predict_query(const double* x, int hidden, const double* w, int n_out, double* out) {
    try {
        const Vec xn = scout::rms_normalize(Vec(x, x + hidden));
        const Vec q = scout::predict_next_query(xn, mat_from(w, hidden, n_out));
        std::memcpy(out, q.data(), sizeof(double) * n_out);
        return 0;
    } catch (const std::invalid_argument&) {
        return -1;
    }
}

// ---- recall policy (recall.hpp:69-126) for n_units independent reference
// engines sharing one schedule: the oracle of the device tier mode's cadence
// and recall set. intervals: [layers], each >= 1.
struct RefRecall {
    scout::RecallSchedule schedule;
    std::vector<scout::RecallPolicyState> state;  // one per unit
};
void* ref_recall_new(int n_units, int layers, const int32_t* intervals, double beta) {
    auto* r = new RefRecall();
    r->schedule.intervals.assign(intervals, intervals + layers);
    r->schedule.beta = beta;
    r->state.assign(static_cast<size_t>(n_units), scout::RecallPolicyState(static_cast<size_t>(layers)));
    return r;
}
void ref_recall_free(void* h) { delete static_cast<RefRecall*>(h); }
// calibrate_intervals (recall.hpp:79-95) on a RatioTrace built from
// [layers][steps] samples (steps 1..steps): 0, or -1 if the reference threw
int ref_calibrate_intervals(const int64_t* cpu, const int64_t* budget, int layers, int steps, double beta,
                            int32_t* out) {
    try {
        scout::RatioTrace trace(static_cast<size_t>(layers));
        for (int l = 0; l < layers; ++l)
            for (int t = 0; t < steps; ++t)
                trace.record(static_cast<size_t>(l), static_cast<size_t>(t + 1),
                             static_cast<size_t>(cpu[static_cast<size_t>(l) * steps + t]),
                             static_cast<size_t>(budget[static_cast<size_t>(l) * steps + t]));
        const scout::RecallSchedule s = scout::calibrate_intervals(trace, beta);
        for (int l = 0; l < layers; ++l) out[l] = static_cast<int32_t>(s.intervals[static_cast<size_t>(l)]);
        return 0;
    } catch (const std::exception&) {
        return -1;
    }
}
// maybe_schedule_recall for one unit: -1 when the layer is not due (nullopt),
// else the number of ids of set_difference(predicted, residency) written to out
int ref_maybe_schedule_recall(void* h, int unit, int layer, long long step, const int32_t* pred, int n_pred,
                              const int32_t* res, int n_res, int32_t* out) {
    auto* r = static_cast<RefRecall*>(h);
    const BlockIdSet p(pred, pred + n_pred), rs(res, res + n_res);
    const auto ids = scout::maybe_schedule_recall(r->schedule, r->state.at(static_cast<size_t>(unit)),
                                                  static_cast<size_t>(layer), static_cast<size_t>(step), p, rs);
    if (!ids) return -1;
    for (size_t i = 0; i < ids->size(); ++i) out[i] = static_cast<int32_t>((*ids)[i]);
    return static_cast<int>(ids->size());
}

#ifdef SCOUT_REF_HARNESS
// recompute_layer_attention (harness.hpp:318-329), the reference's hybrid-query
// oracle of one decode layer, for the G query heads of one unit: the layer's
// whole final K/V stream (n_rows rows, block_size-row blocks) goes into a
// one-layer TieredKvCache; blocks that grew after the attention are truncated
// back to tokens_at_attention; q_true over the resident set, q_pred over the
// CPU set, merged and finalised (both empty -> zeros). out: [G][d]. Returns 0,
// or -1 if the reference threw.
int ref_recompute_layer_attention(int d, int block_size, const double* keys, const double* values, int n_rows,
                                  int tokens_at_attention, int G, const double* q_true, const double* q_pred,
                                  const int32_t* res_ids, int n_res, const int32_t* cpu_ids, int n_cpu, double scale,
                                  double* out) {
    try {
        scout::TieredKvCache cache(1, static_cast<size_t>(block_size), static_cast<size_t>(d), scout::DigestMethod::minmax,
                                   1u << 20);
        for (int r = 0; r < n_rows; ++r)
            cache.append_token(0, Vec(keys + static_cast<size_t>(r) * d, keys + static_cast<size_t>(r + 1) * d),
                               Vec(values + static_cast<size_t>(r) * d, values + static_cast<size_t>(r + 1) * d));
        scout::LayerMetrics lm;
        lm.layer = 0;
        lm.resident_set.assign(res_ids, res_ids + n_res);
        lm.cpu_set.assign(cpu_ids, cpu_ids + n_cpu);
        lm.tokens_at_attention = static_cast<size_t>(tokens_at_attention);
        lm.attn_out.assign(static_cast<size_t>(d), 0.0);
        for (int g = 0; g < G; ++g) {
            lm.q_true.assign(q_true + static_cast<size_t>(g) * d, q_true + static_cast<size_t>(g + 1) * d);
            lm.q_pred.assign(q_pred + static_cast<size_t>(g) * d, q_pred + static_cast<size_t>(g + 1) * d);
            const Vec o = scout::recompute_layer_attention(cache, scale, lm);
            std::memcpy(out + static_cast<size_t>(g) * d, o.data(), sizeof(double) * d);
        }
        return 0;
    } catch (const std::exception&) {
        return -1;
    }
}
#endif

}  // extern "C"
