// The drop-in proof: the reference's own ScoutEngine (engine.hpp, unmodified
// but for the INTEGRATION.md §1 call swaps applied by tests/cpp/Makefile) runs
// its hot path -- select_topk, partial_attention, merge, finalize -- on the
// B200 through include/scout_b200.hpp, on the reference's own types.
//
// Checked against the reference itself, linked into the same binary:
//   1. frozen stream (the scenario of test_engine.cpp:69-102): with alpha = 0
//      the layer inputs never change, so every layer's selection must equal
//      select_topk over a monolithic cache, and every output the single-device
//      oracle reference_block_sparse (engine.hpp:358-369), within 1e-3;
//   2. side by side with the unmodified reference ScoutEngine (alpha 0.1,
//      periodic recall, the layer-ahead CPU worker, serial and threaded):
//      identical predicted / resident / CPU sets and event logs, outputs within
//      1e-3, at the reference tests' geometry (head_dim 10, block 4) and at
//      the GPU's native one (head_dim 128, block 64);
//   3. exact when the budget covers every block (test_engine.cpp:48-67);
//   4. the hybrid-query residual recompute_layer_attention (harness.hpp:318-329)
//      of every (step, layer) of the GPU run, within 1e-3.
// f32 KV on the device: selections are bit-exact (the f64 scoring path),
// attention within 1e-3.
#include <cmath>
#include <cstdio>
#include <string>

#include "scout_b200.hpp"
#include "scout/engine.hpp"
#include "engine_b200.hpp"  // generated: scout::dropin::ScoutEngine
#ifdef SCOUT_REF_HARNESS
#include "scout/harness.hpp"
#endif

static int g_fail = 0, g_pass = 0;
#define CHECK(cond, ...)                                       \
    do {                                                       \
        if (cond) {                                            \
            ++g_pass;                                          \
        } else {                                               \
            ++g_fail;                                          \
            std::printf("FAIL %s:%d: ", __FILE__, __LINE__);   \
            std::printf(__VA_ARGS__);                          \
            std::printf("\n");                                 \
        }                                                      \
    } while (0)

static double max_abs_diff(const scout::Vec& a, const scout::Vec& b) {
    if (a.size() != b.size()) return 1e300;
    double m = 0.0;
    for (size_t i = 0; i < a.size(); ++i) m = std::max(m, std::abs(a[i] - b[i]));
    return m;
}

static scout::ToyDecoderConfig toy(size_t layers, size_t hidden, size_t head_dim, size_t block, double alpha,
                                   uint64_t seed) {
    scout::ToyDecoderConfig c;
    c.layers = layers;
    c.hidden = hidden;
    c.head_dim = head_dim;
    c.block_size = block;
    c.alpha = alpha;
    c.seed = seed;
    return c;
}

// The patched engine lives in scout::dropin with its own copies of the
// engine.hpp types (EngineConfig, StepResult, ...): same fields, so the
// drivers below are templates over them.
template <class EC>
static EC engine_config(size_t k, std::vector<size_t> intervals = {}, bool serial = true) {
    EC c;
    c.k_blocks = k;
    c.recall_intervals = std::move(intervals);
    c.deterministic_serial = serial;
    return c;
}

template <class Engine>
static auto run(const scout::ToyDecoder& dec, Engine& eng, size_t prefill, size_t steps) {
    eng.prefill(dec.make_embeddings(prefill));
    std::vector<decltype(eng.decode_step(scout::Vec{}, 1))> out;
    scout::Vec x = dec.next_input(eng.trace().final_hidden);
    for (size_t s = 1; s <= steps; ++s) {
        out.push_back(eng.decode_step(x, s));
        x = dec.next_input(out.back().final_hidden);
    }
    return out;
}

// 1. frozen stream: selections exact against a monolithic cache, outputs
// against the single-device oracle
static void frozen_stream() {
    const auto cfg = toy(3, 20, 10, 4, 0.0, 22);
    const scout::ToyDecoder dec(cfg);
    const auto ecfg = engine_config<scout::dropin::EngineConfig>(2);
    scout::dropin::ScoutEngine eng(dec, ecfg);
    const auto res = run(dec, eng, 16, 8);
    scout::TieredKvCache cache(cfg.layers, cfg.block_size, cfg.head_dim, scout::DigestMethod::minmax, 1000);
    scout::ResidualTrace trace = dec.prefill(dec.make_embeddings(16), cache);
    scout::Vec x = dec.next_input(trace.final_hidden);
    double worst = 0.0;
    for (size_t s = 0; s < res.size(); ++s) {
        scout::Vec cur = x;
        for (size_t i = 0; i < cfg.layers; ++i) {
            const scout::Vec n = dec.normalize(cur);
            const scout::Vec q = dec.query(i, n);
            const scout::BlockIdSet picked = scout::select_topk(q, cache.digests(i), ecfg.k_blocks);
            const auto& lm = res[s].layers[i];
            CHECK(lm.predicted == picked, "frozen stream: step %zu layer %zu selection", s, i);
            const scout::Vec attn = scout::reference_block_sparse(cache, i, q, ecfg.k_blocks, dec.scale());
            worst = std::max(worst, max_abs_diff(lm.attn_out, attn));
            scout::Vec y = scout::ToyDecoder::add_scaled(cur, dec.apply_output(i, attn), cfg.alpha);
            y = scout::ToyDecoder::add_scaled(y, dec.ffn(i, dec.normalize(y)), cfg.alpha);
            cache.append_token(i, dec.key(i, n), dec.value(i, n));
            cur = y;
        }
        x = dec.next_input(cur);
    }
    CHECK(worst < 1e-3, "frozen stream: attention max |diff| %.3g", worst);
    std::printf("frozen stream: %zu steps, attention max |diff| vs reference_block_sparse %.3g\n", res.size(), worst);
}

// 2. side by side with the unmodified reference engine
static void side_by_side(const char* name, const scout::ToyDecoderConfig& cfg, size_t k, std::vector<size_t> intervals,
                         size_t prefill, size_t steps, bool serial) {
    const scout::ToyDecoder dec(cfg);
    scout::ScoutEngine ref(dec, engine_config<scout::EngineConfig>(k, intervals, serial));
    scout::dropin::ScoutEngine gpu(dec, engine_config<scout::dropin::EngineConfig>(k, intervals, serial));
    const auto a = run(dec, ref, prefill, steps);
    const auto b = run(dec, gpu, prefill, steps);
    double worst = 0.0, worst_hidden = 0.0;
    size_t cpu_tokens = 0, recalls = 0;
    for (size_t s = 0; s < steps; ++s) {
        worst_hidden = std::max(worst_hidden, max_abs_diff(a[s].final_hidden, b[s].final_hidden));
        for (size_t i = 0; i < cfg.layers; ++i) {
            const auto& x = a[s].layers[i];
            const auto& y = b[s].layers[i];
            CHECK(x.predicted == y.predicted && x.resident_set == y.resident_set && x.cpu_set == y.cpu_set,
                  "%s: step %zu layer %zu sets differ", name, s, i);
            CHECK(x.cpu_tokens == y.cpu_tokens && x.resident_tokens == y.resident_tokens,
                  "%s: step %zu layer %zu token accounting differs", name, s, i);
            worst = std::max(worst, max_abs_diff(x.attn_out, y.attn_out));
            cpu_tokens += y.cpu_tokens;
            recalls += y.recalled_blocks;
        }
    }
    const auto& ea = ref.events();
    const auto& eb = gpu.events();
    bool same = ea.size() == eb.size();
    for (size_t e = 0; same && e < ea.size(); ++e)
        same = static_cast<int>(ea[e].kind) == static_cast<int>(eb[e].kind) && ea[e].step == eb[e].step &&
               ea[e].layer == eb[e].layer &&
               ea[e].ids == eb[e].ids;
    CHECK(same, "%s: event logs differ", name);
    CHECK(worst < 1e-3 && worst_hidden < 1e-3, "%s: attention %.3g, hidden %.3g", name, worst, worst_hidden);
    std::printf("%s: %zu steps x %zu layers, identical sets and %zu events, attention max |diff| %.3g, hidden %.3g "
                "(%zu CPU-side tokens, %zu recalled blocks)\n",
                name, steps, cfg.layers, eb.size(), worst, worst_hidden, cpu_tokens, recalls);
#ifdef SCOUT_REF_HARNESS
    // 4. the reference's hybrid-query residual of the GPU run
    double resid = 0.0;
    for (const auto& sr : b)
        for (const auto& m : sr.layers) {
            scout::LayerMetrics lm;  // the reference's type, for its oracle
            lm.layer = m.layer;
            lm.resident_set = m.resident_set;
            lm.cpu_set = m.cpu_set;
            lm.q_true = m.q_true;
            lm.q_pred = m.q_pred;
            lm.attn_out = m.attn_out;
            lm.tokens_at_attention = m.tokens_at_attention;
            resid = std::max(resid, max_abs_diff(scout::recompute_layer_attention(gpu.cache(), dec.scale(), lm), m.attn_out));
        }
    CHECK(resid < 1e-3, "%s: recompute_layer_attention residual %.3g", name, resid);
    std::printf("%s: recompute_layer_attention max residual %.3g\n", name, resid);
#endif
}

// 3. budget covering every block: exact attention
static void exact_when_k_covers() {
    const auto cfg = toy(3, 20, 10, 4, 0.1, 21);
    const scout::ToyDecoder dec(cfg);
    scout::dropin::ScoutEngine eng(dec, engine_config<scout::dropin::EngineConfig>(64));
    const auto res = run(dec, eng, 8, 16);
    scout::TieredKvCache cache(cfg.layers, cfg.block_size, cfg.head_dim, scout::DigestMethod::minmax, 1000);
    scout::ResidualTrace trace = dec.prefill(dec.make_embeddings(8), cache);
    scout::Vec x = dec.next_input(trace.final_hidden);
    double worst = 0.0;
    for (size_t s = 0; s < res.size(); ++s) {
        const scout::Vec out = dec.decode_exact_step(cache, trace, x);
        worst = std::max(worst, max_abs_diff(res[s].final_hidden, out));
        x = dec.next_input(out);
    }
    CHECK(worst < 1e-3, "exact when k covers: %.3g", worst);
    std::printf("k covers every block: final hidden max |diff| vs decode_exact_step %.3g\n", worst);
}

int main() {
    try {
        frozen_stream();
        exact_when_k_covers();
        side_by_side("reference tests' geometry, serial", toy(3, 20, 10, 4, 0.1, 23), 3, {2, 2, 2}, 16, 10, true);
        side_by_side("reference tests' geometry, threaded worker", toy(3, 20, 10, 4, 0.1, 23), 3, {2, 2, 2}, 16, 10,
                     false);
        side_by_side("recall every step", toy(3, 20, 10, 4, 0.1, 27), 2, {1, 1, 1}, 16, 8, true);
        side_by_side("GPU geometry (head_dim 128, block 64)", toy(2, 256, 128, 64, 0.1, 31), 3, {2, 3}, 64 * 5 + 7, 6,
                     true);
    } catch (const std::exception& e) {
        std::printf("FAIL exception: %s\n", e.what());
        return 1;
    }
    std::printf("%d checks passed, %d failed\n", g_pass, g_fail);
    if (g_fail == 0) std::printf("ALL PASS\n");
    return g_fail == 0 ? 0 : 1;
}
