// The C++ drop-in TieredKvCache (include/scout_b200_tier.hpp: the tier state
// machine on the B200, K5) side by side with the reference's own
// scout::TieredKvCache (kv_store.hpp, compiled from /root/reference), both
// driven with the same operations and compared after every one: the tier,
// last_selected mark and in-flight flag of every block, residency_set of every
// layer, the sealed ids append_token returns, the tickets begin_layer applies,
// the blocks fetch_blocks hands out and which calls throw. The drop-in is
// instantiated on the reference's own types (scout::KvBlock, BlockDigest,
// RecallTicket, Tier), so its results are the reference's structs.
//   * the reference's test_kv_store.cpp scenarios at block size 64
//     (LRU eviction with the id tie-break, the open block outside capacity,
//     recall visibility at (m+1, i), rejected recalls, place_after_prefill,
//     demote_block, fetch_blocks on the wrong tier);
//   * random sequences (3 layers, layer 0 pinned, appends that seal and
//     evict, marks, recalls incl. rejected tickets, begin_layer over 10 steps).
#include <cstdio>
#include <functional>
#include <random>
#include <string>

#include "scout_b200_tier.hpp"
#include "scout/kv_store.hpp"

using Ref = scout::TieredKvCache;
using Dev = scout_b200::TieredKvCacheT<scout::KvBlock, scout::BlockDigest, scout::RecallTicket, scout::Tier,
                                       scout::DigestMethod, scout::Mat>;

static int g_fail = 0, g_pass = 0;
#define CHECK(cond, ...)                                     \
    do {                                                     \
        if (cond) {                                          \
            ++g_pass;                                        \
        } else {                                             \
            ++g_fail;                                        \
            std::printf("FAIL %s:%d: ", __FILE__, __LINE__); \
            std::printf(__VA_ARGS__);                        \
            std::printf("\n");                               \
        }                                                    \
    } while (0)

static constexpr std::size_t BS = 64, HD = 8;

static void compare(const Ref& r, const Dev& d, const char* where) {
    for (std::size_t l = 0; l < r.num_layers(); ++l) {
        CHECK(r.block_count(l) == d.block_count(l) && r.total_tokens(l) == d.total_tokens(l), "%s: layer %zu shape",
              where, l);
        for (std::size_t id = 0; id < r.block_count(l); ++id) {
            CHECK(r.tier_of(l, id) == d.tier_of(l, id), "%s: layer %zu block %zu tier", where, l, id);
            CHECK(r.last_selected(l, id) == d.last_selected(l, id), "%s: layer %zu block %zu last_selected %zu vs %zu",
                  where, l, id, r.last_selected(l, id), d.last_selected(l, id));
            CHECK(r.is_in_flight(l, id) == d.is_in_flight(l, id), "%s: layer %zu block %zu in flight", where, l, id);
        }
        CHECK(r.residency_set(l) == d.residency_set(l), "%s: layer %zu residency_set", where, l);
        CHECK(r.sealed_fast_count(l) == d.sealed_fast_count(l), "%s: layer %zu sealed_fast_count", where, l);
        const auto& rd = r.digests(l);
        const auto& dd = d.digests(l);
        bool same = rd.size() == dd.size();
        for (std::size_t i = 0; same && i < rd.size(); ++i) same = rd[i].lo == dd[i].lo && rd[i].hi == dd[i].hi;
        CHECK(same, "%s: layer %zu digests", where, l);
    }
    CHECK(r.clock() == d.clock(), "%s: clock", where);
}

// run fn on both; both must throw std::invalid_argument or neither
template <class F, class G>
static void both(F&& fr, G&& fd, const char* what) {
    bool tr = false, td = false;
    try {
        fr();
    } catch (const std::invalid_argument&) {
        tr = true;
    }
    try {
        fd();
    } catch (const std::invalid_argument&) {
        td = true;
    }
    CHECK(tr == td, "%s: reference threw %d, drop-in threw %d", what, tr, td);
}

static void append_both(Ref& r, Dev& d, std::size_t layer, std::mt19937& rng) {
    std::normal_distribution<double> n;
    scout::Vec k(HD), v(HD);
    for (auto& x : k) x = n(rng);
    for (auto& x : v) x = n(rng);
    const auto a = r.append_token(layer, k, v);
    const auto b = d.append_token(layer, k, v);
    CHECK(a == b, "append_token sealed id (layer %zu)", layer);
}

static bool same_tickets(const std::vector<scout::RecallTicket>& a, const std::vector<scout::RecallTicket>& b) {
    if (a.size() != b.size()) return false;
    for (std::size_t i = 0; i < a.size(); ++i)
        if (a[i].layer != b[i].layer || a[i].ids != b[i].ids || a[i].ready_step != b[i].ready_step ||
            a[i].ready_layer != b[i].ready_layer)
            return false;
    return true;
}

static void scenarios() {
    std::mt19937 rng(3);
    // test_kv_store.cpp:47-75: eviction by last_selected, ties -> lower id; the open block is outside capacity
    {
        Ref r(2, BS, HD, scout::DigestMethod::minmax, 2);
        Dev d(2, BS, HD, scout::DigestMethod::minmax, 2, 64);
        for (std::size_t i = 0; i < 3 * BS; ++i) append_both(r, d, 0, rng);
        compare(r, d, "three sealed blocks, capacity 2");
        CHECK(d.tier_of(0, 0) == scout::Tier::slow && d.tier_of(0, 2) == scout::Tier::fast, "LRU tie -> block 0");
        r.mark_selected(0, {1}, 5);
        d.mark_selected(0, {1}, 5);
        r.begin_layer(6, 0);
        d.begin_layer(6, 0);
        for (std::size_t i = 0; i < BS + 5; ++i) append_both(r, d, 0, rng);  // seals block 3, opens block 4
        compare(r, d, "mark protects block 1");
        // recall visibility (test_kv_store.cpp:76-108): issued at (6, 0), ready at (7, 0)
        const scout::BlockIdSet slow = {0};
        both([&] { r.schedule_recall(0, slow, 6, 0); }, [&] { d.schedule_recall(0, slow, 6, 0); }, "recall block 0");
        compare(r, d, "in flight");
        auto rs = d.residency_set(0);  // clock (6, 0): layer 0 runs next at (6, 0), before the arrival
        CHECK(std::find(rs.begin(), rs.end(), 0) == rs.end(), "planning view at (6, 0) excludes the arriving block");
        both([&] { r.fetch_blocks(0, {0}, scout::Tier::fast); }, [&] { d.fetch_blocks(0, {0}, scout::Tier::fast); },
             "fetch an in-flight block from the fast tier");
        CHECK(same_tickets(r.begin_layer(6, 1), d.begin_layer(6, 1)), "nothing due at (6, 1)");
        compare(r, d, "(6, 1)");
        rs = d.residency_set(0);  // layer 0 runs next at (7, 0): the block arrives by then
        CHECK(std::find(rs.begin(), rs.end(), 0) != rs.end(), "planning view at (6, 1) includes the arriving block");
        r.mark_selected(0, {0}, 7);  // selected again: the recalled block survives the eviction at arrival
        d.mark_selected(0, {0}, 7);
        const auto ta = r.begin_layer(7, 0);
        const auto tb = d.begin_layer(7, 0);
        CHECK(same_tickets(ta, tb) && ta.size() == 1, "applied at (7, 0)");
        compare(r, d, "(7, 0)");
        CHECK(r.tier_of(0, 0) == scout::Tier::fast, "block 0 arrived");
        const auto fb = d.fetch_blocks(0, {0}, scout::Tier::fast);
        CHECK(fb.size() == 1 && fb[0]->keys.data == r.block(0, 0).keys.data, "fetch_blocks hands out the rows");
        // rejected tickets change nothing
        both([&] { r.schedule_recall(0, {2}, 7, 0); }, [&] { d.schedule_recall(0, {2}, 7, 0); }, "recall a fast block");
        both([&] { r.schedule_recall(0, {4}, 7, 0); }, [&] { d.schedule_recall(0, {4}, 7, 0); }, "recall the open block");
        both([&] { r.schedule_recall(0, {}, 7, 0); }, [&] { d.schedule_recall(0, {}, 7, 0); }, "empty ticket");
        both([&] { r.schedule_recall(0, {99}, 7, 0); }, [&] { d.schedule_recall(0, {99}, 7, 0); }, "id out of range");
        compare(r, d, "after rejected tickets");
        // demote_block (kv_store.hpp:257-265)
        both([&] { r.demote_block(0, 4); }, [&] { d.demote_block(0, 4); }, "demote the open block");
        both([&] { r.demote_block(0, 2); }, [&] { d.demote_block(0, 2); }, "demote block 2");
        both([&] { r.demote_block(0, 2); }, [&] { d.demote_block(0, 2); }, "demote a slow block");
        compare(r, d, "after demote");
    }
    // place_after_prefill (kv_store.hpp:268-279) with the pinned layer untouched
    {
        Ref r(2, BS, HD, scout::DigestMethod::minmax, 3);
        Dev d(2, BS, HD, scout::DigestMethod::minmax, 3, 64);
        r.pin_layer(0);
        d.pin_layer(0);
        for (std::size_t l = 0; l < 2; ++l)
            for (std::size_t i = 0; i < 9 * BS + 17; ++i) append_both(r, d, l, rng);
        compare(r, d, "prefill");
        std::normal_distribution<double> n;
        scout::Vec q(HD);
        for (auto& x : q) x = n(rng);
        for (std::size_t l = 0; l < 2; ++l) {
            r.place_after_prefill(l, q);
            d.place_after_prefill(l, q);
        }
        compare(r, d, "place_after_prefill");
    }
}

static void random_sequence(unsigned seed) {
    std::mt19937 rng(seed);
    const std::size_t L = 3, cap = 4;
    Ref r(L, BS, HD, scout::DigestMethod::minmax, cap);
    Dev d(L, BS, HD, scout::DigestMethod::minmax, cap, 128);
    r.pin_layer(0);
    d.pin_layer(0);
    for (std::size_t l = 0; l < L; ++l)
        for (std::size_t i = 0; i < 5 * BS + 10; ++i) append_both(r, d, l, rng);
    compare(r, d, "prefill");
    std::uniform_real_distribution<double> u01;
    for (std::size_t step = 1; step <= 10; ++step) {
        for (std::size_t layer = 0; layer < L; ++layer) {
            CHECK(same_tickets(r.begin_layer(step, layer), d.begin_layer(step, layer)), "begin_layer(%zu, %zu)", step,
                  layer);
            compare(r, d, "begin_layer");
            const std::size_t tgt = (layer + 1) % L;
            const std::size_t nb = r.block_count(tgt);
            scout::BlockIdSet marks;
            for (std::size_t b = 0; b < nb; ++b)
                if (u01(rng) < 3.0 / static_cast<double>(nb)) marks.push_back(b);
            r.mark_selected(tgt, marks, step);
            d.mark_selected(tgt, marks, step);
            const int appends = 1 + static_cast<int>(u01(rng) * 40);
            for (int i = 0; i < appends; ++i) append_both(r, d, layer, rng);
            compare(r, d, "append");
            scout::BlockIdSet cand, pick;
            for (std::size_t b = 0; b < r.block_count(layer); ++b)
                if (r.tier_of(layer, b) == scout::Tier::slow && !r.is_in_flight(layer, b) && r.block(layer, b).sealed)
                    cand.push_back(b);
            std::shuffle(cand.begin(), cand.end(), rng);
            const std::size_t n = std::min<std::size_t>(cand.size(), static_cast<std::size_t>(u01(rng) * 4));
            pick.assign(cand.begin(), cand.begin() + static_cast<std::ptrdiff_t>(n));
            if (!pick.empty() && u01(rng) < 0.2)
                for (std::size_t b = 0; b < r.block_count(layer); ++b)
                    if (r.tier_of(layer, b) == scout::Tier::fast) {
                        pick.push_back(b);  // a fast id: the whole ticket is rejected
                        break;
                    }
            std::sort(pick.begin(), pick.end());
            pick.erase(std::unique(pick.begin(), pick.end()), pick.end());
            if (!pick.empty())
                both([&] { r.schedule_recall(layer, pick, step, layer); },
                     [&] { d.schedule_recall(layer, pick, step, layer); }, "schedule_recall");
            compare(r, d, "schedule_recall");
            // the split the engine makes (engine.hpp:239-247): fetch both sides
            const auto res = r.residency_set(layer);
            scout::BlockIdSet fast, slow;
            for (std::size_t b = 0; b < r.block_count(layer); ++b)
                (r.tier_of(layer, b) == scout::Tier::fast ? fast : slow).push_back(b);
            const auto fr = r.fetch_blocks(layer, fast, scout::Tier::fast);
            const auto fd = d.fetch_blocks(layer, fast, scout::Tier::fast);
            bool same = fr.size() == fd.size();
            for (std::size_t i = 0; same && i < fr.size(); ++i) same = fr[i]->keys.data == fd[i]->keys.data;
            CHECK(same, "fetch_blocks fast contents");
            both([&] { r.fetch_blocks(layer, slow, scout::Tier::fast); },
                 [&] { d.fetch_blocks(layer, slow, scout::Tier::fast); }, "fetch slow blocks as fast");
            (void)res;
        }
    }
}

// the default instantiation on scout_b200's own mirror types
static void mirror_types() {
    scout_b200::TieredKvCache m(1, BS, HD, scout_b200::DigestMethod::minmax, 2, 64);
    std::mt19937 rng(5);
    std::normal_distribution<double> n;
    std::optional<std::size_t> last;
    for (std::size_t i = 0; i < 3 * BS; ++i) {
        scout_b200::Vec k(HD), v(HD);
        for (auto& x : k) x = n(rng);
        for (auto& x : v) x = n(rng);
        last = m.append_token(0, k, v);
    }
    CHECK(last && *last == 2, "mirror types: third block sealed");
    CHECK(m.tier_of(0, 0) == scout_b200::Tier::slow && m.tier_of(0, 1) == scout_b200::Tier::fast,
          "mirror types: LRU eviction");
    const auto t = m.schedule_recall(0, {0}, 1, 0);
    CHECK(t.ready_step == 2 && m.is_in_flight(0, 0), "mirror types: ticket");
}

int main() {
    mirror_types();
    scenarios();
    for (unsigned s = 0; s < 3; ++s) random_sequence(11 + s);
    std::printf("%d checks passed, %d failed\n", g_pass, g_fail);
    if (g_fail == 0) std::printf("ALL PASS\n");
    return g_fail == 0 ? 0 : 1;
}
