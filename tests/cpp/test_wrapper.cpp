// The reference's own unit-test cases (proj/tests/test_digest.cpp,
// test_attention.cpp), restated against the header-only GPU drop-in
// include/scout_b200.hpp. Each CHECK names the reference case it mirrors.
#include <cstdio>
#include <random>
#include <stdexcept>

#include "scout_b200.hpp"

namespace sb = scout_b200;
static int g_fail = 0, g_pass = 0;
#define CHECK(cond, what)                                                         \
    do {                                                                          \
        if (cond) ++g_pass;                                                       \
        else { ++g_fail; std::printf("FAIL %s (%s:%d)\n", what, __FILE__, __LINE__); } \
    } while (0)
template <class F>
static bool throws_invalid(F f) {
    try { f(); } catch (const std::invalid_argument&) { return true; } catch (...) { return false; }
    return false;
}

static sb::Mat mat(std::initializer_list<sb::Vec> rows) {
    sb::Mat m(rows.size(), rows.begin()->size());
    std::size_t r = 0;
    for (const auto& v : rows) { for (std::size_t c = 0; c < v.size(); ++c) m.data[r * m.cols + c] = v[c]; ++r; }
    return m;
}
// f32-representable N(0,1) values (the GPU cache stores f32 / bf16)
static double rnd(std::mt19937_64& g) { std::normal_distribution<double> d(0, 1); return static_cast<float>(d(g)); }
static double host_score(const sb::Vec& q, const sb::BlockDigest& d) {  // digest.hpp:62-72, restated
    double s = 0.0;
    for (std::size_t c = 0; c < q.size(); ++c) {
        if (d.method == sb::DigestMethod::minmax) { const double a = q[c] * d.lo[c], b = q[c] * d.hi[c]; s += (a < b) ? b : a; }
        else s += q[c] * d.mean[c];
    }
    return s;
}

int main() {
    // test_digest.cpp:35-44 — minmax digest tracks channel-wise bounds
    {
        const sb::BlockDigest d = sb::build_digest(mat({{0.0, 1.0}, {3.0, -2.0}, {1.0, 0.5}}), sb::DigestMethod::minmax, 4, 2);
        CHECK(d.lo == (sb::Vec{0.0, -2.0}) && d.hi == (sb::Vec{3.0, 1.0}), "minmax digest bounds");
        CHECK(d.block_id == 4 && d.layer == 2, "digest ids");
        CHECK(throws_invalid([] { sb::build_digest(sb::Mat(0, 2), sb::DigestMethod::minmax); }), "empty block throws");
    }
    // test_digest.cpp:46-55 — minmax score hand-worked example (= 5)
    {
        sb::BlockDigest d;
        d.lo = {0.0, -2.0};
        d.hi = {3.0, 1.0};
        CHECK(sb::digest_score(sb::Vec{1.0, -1.0}, d) == 5.0, "minmax score KAT");
        CHECK(throws_invalid([&] { sb::digest_score(sb::Vec{1.0, -1.0, 0.0}, d); }), "score dim mismatch throws");
    }
    // test_digest.cpp:57-62 — mean digest
    {
        const sb::BlockDigest d = sb::build_digest(mat({{2.0, 4.0}, {0.0, -2.0}}), sb::DigestMethod::mean);
        CHECK(d.mean == (sb::Vec{1.0, 1.0}), "mean digest");
        CHECK(sb::digest_score(sb::Vec{0.5, 2.0}, d) == 2.5, "mean score KAT");
    }
    // test_digest.cpp:64-82 — minmax score upper-bounds every row's dot product
    {
        std::mt19937_64 g(17);
        bool ok = true;
        for (int trial = 0; trial < 60; ++trial) {
            const std::size_t rows = 1 + g() % 12;
            sb::Mat keys(rows, 6);
            for (double& v : keys.data) v = rnd(g);
            const sb::BlockDigest d = sb::build_digest(keys, sb::DigestMethod::minmax);
            sb::Vec q(6);
            for (double& v : q) v = rnd(g);
            const double bound = sb::digest_score(q, d);
            for (std::size_t r = 0; r < rows; ++r) {
                double s = 0;
                for (int c = 0; c < 6; ++c) s += q[c] * keys.row(r)[c];
                ok = ok && s <= bound + 1e-12;
            }
        }
        CHECK(ok, "minmax upper bound");
    }
    // test_digest.cpp:84-105 — select_topk hand-worked examples
    {
        std::vector<sb::BlockDigest> ds(3);
        for (std::size_t i = 0; i < 3; ++i) { ds[i].method = sb::DigestMethod::mean; ds[i].block_id = i; }
        ds[0].mean = {5.0}; ds[1].mean = {1.0}; ds[2].mean = {3.0};
        CHECK(sb::select_topk(sb::Vec{1.0}, ds, 2) == (sb::BlockIdSet{0, 2}), "topk {0,2}");
        CHECK(sb::select_topk(sb::Vec{1.0}, ds, 10) == (sb::BlockIdSet{0, 1, 2}), "topk k > n");
        ds[0].mean = {2.0}; ds[1].mean = {2.0}; ds[2].mean = {1.0};
        CHECK(sb::select_topk(sb::Vec{1.0}, ds, 1) == (sb::BlockIdSet{0}), "tie -> lower id");
        CHECK(sb::select_topk(sb::Vec{1.0}, ds, 2) == (sb::BlockIdSet{0, 1}), "tie k=2");
        CHECK(throws_invalid([&] { sb::select_topk(sb::Vec{1.0}, ds, 0); }), "k = 0 throws");
    }
    // test_digest.cpp:107-127 — select_topk equals brute force, ties included
    {
        std::mt19937_64 g(23);
        std::normal_distribution<double> dist(0.0, 1.0);
        std::uniform_int_distribution<int> coarse(-2, 2);
        bool ok = true;
        for (int trial = 0; trial < 300; ++trial) {
            const std::size_t n = 1 + g() % 20;
            const bool tie = trial % 2 == 0;
            std::vector<sb::BlockDigest> ds(n);
            for (std::size_t i = 0; i < n; ++i) {
                ds[i].method = (trial % 3 == 0) ? sb::DigestMethod::minmax : sb::DigestMethod::mean;
                ds[i].block_id = i;
                auto draw = [&] { return tie ? static_cast<double>(coarse(g)) : dist(g); };
                if (ds[i].method == sb::DigestMethod::mean) ds[i].mean = {draw(), draw(), draw()};
                else {
                    ds[i].lo = {draw(), draw(), draw()};
                    ds[i].hi = ds[i].lo;
                    for (double& v : ds[i].hi) v += tie ? coarse(g) + 2 : std::abs(dist(g));
                }
            }
            sb::Vec q(3);
            for (double& v : q) v = tie ? 1.0 : dist(g);
            const std::size_t k = 1 + g() % n;
            std::vector<std::pair<double, std::size_t>> sc;
            for (const auto& d : ds) sc.emplace_back(host_score(q, d), d.block_id);
            std::stable_sort(sc.begin(), sc.end(), [](const auto& a, const auto& b) {
                if (a.first != b.first) return a.first > b.first;
                return a.second < b.second;
            });
            sb::BlockIdSet want;
            for (std::size_t i = 0; i < std::min(k, sc.size()); ++i) want.push_back(sc[i].second);
            std::sort(want.begin(), want.end());
            ok = ok && sb::select_topk(q, ds, k) == want;
        }
        CHECK(ok, "topk == brute force (300 cases, half tie-prone)");
    }
    // test_digest.cpp:129-139 — scores below the k-th never change the selection
    {
        std::vector<sb::BlockDigest> ds(5);
        for (std::size_t i = 0; i < 5; ++i) { ds[i].method = sb::DigestMethod::mean; ds[i].block_id = i; ds[i].mean = {10.0 - i}; }
        const auto before = sb::select_topk(sb::Vec{1.0}, ds, 3);
        ds[4].mean = {1.0};
        CHECK(sb::select_topk(sb::Vec{1.0}, ds, 3) == before, "sub-k-th invariance");
    }
    // test_attention.cpp:81-107 / acceptance crit 1 — any partition merges to the same attention
    {
        std::mt19937_64 g(37);
        const std::size_t dim = 5;
        std::vector<sb::KvBlock> blocks(6);
        std::vector<double> K, V;
        for (std::size_t i = 0; i < 6; ++i) {
            const std::size_t rows = 1 + g() % 7;
            blocks[i].keys = sb::Mat(rows, dim);
            blocks[i].values = sb::Mat(rows, dim);
            for (double& v : blocks[i].keys.data) v = rnd(g);
            for (double& v : blocks[i].values.data) v = rnd(g);
            K.insert(K.end(), blocks[i].keys.data.begin(), blocks[i].keys.data.end());
            V.insert(V.end(), blocks[i].values.data.begin(), blocks[i].values.data.end());
        }
        sb::Vec q(dim);
        for (double& v : q) v = rnd(g);
        // softmax composition reference (test_attention.cpp:26-36), restated
        const std::size_t n = K.size() / dim;
        std::vector<double> lg(n);
        double mx = -1e300;
        for (std::size_t r = 0; r < n; ++r) { double s = 0; for (std::size_t c = 0; c < dim; ++c) s += q[c] * K[r * dim + c]; lg[r] = 0.5 * s; mx = std::max(mx, lg[r]); }
        double den = 0;
        sb::Vec whole(dim, 0.0);
        for (std::size_t r = 0; r < n; ++r) { const double w = std::exp(lg[r] - mx); den += w; for (std::size_t c = 0; c < dim; ++c) whole[c] += w * V[r * dim + c]; }
        for (double& v : whole) v /= den;
        double worst = 0;
        bool counts = true;
        for (int trial = 0; trial < 20; ++trial) {
            std::vector<const sb::KvBlock*> left, right;
            for (const auto& b : blocks) (g() % 2 ? left : right).push_back(&b);
            const auto m = sb::merge(sb::partial_attention(q, left, 0.5), sb::partial_attention(q, right, 0.5));
            counts = counts && m.token_count == n;
            const auto o = sb::finalize(m);
            for (std::size_t c = 0; c < dim; ++c) worst = std::max(worst, std::abs(o[c] - whole[c]));
        }
        CHECK(counts, "merged token count");
        CHECK(worst < 1e-3, "partition invariance within the f32 tolerance (1e-3)");
    }
    // test_attention.cpp:109-128 — merge commutative / associative
    {
        std::mt19937_64 g(41);
        sb::KvBlock b[3];
        const std::size_t rows[3] = {3, 5, 2};
        for (int i = 0; i < 3; ++i) {
            b[i].keys = sb::Mat(rows[i], 4);
            b[i].values = sb::Mat(rows[i], 4);
            for (double& v : b[i].keys.data) v = rnd(g);
            for (double& v : b[i].values.data) v = rnd(g);
        }
        sb::Vec q(4);
        for (double& v : q) v = rnd(g);
        auto part = [&](int i) { return sb::partial_attention(q, std::vector<const sb::KvBlock*>{&b[i]}, 0.5); };
        const auto p0 = part(0), p1 = part(1), p2 = part(2);
        const auto ab = sb::finalize(sb::merge(p0, p1)), ba = sb::finalize(sb::merge(p1, p0));
        const auto l = sb::finalize(sb::merge(sb::merge(p0, p1), p2)), r = sb::finalize(sb::merge(p0, sb::merge(p1, p2)));
        double e1 = 0, e2 = 0;
        for (int c = 0; c < 4; ++c) { e1 = std::max(e1, std::abs(ab[c] - ba[c])); e2 = std::max(e2, std::abs(l[c] - r[c])); }
        CHECK(e1 < 1e-5 && e2 < 1e-5, "merge commutative / associative");
    }
    // test_attention.cpp:130-154 — empty partials
    {
        std::mt19937_64 g(43);
        sb::KvBlock b;
        b.keys = sb::Mat(4, 3);
        b.values = sb::Mat(4, 3);
        for (double& v : b.keys.data) v = rnd(g);
        for (double& v : b.values.data) v = rnd(g);
        sb::Vec q(3);
        for (double& v : q) v = rnd(g);
        const sb::PartialAttention p = sb::partial_attention(q, std::vector<const sb::KvBlock*>{&b}, 1.0);
        const auto e = sb::PartialAttention::empty(3);
        const auto m1 = sb::merge(p, e), m2 = sb::merge(e, p);
        CHECK(m1.o_acc == p.o_acc && m1.denom == p.denom && m1.max_logit == p.max_logit && m2.o_acc == p.o_acc,
              "empty partial is an exact identity");
        const auto both = sb::merge(e, sb::PartialAttention::empty(3));
        CHECK(both.is_empty(), "empty + empty is empty");
        CHECK(throws_invalid([&] { sb::finalize(both); }), "finalize(empty) throws");
        const auto none = sb::partial_attention(sb::Vec{1.0, 2.0}, std::vector<const sb::KvBlock*>{}, 1.0);
        CHECK(none.is_empty() && none.token_count == 0, "partial over no blocks is empty");
        CHECK(throws_invalid([&] { sb::partial_attention(q, std::vector<const sb::KvBlock*>{&b}, 0.0); }),
              "scale <= 0 throws");
    }
    std::printf("%s: %d passed, %d failed\n", g_fail ? "FAILED" : "ALL PASS", g_pass, g_fail);
    return g_fail ? 1 : 0;
}
