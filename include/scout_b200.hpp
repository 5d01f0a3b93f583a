// scout_b200.hpp — header-only C++ drop-in for the reference's hot-path API,
// running on the B200 through the C ABI (scout_b200.h).
//
// Restated reference signatures (reference proj/include/scout/):
//   BlockDigest      build_digest(const Mat&, DigestMethod, block_id, layer)  digest.hpp:34
//   double           digest_score(const Vec&, const BlockDigest&)              digest.hpp:62
//   BlockIdSet       select_topk(const Vec&, const vector<BlockDigest>&, k)    digest.hpp:101
//   PartialAttention partial_attention(const Vec&, span<const KvBlock*>, s)   attention.hpp:73 / :91
//   PartialAttention merge(const PartialAttention&, const PartialAttention&)   attention.hpp:100
//   Vec              finalize(const PartialAttention&)                         attention.hpp:117
//
// The functions are templates over the argument types, so they take the
// reference's own scout:: structs unchanged (any type with the same member
// names works), and their results convert to them (PartialResult,
// DigestResult): the reference's ScoutEngine compiles with its hot-path call
// sites swapped to scout_b200:: and nothing else changed (INTEGRATION.md §1,
// proven by tests/cpp/test_dropin_engine.cpp); scout_b200::* mirror types are
// provided for code that does not include the reference headers. Error behaviour follows the reference:
// std::invalid_argument for argument errors (k == 0, scale <= 0, empty block,
// dimension mismatch), std::runtime_error for device failures.
//
// Numerics: select_topk / digest_score run the exact f64 path
// (bit-identical to the reference for any doubles); build_digest,
// partial_attention and merge run on f32 KV (exact for min/max of
// f32-representable keys; attention within 1e-3 max-abs), which is the GPU
// cache's storage precision. Head dimension <= 128 (zero padded), block rows
// <= 64. Per-call device buffers: this is the compatibility API; the batched
// entry points (scout_score_topk_split / scout_sparse_decode / scout_engine_*)
// are the performance path.
#pragma once

#include <cuda_runtime.h>

#include <algorithm>
#include <cmath>
#include <cstddef>
#include <cstdint>
#include <limits>
#include <numeric>
#include <span>
#include <stdexcept>
#include <string>
#include <vector>

#include "scout_b200.h"

namespace scout_b200 {

// ------------------------------------------------------------ mirror types
using Vec = std::vector<double>;
using BlockIdSet = std::vector<std::size_t>;
enum class DigestMethod { minmax, mean };

struct Mat {
    std::size_t rows = 0, cols = 0;
    std::vector<double> data;
    Mat() = default;
    Mat(std::size_t r, std::size_t c) : rows(r), cols(c), data(r * c, 0.0) {}
    const double* row(std::size_t r) const { return data.data() + r * cols; }
    Vec row_vec(std::size_t r) const { return Vec(row(r), row(r) + cols); }
    void append_row(const Vec& v) {
        if (rows == 0 && cols == 0) cols = v.size();
        if (v.size() != cols) throw std::invalid_argument("Mat::append_row: width mismatch");
        data.insert(data.end(), v.begin(), v.end());
        ++rows;
    }
};
struct BlockDigest {
    DigestMethod method = DigestMethod::minmax;
    Vec lo, hi, mean;
    std::size_t block_id = 0;
    std::size_t layer = 0;
};
struct KvBlock {
    std::size_t block_id = 0, layer = 0;
    Mat keys, values;
    bool sealed = false;
};
struct PartialAttention {
    Vec o_acc;
    double max_logit = -std::numeric_limits<double>::infinity();
    double denom = 0.0;
    std::size_t token_count = 0;
    static PartialAttention empty(std::size_t dim) {
        PartialAttention p;
        p.o_acc.assign(dim, 0.0);
        return p;
    }
    bool is_empty() const { return token_count == 0; }
};

// Results that convert to the caller's own structs: a reference call site
// such as `const PartialAttention gpu = scout_b200::partial_attention(...)`
// (scout::PartialAttention) or `st.digests.back() = scout_b200::build_digest(...)`
// (scout::BlockDigest) compiles unchanged; the mirror types above are the
// results' bases, so code without the reference headers uses them directly.
struct PartialResult : PartialAttention {
    PartialResult() = default;
    explicit PartialResult(const PartialAttention& p) : PartialAttention(p) {}
    template <class T, class = decltype(T{}.o_acc), class = decltype(T{}.token_count)>
    operator T() const {
        T t;
        t.o_acc = o_acc;
        t.max_logit = max_logit;
        t.denom = denom;
        t.token_count = token_count;
        return t;
    }
};
struct DigestResult : BlockDigest {
    template <class T, class = decltype(T{}.lo), class = decltype(T{}.block_id)>
    operator T() const {
        T t;
        t.method = static_cast<decltype(t.method)>(static_cast<int>(method));
        t.lo = lo;
        t.hi = hi;
        t.mean = mean;
        t.block_id = block_id;
        t.layer = layer;
        return t;
    }
};

namespace detail {

inline void check(int rc) {
    if (rc == SCOUT_OK) return;
    const std::string msg = scout_last_error();
    if (rc == SCOUT_ERR_INVALID_ARGUMENT) throw std::invalid_argument(msg);
    throw std::runtime_error("scout_b200: " + msg);
}
inline void cuda(cudaError_t e, const char* what) {
    if (e != cudaSuccess) throw std::runtime_error(std::string("scout_b200: ") + what + ": " + cudaGetErrorString(e));
}

// RAII device buffer
struct DevBuf {
    void* p = nullptr;
    explicit DevBuf(std::size_t n) { cuda(cudaMalloc(&p, n ? n : 16), "cudaMalloc"); }
    ~DevBuf() { if (p) cudaFree(p); }
    DevBuf(const DevBuf&) = delete;
    DevBuf& operator=(const DevBuf&) = delete;
    template <class T> T* as() const { return static_cast<T*>(p); }
};
template <class T>
inline void h2d(const DevBuf& d, const std::vector<T>& h) {
    cuda(cudaMemcpy(d.p, h.data(), h.size() * sizeof(T), cudaMemcpyHostToDevice), "H2D");
}
template <class T>
inline void d2h(std::vector<T>& h, const DevBuf& d) {
    cuda(cudaMemcpy(h.data(), d.p, h.size() * sizeof(T), cudaMemcpyDeviceToHost), "D2H");
}

template <class M>
inline bool is_minmax(const M& m) { return static_cast<int>(m) == static_cast<int>(DigestMethod::minmax); }

// scores of n single-head digests on the exact f64 path (K1, MODE 1/2)
template <class Digests>
inline std::vector<double> scores_and_topk(const Vec& q, const Digests& ds, std::size_t k, BlockIdSet* out) {
    const std::size_t n = ds.size();
    const std::size_t dim = q.size();
    if (dim > SCOUT_HEAD_DIM) throw std::invalid_argument("scout_b200: query dimension > 128 unsupported");
    if (n > SCOUT_MAX_BLOCKS) throw std::invalid_argument("scout_b200: more than 4096 digests");
    // reference ties break on block_id: order the digests by id (stable)
    std::vector<std::size_t> order(n);
    std::iota(order.begin(), order.end(), std::size_t{0});
    std::stable_sort(order.begin(), order.end(), [&](std::size_t a, std::size_t b) { return ds[a].block_id < ds[b].block_id; });
    const bool minmax = n == 0 || is_minmax(ds[0].method);
    const int nbs = static_cast<int>(std::max<std::size_t>(8, (n + 7) / 8 * 8));
    const std::size_t rows = minmax ? 2 * SCOUT_HEAD_DIM : SCOUT_HEAD_DIM;
    std::vector<double> dig(rows * nbs, 0.0), qq(SCOUT_HEAD_DIM, 0.0);
    std::copy(q.begin(), q.end(), qq.begin());
    for (std::size_t j = 0; j < n; ++j) {
        const auto& d = ds[order[j]];
        if (is_minmax(d.method) != minmax) throw std::invalid_argument("scout_b200: mixed digest methods");
        const auto& a = minmax ? d.lo : d.mean;
        if (a.size() != dim || (minmax && d.hi.size() != dim))
            throw std::invalid_argument("digest_score: query/digest dimension mismatch");
        for (std::size_t c = 0; c < dim; ++c) {
            dig[c * nbs + j] = a[c];
            if (minmax) dig[(SCOUT_HEAD_DIM + c) * nbs + j] = d.hi[c];
        }
    }
    DevBuf dq(qq.size() * 8), dd(dig.size() * 8), dn(4), dsel((k ? k : 1) * 4), dns(4), dsc(nbs * 8);
    h2d(dq, qq);
    h2d(dd, dig);
    const std::vector<int32_t> ntok{static_cast<int32_t>(n * SCOUT_BLOCK_SIZE)};
    h2d(dn, ntok);
    scout_topk_args a{};
    a.n_units = 1;
    a.group = 1;
    a.digest_dtype = SCOUT_F64;
    a.method = minmax ? SCOUT_DIGEST_MINMAX : SCOUT_DIGEST_MEAN;
    a.k = static_cast<int>(std::min<std::size_t>(k, SCOUT_MAX_K));
    if (k > SCOUT_MAX_K && k < n) throw std::invalid_argument("scout_b200: k > 512 unsupported");
    a.k_stride = std::max(a.k, 1);
    a.nb_stride = nbs;
    a.q = dq.p;
    a.digests = dd.p;
    a.n_tokens = dn.as<int32_t>();
    a.sel_ids = dsel.as<int32_t>();
    a.n_sel = dns.as<int32_t>();
    a.scores_out = dsc.as<double>();
    check(scout_score_topk_split(&a, nullptr));
    cuda(cudaDeviceSynchronize(), "score_topk");
    std::vector<double> sc(nbs);
    d2h(sc, dsc);
    std::vector<double> by_input(n);
    for (std::size_t j = 0; j < n; ++j) by_input[order[j]] = sc[j];
    if (out) {
        std::vector<int32_t> ns(1), sel(a.k_stride);
        d2h(ns, dns);
        d2h(sel, dsel);
        out->clear();
        for (int i = 0; i < ns[0]; ++i) out->push_back(ds[order[sel[i]]].block_id);
        std::sort(out->begin(), out->end());
    }
    return by_input;
}

}  // namespace detail

// -------------------------------------------------------------- digest.hpp
template <class MatT, class Method>
inline DigestResult build_digest(const MatT& keys, Method method, std::size_t block_id = 0, std::size_t layer = 0) {
    if (keys.rows == 0) throw std::invalid_argument("build_digest: empty block");
    if (keys.rows > SCOUT_BLOCK_SIZE || keys.cols > SCOUT_HEAD_DIM)
        throw std::invalid_argument("scout_b200: block larger than 64 x 128 unsupported");
    using namespace detail;
    const bool minmax = is_minmax(method);
    std::vector<float> k(SCOUT_BLOCK_SIZE * SCOUT_HEAD_DIM, 0.f);
    for (std::size_t r = 0; r < keys.rows; ++r)
        for (std::size_t c = 0; c < keys.cols; ++c) k[r * SCOUT_HEAD_DIM + c] = static_cast<float>(keys.row(r)[c]);
    const std::size_t sb = scout_slot_bytes(SCOUT_F32);
    DevBuf pool(sb), rowsf(k.size() * 4), slots(SCOUT_BLOCK_SIZE * 4), rr(SCOUT_BLOCK_SIZE * 4), meta(4 * 4),
        dig((minmax ? 2 : 1) * SCOUT_HEAD_DIM * 8 * 8);
    h2d(rowsf, k);
    std::vector<int32_t> sl(SCOUT_BLOCK_SIZE, 0), ri(SCOUT_BLOCK_SIZE);
    std::iota(ri.begin(), ri.end(), 0);
    h2d(slots, sl);
    h2d(rr, ri);
    check(scout_kv_write_tokens(pool.p, SCOUT_F32, slots.as<int32_t>(), rr.as<int32_t>(), rowsf.as<float>(),
                                rowsf.as<float>(), SCOUT_BLOCK_SIZE, nullptr));
    const std::vector<int32_t> m{0, static_cast<int32_t>(keys.rows), 0, 0};  // slot, rows, unit, block
    h2d(meta, m);
    const int32_t* mp = meta.as<int32_t>();
    check(scout_digest_build(pool.p, SCOUT_F32, minmax ? SCOUT_DIGEST_MINMAX : SCOUT_DIGEST_MEAN, 1, mp, mp + 1, mp + 2,
                             mp + 3, dig.p, 8, nullptr));
    cuda(cudaDeviceSynchronize(), "build_digest");
    DigestResult d;
    d.method = minmax ? DigestMethod::minmax : DigestMethod::mean;
    d.block_id = block_id;
    d.layer = layer;
    if (minmax) {
        std::vector<float> h(2 * SCOUT_HEAD_DIM * 8);
        d2h(h, dig);
        for (std::size_t c = 0; c < keys.cols; ++c) {
            d.lo.push_back(h[c * 8]);
            d.hi.push_back(h[(SCOUT_HEAD_DIM + c) * 8]);
        }
    } else {
        std::vector<double> h(SCOUT_HEAD_DIM * 8);
        d2h(h, dig);
        for (std::size_t c = 0; c < keys.cols; ++c) d.mean.push_back(h[c * 8]);
    }
    return d;
}

template <class Digest>
inline double digest_score(const Vec& q, const Digest& d) {
    const std::vector<Digest> one{d};
    return detail::scores_and_topk(q, one, 1, nullptr)[0];
}

template <class Digests>
inline BlockIdSet select_topk(const Vec& q, const Digests& digests, std::size_t k) {
    if (k == 0) throw std::invalid_argument("select_topk: k must be >= 1");
    BlockIdSet out;
    if (digests.empty()) return out;
    detail::scores_and_topk(q, digests, k, &out);
    return out;
}

// ----------------------------------------------------------- attention.hpp
template <class BlockPtrs>
inline PartialAttention partial_attention_impl(const Vec& q, const BlockPtrs& blocks, double scale) {
    using namespace detail;
    if (!(scale > 0.0)) throw std::invalid_argument("partial_attention: scale must be > 0");
    if (q.size() > SCOUT_HEAD_DIM) throw std::invalid_argument("scout_b200: query dimension > 128 unsupported");
    PartialAttention p = PartialAttention::empty(q.size());
    std::size_t n = 0;
    for (const auto* b : blocks) {
        if (b->keys.cols != q.size()) throw std::invalid_argument("partial_attention: query/key dimension mismatch");
        n += b->keys.rows;
    }
    if (n == 0) return p;
    // rows repacked contiguously (visit order kept) into 64-row f32 slots
    const std::size_t nb = (n + SCOUT_BLOCK_SIZE - 1) / SCOUT_BLOCK_SIZE;
    std::vector<float> kr(n * SCOUT_HEAD_DIM, 0.f), vr(n * SCOUT_HEAD_DIM, 0.f);
    std::vector<int32_t> slot(n), row(n);
    std::size_t t = 0;
    for (const auto* b : blocks)
        for (std::size_t r = 0; r < b->keys.rows; ++r, ++t) {
            for (std::size_t c = 0; c < q.size(); ++c) {
                kr[t * SCOUT_HEAD_DIM + c] = static_cast<float>(b->keys.row(r)[c]);
                vr[t * SCOUT_HEAD_DIM + c] = static_cast<float>(b->values.row(r)[c]);
            }
            slot[t] = static_cast<int32_t>(t / SCOUT_BLOCK_SIZE);
            row[t] = static_cast<int32_t>(t % SCOUT_BLOCK_SIZE);
        }
    const std::size_t sb = scout_slot_bytes(SCOUT_F32);
    DevBuf pool(nb * sb), dk(kr.size() * 4), dv(vr.size() * 4), ds(n * 4), dr(n * 4);
    h2d(dk, kr);
    h2d(dv, vr);
    h2d(ds, slot);
    h2d(dr, row);
    check(scout_kv_write_tokens(pool.p, SCOUT_F32, ds.as<int32_t>(), dr.as<int32_t>(), dk.as<float>(), dv.as<float>(),
                                static_cast<int>(n), nullptr));
    std::vector<float> qf(SCOUT_HEAD_DIM, 0.f);
    for (std::size_t c = 0; c < q.size(); ++c) qf[c] = static_cast<float>(q[c]);
    std::vector<int32_t> ids(nb);
    std::iota(ids.begin(), ids.end(), 0);
    const std::vector<int32_t> nres{static_cast<int32_t>(nb)}, ntok{static_cast<int32_t>(n)};
    const size_t wsb = scout_sparse_decode_workspace_bytes(1, 1, 0);
    DevBuf dq(qf.size() * 4), dslots(nb * 4), dids(nb * 4), dnres(4), dntok(4), dout(SCOUT_HEAD_DIM * 4), dml(8),
        ws(wsb);
    cuda(cudaMemset(ws.p, 0, wsb), "memset");
    h2d(dq, qf);
    h2d(dslots, ids);
    h2d(dids, ids);
    h2d(dnres, nres);
    h2d(dntok, ntok);
    scout_decode_args a{};
    a.n_units = 1;
    a.group = 1;
    a.kv_dtype = SCOUT_F32;
    a.k_stride = static_cast<int>(nb);
    a.scale = static_cast<float>(scale);
    a.q = dq.as<float>();
    a.kv_pool = pool.p;
    a.res_slots = dslots.as<int32_t>();
    a.res_ids = dids.as<int32_t>();
    a.n_res = dnres.as<int32_t>();
    a.n_tokens = dntok.as<int32_t>();
    a.o = dout.as<float>();
    a.ml = dml.as<float>();
    a.workspace = ws.p;
    a.workspace_bytes = wsb;
    check(scout_sparse_decode(&a, nullptr));
    cuda(cudaDeviceSynchronize(), "partial_attention");
    std::vector<float> o(SCOUT_HEAD_DIM), ml(2);
    d2h(o, dout);
    d2h(ml, dml);
    // (o normalised, m, l) -> the reference's unnormalised (o_acc, max_logit, denom)
    p.max_logit = ml[0];
    p.denom = ml[1];
    for (std::size_t c = 0; c < q.size(); ++c) p.o_acc[c] = static_cast<double>(o[c]) * ml[1];
    p.token_count = n;
    return p;
}

template <class KvBlockT>
inline PartialResult partial_attention(const Vec& q, std::span<const KvBlockT* const> blocks, double scale) {
    return PartialResult(partial_attention_impl(q, blocks, scale));
}
template <class KvBlockT>
inline PartialResult partial_attention(const Vec& q, const std::vector<const KvBlockT*>& blocks, double scale) {
    return PartialResult(partial_attention_impl(q, blocks, scale));
}

namespace detail {
// a partial of one struct type as another (same four fields)
template <class P, class Q>
inline P partial_as(const Q& q) {
    P p{};
    p.o_acc = q.o_acc;
    p.max_logit = q.max_logit;
    p.denom = q.denom;
    p.token_count = q.token_count;
    return p;
}
}  // namespace detail

// merge (attention.hpp:100-114); the result has the first operand's type (the
// operands may be a PartialResult and a plain partial, e.g. an empty one)
template <class P, class Q>
inline P merge(const P& a, const Q& b) {
    using namespace detail;
    if (a.is_empty()) return partial_as<P>(b);  // exact identity (attention.hpp:101-102)
    if (b.is_empty()) return a;
    if (a.o_acc.size() != b.o_acc.size()) throw std::invalid_argument("merge: dimension mismatch");
    const std::size_t d = a.o_acc.size();
    if (d > SCOUT_HEAD_DIM) throw std::invalid_argument("scout_b200: dimension > 128 unsupported");
    std::vector<float> ao(SCOUT_HEAD_DIM, 0.f), bo(SCOUT_HEAD_DIM, 0.f);
    for (std::size_t c = 0; c < d; ++c) {
        ao[c] = static_cast<float>(a.o_acc[c] / a.denom);
        bo[c] = static_cast<float>(b.o_acc[c] / b.denom);
    }
    const std::vector<float> aml{static_cast<float>(a.max_logit), static_cast<float>(a.denom)};
    const std::vector<float> bml{static_cast<float>(b.max_logit), static_cast<float>(b.denom)};
    DevBuf dao(ao.size() * 4), dbo(bo.size() * 4), daml(8), dbml(8), doo(ao.size() * 4), doml(8);
    h2d(dao, ao);
    h2d(dbo, bo);
    h2d(daml, aml);
    h2d(dbml, bml);
    check(scout_merge_partials(dao.as<float>(), daml.as<float>(), dbo.as<float>(), dbml.as<float>(), doo.as<float>(),
                               doml.as<float>(), 1, nullptr));
    cuda(cudaDeviceSynchronize(), "merge");
    std::vector<float> o(SCOUT_HEAD_DIM), ml(2);
    d2h(o, doo);
    d2h(ml, doml);
    P out = a;
    out.max_logit = ml[0];
    out.denom = ml[1];
    for (std::size_t c = 0; c < d; ++c) out.o_acc[c] = static_cast<double>(o[c]) * ml[1];
    out.token_count = a.token_count + b.token_count;
    return out;
}

// finalize is o_acc / denom (attention.hpp:117-122): on the device path K2
// fuses it; on this compatibility path the partial already lives on the host.
template <class P>
inline Vec finalize(const P& p) {
    if (p.is_empty()) throw std::invalid_argument("finalize: empty partial");
    Vec out(p.o_acc.size());
    for (std::size_t c = 0; c < out.size(); ++c) out[c] = p.o_acc[c] / p.denom;
    return out;
}

}  // namespace scout_b200
