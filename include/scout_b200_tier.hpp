// scout_b200_tier.hpp — header-only C++ drop-in for the reference's
// TieredKvCache (proj/include/scout/kv_store.hpp) whose tier state machine
// runs on the B200: the tier flags, last_selected marks, in-flight recall
// tickets, LRU eviction and the residency planning view live in device
// memory and only the K5 kernels touch them (scout_tier_* in scout_b200.h).
//
// Restated reference API (kv_store.hpp line):
//   TieredKvCache(layers, block_size, head_dim, method, fast_capacity)   :66
//   pin_layer :81   fast_capacity :85   append_token :90   total_tokens :119
//   block_count :120   sealed_count :122   digests :128   block :130
//   tier_of :136   is_in_flight :142   last_selected :148   residency_set :156
//   schedule_recall :175   begin_layer :201   clock :221   mark_selected :222
//   fetch_blocks :231   fetch_blocks_any :245   demote_block :257
//   place_after_prefill :268   sealed_fast_count :281   dump_residency :289
//
// The blocks' rows and digests stay on the host, as the reference keeps them
// (fetch_blocks hands out stable KvBlock pointers for the CPU side, digests()
// feeds select_topk); the open block's digest is rebuilt exactly in double on
// every append as in kv_store.hpp:108 (the device fold of the product path is
// K0's scout_kv_append). Block size must be 64 (the GPU pool's block); a layer
// holds at most max_blocks blocks (constructor, default 4096). The class is a
// template over the block / digest / ticket / tier / method / matrix types so
// it can hand out the reference's own scout:: types (TieredKvCacheT<...>);
// scout_b200::TieredKvCache uses the mirror types of scout_b200.hpp. Errors
// follow the reference: std::invalid_argument for argument and sequencing
// errors (a rejected recall ticket included), std::runtime_error for device
// failures. Every call synchronises (compatibility API: the decode engine's
// device tier mode runs the same kernels batched, without host round trips).
#pragma once

#include <cuda_runtime.h>

#include <algorithm>
#include <cstddef>
#include <cstdint>
#include <deque>
#include <limits>
#include <optional>
#include <ostream>
#include <stdexcept>
#include <string>
#include <utility>
#include <vector>

#include "scout_b200.hpp"

namespace scout_b200 {

enum class Tier { fast, slow };

struct RecallTicket {
    std::size_t layer = 0;
    BlockIdSet ids;
    std::size_t issue_step = 0;
    std::size_t issue_layer = 0;
    std::size_t ready_step = 0;
    std::size_t ready_layer = 0;
};

template <class KvBlockT = KvBlock, class DigestT = BlockDigest, class TicketT = RecallTicket, class TierT = Tier,
          class MethodT = DigestMethod, class MatT = Mat>
class TieredKvCacheT {
public:
    TieredKvCacheT(std::size_t layers, std::size_t block_size, std::size_t head_dim, MethodT method,
                   std::size_t fast_capacity, std::size_t max_blocks = 4096)
        : head_dim_(head_dim), method_(method), nbs_(static_cast<int>((max_blocks + 7) / 8 * 8)), layers_(layers) {
        if (layers == 0) throw std::invalid_argument("TieredKvCache: layers must be >= 1");
        if (block_size == 0) throw std::invalid_argument("TieredKvCache: block_size must be >= 1");
        if (fast_capacity == 0) throw std::invalid_argument("TieredKvCache: fast_capacity must be >= 1");
        if (block_size != SCOUT_BLOCK_SIZE)
            throw std::invalid_argument("scout_b200::TieredKvCache: block_size must be 64 (the GPU pool's block)");
        if (max_blocks == 0 || max_blocks > (1u << 20))
            throw std::invalid_argument("scout_b200::TieredKvCache: max_blocks out of range");
        if (fast_capacity > static_cast<std::size_t>(std::numeric_limits<int>::max()))
            fast_capacity = static_cast<std::size_t>(std::numeric_limits<int>::max());
        for (auto& st : layers_) st.capacity = fast_capacity;
        // per layer, one unit: table | last_sel | ready | ticket | warm [nbs] int32,
        // free ring + owners [nbs] int32, n_free | err | head | n_tokens int32, tier [nbs] u8
        const std::size_t L = layers, n = static_cast<std::size_t>(nbs_);
        per_layer_ = (7 * n + 4) * 4 + (n + 15) / 16 * 16;
        detail::cuda(cudaMalloc(&dev_, per_layer_ * L), "TieredKvCache: device state");
        detail::cuda(cudaStreamCreateWithFlags(&st_, cudaStreamNonBlocking), "TieredKvCache: stream");
        std::vector<int32_t> init(7 * n + 4, -1);
        for (std::size_t i = 0; i < n; ++i) {
            init[3 * n + i] = 0;                          // ticket
            init[5 * n + i] = static_cast<int32_t>(i);    // free ring: this unit's slots 0 .. nbs-1
        }
        for (std::size_t i = 0; i < n; ++i) init[i + n] = 0;  // last_sel
        init[7 * n + 0] = static_cast<int32_t>(n);            // n_free
        init[7 * n + 1] = 0;                                  // err
        init[7 * n + 2] = 0;                                  // ring head
        init[7 * n + 3] = 0;                                  // n_tokens
        std::vector<uint8_t> zero((n + 15) / 16 * 16, 0);
        for (std::size_t l = 0; l < L; ++l) {
            uint8_t* base = static_cast<uint8_t*>(dev_) + l * per_layer_;
            detail::cuda(cudaMemcpy(base, init.data(), init.size() * 4, cudaMemcpyHostToDevice), "TieredKvCache: init");
            detail::cuda(cudaMemcpy(base + init.size() * 4, zero.data(), zero.size(), cudaMemcpyHostToDevice),
                         "TieredKvCache: init");
        }
        detail::cuda(cudaMalloc(&scratch_, n * 4 * 2 + 64), "TieredKvCache: scratch");
    }
    ~TieredKvCacheT() {
        if (scratch_) cudaFree(scratch_);
        if (dev_) cudaFree(dev_);
        if (st_) cudaStreamDestroy(st_);
    }
    TieredKvCacheT(const TieredKvCacheT&) = delete;
    TieredKvCacheT& operator=(const TieredKvCacheT&) = delete;

    std::size_t num_layers() const { return layers_.size(); }
    std::size_t block_size() const { return SCOUT_BLOCK_SIZE; }

    void pin_layer(std::size_t layer) { state(layer).capacity = std::numeric_limits<std::size_t>::max(); }
    std::size_t fast_capacity(std::size_t layer) const { return state(layer).capacity; }

    // append_token (kv_store.hpp:90-117): rows and the open block's digest on
    // the host; the block's opening (a pool slot, fast, marked) and its seal
    // (mark, enforce_capacity) on the device
    std::optional<std::size_t> append_token(std::size_t layer, const Vec& k, const Vec& v) {
        if (k.size() != head_dim_ || v.size() != head_dim_)
            throw std::invalid_argument("append_token: expected head_dim = " + std::to_string(head_dim_));
        LayerState& st = state(layer);
        const bool opening = st.blocks.empty() || st.blocks.back().sealed;
        if (opening && st.blocks.size() >= static_cast<std::size_t>(nbs_))
            throw std::invalid_argument("scout_b200::TieredKvCache: layer full (max_blocks)");
        scout_tier_layer d = desc(layer);
        int32_t* ptr = scratch_;
        detail::check(scout_tier_append(&d, 1, nbs_, ntok_dev(layer), static_cast<int>(clock_step_), ptr, ptr + 1, st_));
        std::vector<int32_t> out(2);
        sync_d2h(out.data(), ptr, 8);
        check_err(layer, "append_token");
        if (opening) {
            KvBlockT b;
            b.block_id = st.blocks.size();
            b.layer = layer;
            b.keys = MatT(0, head_dim_);
            b.values = MatT(0, head_dim_);
            st.blocks.push_back(std::move(b));
            st.digests.emplace_back();
        }
        KvBlockT& open = st.blocks.back();
        open.keys.append_row(k);
        open.values.append_row(v);
        st.digests.back() = host_digest(open.keys, open.block_id, layer);
        st.tokens += 1;
        const int32_t nt = static_cast<int32_t>(st.tokens);
        detail::cuda(cudaMemcpyAsync(ntok_dev(layer), &nt, 4, cudaMemcpyHostToDevice, st_), "append_token");
        detail::cuda(cudaStreamSynchronize(st_), "append_token");
        if (open.keys.rows == SCOUT_BLOCK_SIZE) {
            open.sealed = true;
            if (out[1] != static_cast<int32_t>(open.block_id))
                throw std::runtime_error("scout_b200::TieredKvCache: device seal disagrees with the host rows");
            return open.block_id;
        }
        return std::nullopt;
    }

    std::size_t total_tokens(std::size_t layer) const { return state(layer).tokens; }
    std::size_t block_count(std::size_t layer) const { return state(layer).blocks.size(); }
    std::size_t sealed_count(std::size_t layer) const {
        const LayerState& st = state(layer);
        if (st.blocks.empty()) return 0;
        return st.blocks.back().sealed ? st.blocks.size() : st.blocks.size() - 1;
    }
    const std::vector<DigestT>& digests(std::size_t layer) const { return state(layer).digests; }
    const KvBlockT& block(std::size_t layer, std::size_t id) const {
        const LayerState& st = state(layer);
        check_id(st, id);
        return st.blocks[id];
    }

    TierT tier_of(std::size_t layer, std::size_t id) const {
        check_id(state(layer), id);
        return device_tier(layer)[id] ? TierT::fast : TierT::slow;
    }
    bool is_in_flight(std::size_t layer, std::size_t id) const {
        check_id(state(layer), id);
        return device_i32(layer, READY)[id] >= 0;
    }
    std::size_t last_selected(std::size_t layer, std::size_t id) const {
        check_id(state(layer), id);
        return static_cast<std::size_t>(device_i32(layer, LAST_SEL)[id]);
    }

    // residency_set (kv_store.hpp:156-170): fast blocks plus in-flight ones
    // that arrive by next_run_of(layer), from the device planning view
    BlockIdSet residency_set(std::size_t layer) const {
        state(layer);
        scout_tier_layer d = desc(layer);
        const auto nr = next_run_of(layer);
        detail::check(scout_tier_plan(&d, 1, nbs_, ntok_dev(layer), tick(nr.first, nr.second), scratch_,
                                      st_));
        std::vector<int32_t> tab(nbs_);
        sync_d2h(tab.data(), scratch_, tab.size() * 4);
        BlockIdSet out;
        for (int b = 0; b < nbs_; ++b)
            if (tab[b] >= 0) out.push_back(static_cast<std::size_t>(b));
        return out;
    }

    // schedule_recall (kv_store.hpp:175-197): validated on the device (sealed,
    // slow, not in flight); a rejected ticket changes nothing and throws
    TicketT schedule_recall(std::size_t layer, const BlockIdSet& ids, std::size_t issue_step, std::size_t issue_layer) {
        const LayerState& st = state(layer);
        if (ids.empty()) throw std::invalid_argument("schedule_recall: empty id set");
        for (std::size_t id : ids) check_id(st, id);
        if (ids.size() > static_cast<std::size_t>(nbs_))
            throw std::invalid_argument("schedule_recall: more ids than blocks");
        std::vector<int32_t> h(ids.begin(), ids.end());
        const int32_t n = static_cast<int32_t>(h.size());
        int32_t* dids = scratch_;
        int32_t* dn = dids + nbs_;
        detail::cuda(cudaMemcpyAsync(dids, h.data(), h.size() * 4, cudaMemcpyHostToDevice, st_), "schedule_recall");
        detail::cuda(cudaMemcpyAsync(dn, &n, 4, cudaMemcpyHostToDevice, st_), "schedule_recall");
        detail::DevBuf dst(static_cast<std::size_t>(nbs_) * 4);  // the slots (no pool behind this cache)
        scout_tier_layer d = desc(layer);
        detail::check(scout_tier_schedule_recall(&d, 1, nbs_, ntok_dev(layer), dids, dn, nbs_,
                                                 tick(issue_step + 1, issue_layer), n_tickets_, dst.as<int32_t>(), st_));
        detail::cuda(cudaStreamSynchronize(st_), "schedule_recall");
        int32_t err = 0;
        sync_d2h(&err, i32(layer, ERR), 4);
        if (err != 0) {
            clear_err(layer);
            throw std::invalid_argument("schedule_recall: ticket rejected (a block unsealed, already fast or in flight)");
        }
        ++n_tickets_;
        TicketT t;
        t.layer = layer;
        t.ids = ids;
        t.issue_step = issue_step;
        t.issue_layer = issue_layer;
        t.ready_step = issue_step + 1;
        t.ready_layer = issue_layer;
        in_flight_.push_back(t);
        return t;
    }

    // begin_layer (kv_store.hpp:201-218): every ticket whose ready point has
    // been reached becomes fast on the device, per layer in issue order, each
    // followed by enforce_capacity; returns the applied tickets in issue order
    std::vector<TicketT> begin_layer(std::size_t step, std::size_t layer) {
        clock_step_ = step;
        clock_layer_ = layer;
        const int now = tick(step, layer);
        std::vector<TicketT> applied;
        std::vector<bool> due(layers_.size(), false);
        for (std::size_t i = 0; i < in_flight_.size();) {
            const TicketT& t = in_flight_[i];
            if (std::make_pair(t.ready_step, t.ready_layer) <= std::make_pair(step, layer)) {
                due[t.layer] = true;
                applied.push_back(t);
                in_flight_.erase(in_flight_.begin() + static_cast<std::ptrdiff_t>(i));
            } else {
                ++i;
            }
        }
        for (std::size_t l = 0; l < layers_.size(); ++l) {
            if (!due[l]) continue;
            scout_tier_layer d = desc(l);
            detail::check(scout_tier_apply(&d, 1, nbs_, ntok_dev(l), now, nullptr, st_));
        }
        detail::cuda(cudaStreamSynchronize(st_), "begin_layer");
        return applied;
    }

    std::pair<std::size_t, std::size_t> clock() const { return {clock_step_, clock_layer_}; }

    void mark_selected(std::size_t layer, const BlockIdSet& ids, std::size_t step) {
        const LayerState& st = state(layer);
        for (std::size_t id : ids) check_id(st, id);
        if (ids.empty()) return;
        std::vector<int32_t> h(ids.begin(), ids.end());
        const int32_t n = static_cast<int32_t>(h.size());
        detail::DevBuf dids(h.size() * 4), dn(4);
        detail::cuda(cudaMemcpyAsync(dids.p, h.data(), h.size() * 4, cudaMemcpyHostToDevice, st_), "mark_selected");
        detail::cuda(cudaMemcpyAsync(dn.p, &n, 4, cudaMemcpyHostToDevice, st_), "mark_selected");
        scout_tier_layer d = desc(layer);
        detail::check(scout_tier_mark(&d, 1, nbs_, dids.as<int32_t>(), dn.as<int32_t>(), n, static_cast<int>(step), st_));
        detail::cuda(cudaStreamSynchronize(st_), "mark_selected");
    }

    // fetch_blocks (kv_store.hpp:231-244): blocks that must sit in `tier`
    // (checked against the device tier flags)
    std::vector<const KvBlockT*> fetch_blocks(std::size_t layer, const BlockIdSet& ids, TierT tier) const {
        const LayerState& st = state(layer);
        const std::vector<uint8_t> tf = device_tier(layer);
        std::vector<const KvBlockT*> out;
        out.reserve(ids.size());
        for (std::size_t id : ids) {
            check_id(st, id);
            const bool fast = tf[id] != 0;
            if (fast != (tier == TierT::fast))
                throw std::invalid_argument("fetch_blocks: block " + std::to_string(id) + " not in " +
                                            (tier == TierT::fast ? "fast" : "slow") + " tier");
            out.push_back(&st.blocks[id]);
        }
        return out;
    }
    std::vector<const KvBlockT*> fetch_blocks_any(std::size_t layer, const BlockIdSet& ids) const {
        const LayerState& st = state(layer);
        std::vector<const KvBlockT*> out;
        out.reserve(ids.size());
        for (std::size_t id : ids) {
            check_id(st, id);
            out.push_back(&st.blocks[id]);
        }
        return out;
    }

    // demote_block (kv_store.hpp:257-265): the device placement with every
    // other sealed fast block kept (no promotion, no capacity enforcement)
    void demote_block(std::size_t layer, std::size_t id) {
        const LayerState& st = state(layer);
        check_id(st, id);
        if (!st.blocks[id].sealed) throw std::invalid_argument("demote_block: open block must stay fast");
        const std::vector<uint8_t> tf = device_tier(layer);
        if (!tf[id]) throw std::invalid_argument("demote_block: block " + std::to_string(id) + " not fast");
        BlockIdSet keep;
        for (std::size_t b = 0; b < st.blocks.size(); ++b)
            if (st.blocks[b].sealed && tf[b] && b != id) keep.push_back(b);
        place(layer, keep);
    }

    // place_after_prefill (kv_store.hpp:268-279): select_topk of the sealed
    // digests (the exact f64 path on the device), then the device placement
    template <class QVec>
    void place_after_prefill(std::size_t layer, const QVec& q) {
        const LayerState& st = state(layer);
        if (st.capacity == std::numeric_limits<std::size_t>::max()) return;  // pinned
        std::vector<DigestT> sealed;
        for (std::size_t id = 0; id < st.blocks.size(); ++id)
            if (st.blocks[id].sealed) sealed.push_back(st.digests[id]);
        if (sealed.empty()) return;
        const BlockIdSet keep = select_topk(Vec(q.begin(), q.end()), sealed, st.capacity);
        place(layer, keep);
    }

    std::size_t sealed_fast_count(std::size_t layer) const {
        const LayerState& st = state(layer);
        const std::vector<uint8_t> tf = device_tier(layer);
        std::size_t n = 0;
        for (std::size_t id = 0; id < st.blocks.size(); ++id)
            if (st.blocks[id].sealed && tf[id]) ++n;
        return n;
    }

    void dump_residency(std::ostream& os) const {
        os << "# layer block tier last_selected\n";
        for (std::size_t layer = 0; layer < layers_.size(); ++layer) {
            const std::vector<uint8_t> tf = device_tier(layer);
            const std::vector<int32_t> ls = device_i32(layer, LAST_SEL);
            for (std::size_t id = 0; id < layers_[layer].blocks.size(); ++id)
                os << layer << ' ' << id << ' ' << (tf[id] ? "fast" : "slow") << ' ' << ls[id] << '\n';
        }
    }

private:
    enum Field { TABLE = 0, LAST_SEL = 1, READY = 2, TICKET = 3, WARM = 4, RING = 5, OWNER = 6, N_FREE = 7, ERR = 8,
                 HEAD = 9, NTOK = 10 };
    struct LayerState {
        std::deque<KvBlockT> blocks;  // stable element addresses across appends
        std::vector<DigestT> digests;
        std::size_t tokens = 0;
        std::size_t capacity = 0;
    };

    LayerState& state(std::size_t layer) {
        if (layer >= layers_.size()) throw std::invalid_argument("layer out of range");
        return layers_[layer];
    }
    const LayerState& state(std::size_t layer) const {
        if (layer >= layers_.size()) throw std::invalid_argument("layer out of range");
        return layers_[layer];
    }
    static void check_id(const LayerState& st, std::size_t id) {
        if (id >= st.blocks.size()) throw std::invalid_argument("block id out of range");
    }
    std::pair<std::size_t, std::size_t> next_run_of(std::size_t layer) const {  // kv_store.hpp:328-331
        if (clock_layer_ <= layer) return {clock_step_, layer};
        return {clock_step_ + 1, layer};
    }
    int tick(std::size_t step, std::size_t layer) const {
        return static_cast<int>(step * layers_.size() + layer);
    }

    int32_t* i32(std::size_t layer, Field f) const {
        auto* base = reinterpret_cast<int32_t*>(static_cast<uint8_t*>(dev_) + layer * per_layer_);
        const std::size_t n = static_cast<std::size_t>(nbs_);
        return f <= OWNER ? base + f * n : base + 7 * n + (f - N_FREE);
    }
    int32_t* ntok_dev(std::size_t layer) const { return i32(layer, NTOK); }
    uint8_t* tier_dev(std::size_t layer) const {
        return static_cast<uint8_t*>(dev_) + layer * per_layer_ + (7 * static_cast<std::size_t>(nbs_) + 4) * 4;
    }
    scout_tier_layer desc(std::size_t layer) const {
        scout_tier_layer d{};
        d.table = i32(layer, TABLE);
        d.tier = tier_dev(layer);
        d.last_sel = i32(layer, LAST_SEL);
        d.ready = i32(layer, READY);
        d.ticket = i32(layer, TICKET);
        d.free_slots = i32(layer, RING);
        d.n_free = i32(layer, N_FREE);
        d.err = i32(layer, ERR);
        const std::size_t cap = layers_[layer].capacity;
        d.capacity = cap == std::numeric_limits<std::size_t>::max() ? 0 : static_cast<int>(cap);
        d.slots_per_unit = nbs_;
        d.free_head = i32(layer, HEAD);
        d.free_owner = i32(layer, OWNER);
        d.warm = i32(layer, WARM);
        return d;
    }
    void sync_d2h(void* h, const void* d, std::size_t bytes) const {
        detail::cuda(cudaMemcpyAsync(h, d, bytes, cudaMemcpyDeviceToHost, st_), "TieredKvCache: read back");
        detail::cuda(cudaStreamSynchronize(st_), "TieredKvCache: read back");
    }
    std::vector<uint8_t> device_tier(std::size_t layer) const {
        std::vector<uint8_t> h(nbs_);
        sync_d2h(h.data(), tier_dev(layer), h.size());
        return h;
    }
    std::vector<int32_t> device_i32(std::size_t layer, Field f) const {
        std::vector<int32_t> h(nbs_);
        sync_d2h(h.data(), i32(layer, f), h.size() * 4);
        return h;
    }
    void clear_err(std::size_t layer) {
        const int32_t z = 0;
        detail::cuda(cudaMemcpyAsync(i32(layer, ERR), &z, 4, cudaMemcpyHostToDevice, st_), "TieredKvCache");
        detail::cuda(cudaStreamSynchronize(st_), "TieredKvCache");
    }
    void check_err(std::size_t layer, const char* what) {
        int32_t err = 0;
        sync_d2h(&err, i32(layer, ERR), 4);
        if (err != 0) {
            clear_err(layer);
            throw std::runtime_error(std::string("scout_b200::TieredKvCache: ") + what + ": device error " +
                                     std::to_string(err));
        }
    }
    void place(std::size_t layer, const BlockIdSet& keep) {
        std::vector<int32_t> h(keep.begin(), keep.end());
        const int32_t n = static_cast<int32_t>(h.size());
        detail::DevBuf dk((h.size() ? h.size() : 1) * 4), dn(4);
        if (!h.empty())
            detail::cuda(cudaMemcpyAsync(dk.p, h.data(), h.size() * 4, cudaMemcpyHostToDevice, st_), "place");
        detail::cuda(cudaMemcpyAsync(dn.p, &n, 4, cudaMemcpyHostToDevice, st_), "place");
        scout_tier_layer d = desc(layer);
        detail::check(scout_tier_place(&d, 1, nbs_, ntok_dev(layer), dk.as<int32_t>(), dn.as<int32_t>(),
                                       std::max<int>(n, 1), nullptr, st_));
        detail::cuda(cudaStreamSynchronize(st_), "place");
        check_err(layer, "place");
    }
    // build_digest (digest.hpp:34-60) in double on the host, the reference's fold
    DigestT host_digest(const MatT& keys, std::size_t block_id, std::size_t layer) const {
        DigestT d;
        d.method = method_;
        d.block_id = block_id;
        d.layer = layer;
        const std::size_t cols = keys.cols;
        if (detail::is_minmax(method_)) {
            d.lo.assign(keys.row(0), keys.row(0) + cols);
            d.hi = d.lo;
            for (std::size_t r = 1; r < keys.rows; ++r)
                for (std::size_t c = 0; c < cols; ++c) {
                    d.lo[c] = std::min(d.lo[c], keys.row(r)[c]);
                    d.hi[c] = std::max(d.hi[c], keys.row(r)[c]);
                }
        } else {
            d.mean.assign(cols, 0.0);
            for (std::size_t r = 0; r < keys.rows; ++r)
                for (std::size_t c = 0; c < cols; ++c) d.mean[c] += keys.row(r)[c];
            for (std::size_t c = 0; c < cols; ++c) d.mean[c] /= static_cast<double>(keys.rows);
        }
        return d;
    }

    std::size_t head_dim_;
    MethodT method_;
    int nbs_;
    std::vector<LayerState> layers_;
    std::vector<TicketT> in_flight_;  // the host ledger: which layers begin_layer must visit
    std::size_t clock_step_ = 0, clock_layer_ = 0;
    int n_tickets_ = 0;
    void* dev_ = nullptr;
    std::size_t per_layer_ = 0;
    cudaStream_t st_ = nullptr;
    int32_t* scratch_ = nullptr;  // [2 * nbs + 16] id lists / tables read back
};

using TieredKvCache = TieredKvCacheT<>;

}  // namespace scout_b200
