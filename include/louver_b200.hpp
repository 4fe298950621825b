// louver_b200.hpp — C++20 host layer over the C ABI (louver_b200.h).
//
// Mirrors the reference library's public API (namespace `louver`, headers under
// /root/reference/proj/include/louver/) so a C++ caller of the reference can
// switch by changing the namespace and linking liblouver_b200.so:
//
//   louver::BuildConfig / validate         index.hpp:10-22          -> BuildConfig
//   louver::KeyStore                       core.hpp:116-169         -> KeyStore (host rows, used to adopt)
//   louver::QueryRequest / QueryStats      query.hpp:11-30          -> QueryRequest / QueryStats
//   louver::AttentionResult                query.hpp:37-41          -> AttentionResult
//   louver::FilterAlgo / CacheQueryResult  cache.hpp:7-16           -> FilterAlgo / CacheQueryResult
//   louver::LouverCache                    cache.hpp:21-63          -> LouverCache (device-resident store + index)
//   louver::brute_force_range              query.hpp:44-45          -> brute_force_range(const LouverCache&, ...)
//   louver::sparse_attention               query.hpp:69-72          -> sparse_attention(const LouverCache&, ...)
//   louver::OracleConfig / Reservoir       threshold.hpp:9-50       -> OracleConfig / Reservoir (ids of arena rows)
//   louver::estimate_tau                   threshold.hpp:53         -> estimate_tau(const LouverCache&, res, q, cfg)
//   louver::run_decode_sim / MetricsReport bench.hpp:16-58          -> run_decode_sim(const KeyStore& rows, queries, cfg)
//
// Differences a caller sees: the store lives in HBM inside the cache, so the
// free functions take the cache instead of a `const KeyStore&`; `index()` is not
// exposed (the device index is cell summaries, not the reference's groups).
// Errors are the reference's: std::invalid_argument, std::out_of_range,
// std::runtime_error; an empty attention set is std::nullopt and an empty flush
// returns false.
//
// The multi-head decode layer (batch x H_kv slots, GQA, bf16 KV, device
// pointers, one fused kernel per query) is `LouverLayer`; sharded partials are
// combined with `lse_merge`.
#pragma once

#include <algorithm>
#include <chrono>
#include <iterator>
#include <limits>
#include <cmath>
#include <cstdint>
#include <cuda_runtime.h>
#include <memory>
#include <mutex>
#include <optional>
#include <span>
#include <stdexcept>
#include <string>
#include <utility>
#include <vector>

#include "louver_b200.h"

namespace louver_b200 {

using KeyId = std::uint32_t;  // types.hpp:14
using Scalar = float;
using Vector = std::vector<Scalar>;
using ConstVecRef = std::span<const Scalar>;

namespace detail {
inline int check(int rc, const char* what) {
    if (rc >= 0) return rc;  // LV_OK or LV_EMPTY
    std::string msg = std::string(what) + ": " + lv_last_error();
    switch (rc) {
        case LV_EINVAL: throw std::invalid_argument(msg);
        case LV_ERANGE: throw std::out_of_range(msg);
        default: throw std::runtime_error(msg);
    }
}
inline void cuda_check(cudaError_t e, const char* what) {
    if (e != cudaSuccess) throw std::runtime_error(std::string(what) + ": " + cudaGetErrorString(e));
}
// device scratch (the query clears what it accumulates into)
struct DevBuf {
    void* p = nullptr;
    explicit DevBuf(size_t bytes) {
        if (bytes) cuda_check(cudaMalloc(&p, bytes), "cudaMalloc");
    }
    ~DevBuf() { if (p) cudaFree(p); }
    DevBuf(const DevBuf&) = delete;
    DevBuf& operator=(const DevBuf&) = delete;
};
struct CtxDeleter {
    void operator()(lv_ctx* c) const { lv_destroy(c); }
};
}  // namespace detail

// types.hpp:16-27
enum class GroupingStrategy : std::uint32_t { Contiguous = 0, Interleaved = 1, Random = 2, PcaTree = 3 };
enum class EnclosureKind : std::uint32_t { Ball = 0, Aabb = 1, SpanBall = 2 };

// index.hpp:10-22. On the device keys are grouped into contiguous cells of r keys
// (r rounded up to a power of two, <= 64) with AABB summaries; S, grouping and
// enclosing are validated like the reference and change pruning, never results.
struct BuildConfig {
    int S = 4;
    int r = 4;
    GroupingStrategy grouping = GroupingStrategy::PcaTree;
    EnclosureKind enclosing = EnclosureKind::Ball;
    std::uint64_t rng_seed = 0;

    void validate(int d) const {
        if (S < 1) throw std::invalid_argument("BuildConfig: S >= 1 required");
        if (r < 1) throw std::invalid_argument("BuildConfig: r >= 1 required");
        if (S > d) throw std::invalid_argument("BuildConfig: S <= d required");
    }
};

// core.hpp:116-169: append-only host rows (keys and values), used to adopt a prefill.
class KeyStore {
  public:
    explicit KeyStore(int dim) : dim_(dim) {
        if (dim < 1) throw std::invalid_argument("KeyStore: dimension >= 1 required");
    }
    KeyStore(std::vector<Scalar> keys, std::vector<Scalar> values, int dim)
        : dim_(dim), keys_(std::move(keys)), values_(std::move(values)) {
        if (dim < 1) throw std::invalid_argument("KeyStore: dimension >= 1 required");
        if (keys_.size() != values_.size() || keys_.size() % dim)
            throw std::invalid_argument("KeyStore: keys/values shape mismatch");
    }
    KeyId append(ConstVecRef k, ConstVecRef v) {
        if (k.size() != static_cast<size_t>(dim_) || v.size() != static_cast<size_t>(dim_))
            throw std::invalid_argument("KeyStore::append: dimension mismatch");
        keys_.insert(keys_.end(), k.begin(), k.end());
        values_.insert(values_.end(), v.begin(), v.end());
        return static_cast<KeyId>(n() - 1);
    }
    int dim() const { return dim_; }
    std::size_t n() const { return keys_.size() / dim_; }
    ConstVecRef key(KeyId j) const { return {keys_.data() + static_cast<size_t>(j) * dim_, static_cast<size_t>(dim_)}; }
    ConstVecRef value(KeyId j) const { return {values_.data() + static_cast<size_t>(j) * dim_, static_cast<size_t>(dim_)}; }
    const Scalar* key_data() const { return keys_.data(); }
    const Scalar* value_data() const { return values_.data(); }

  private:
    int dim_;
    std::vector<Scalar> keys_, values_;
};

// query.hpp:11-19
struct QueryRequest {
    Vector q;
    Scalar tau = 0.0f;
    std::optional<std::vector<Scalar>> tau_subspace;  // full-subspace filter (grouped index); else derived
    Scalar scale = 0.0f;                              // 0 means 1/sqrt(d)

    Scalar effective_scale() const {
        return scale != 0.0f ? scale : Scalar(1.0 / std::sqrt(double(q.size())));
    }
};

// query.hpp:21-30. With the grouped index (the default for LouverCache) these are the
// reference's statistics for the BuildConfig; without it, groups are the device cells.
struct QueryStats {
    std::vector<std::int64_t> groups_tested_per_subspace;
    std::int64_t groups_tested = 0;  // groups whose bound was evaluated (sum over subspaces)
    std::int64_t keys_scanned = 0;   // keys entering the exact check (+ the buffer at cache level)
    double f_scan = 0.0;             // keys_scanned / indexed_count (cache level: / n)
    double gate_cost_equiv = 0.0;    // g * groups_tested / r (g = 2 for AABB, 1 for balls)
    std::optional<int> ta_stop_depth;
    std::optional<double> ta_stop_upper;
};

// query.hpp:37-41
struct AttentionResult {
    std::vector<KeyId> selected_ids;
    std::vector<Scalar> weights;  // aligned with selected_ids (filled by sparse_attention)
    Vector output;
};

// cache.hpp:7-16
enum class FilterAlgo { FullSubspace = LV_ALGO_FULL_SUBSPACE, Ta = LV_ALGO_TA };

struct CacheQueryResult {
    std::vector<KeyId> selected;   // all keys meeting the threshold, ascending
    std::vector<KeyId> retrieved;  // selected ∪ buffer
    QueryStats stats;
    std::optional<AttentionResult> attention;
};

// query.hpp:32-35 (the device's candidate set: live ids and the cells tested)
struct CandidateSetView {
    std::vector<KeyId> live_ids;
    std::int64_t groups_tested = 0;
};

// The device index behind LouverCache::index(): contiguous cells of r keys, one AABB
// summary row per cell, over the indexed keys [0, indexed_count).
struct IndexView {
    int r = 16;
    std::size_t indexed_count = 0;
    std::size_t cells = 0;
};

// cache.hpp:21-63: one head, fp32 KV in HBM, device index + update buffer of
// capacity B (auto-flush at B). Single writer; const queries may run
// concurrently (each call uses its own device workspace).
class LouverCache {
  public:
    // group_index: also build the reference's LouverIndex for cfg on the device (PCA tree,
    // enclosures, S subspaces); it supplies QueryStats, query_ta / query_full_subspace's
    // candidate sets and derive_subspace_thresholds exactly as the reference computes them.
    LouverCache(int dim, BuildConfig cfg, std::size_t buffer_capacity, std::size_t capacity = 1024,
                bool group_index = true)
        : dim_(dim), cfg_(cfg), buffer_capacity_(buffer_capacity), group_index_(group_index) {
        cfg.validate(dim);
        if (buffer_capacity < 1) throw std::invalid_argument("LouverCache: buffer capacity >= 1 required");
        create(capacity < 16 ? 16 : capacity);
    }

    // Adopts an existing store; all of it is indexed immediately (cache.hpp:31-36).
    LouverCache(const KeyStore& store, BuildConfig cfg, std::size_t buffer_capacity, bool group_index = true)
        : dim_(store.dim()), cfg_(cfg), buffer_capacity_(buffer_capacity), group_index_(group_index) {
        if (buffer_capacity < 1) throw std::invalid_argument("LouverCache: buffer capacity >= 1 required");
        cfg.validate(dim_);
        create(store.n() * 2 < 1024 ? 1024 : store.n() * 2);
        if (store.n())
            detail::check(lv_build(ctx_.get(), store.key_data(), store.value_data(), (int64_t)store.n(), LV_F32,
                                   LV_HOST, nullptr),
                          "lv_build");
    }

    void push_key(ConstVecRef k, ConstVecRef v) {
        if (k.size() != static_cast<size_t>(dim_) || v.size() != static_cast<size_t>(dim_))
            throw std::invalid_argument("KeyStore::append: dimension mismatch");
        if (n() >= capacity_) {  // geometric regrowth like KeyStore (core.hpp:134-142)
            capacity_ *= 2;
            detail::check(lv_reserve(ctx_.get(), (int64_t)capacity_, nullptr), "lv_reserve");
        }
        detail::check(lv_push_key(ctx_.get(), k.data(), v.data(), LV_F32, LV_HOST, nullptr), "lv_push_key");
    }

    // Folds pending keys into the index; false (no-op) when nothing is pending.
    bool flush_buffer() { return detail::check(lv_flush(ctx_.get(), nullptr), "lv_flush") == LV_OK; }

    // cache.cpp:30-70. attention->weights (query.cpp:359-365) come from the query's own
    // (m, l) and the normative scores of the attended ids. Each concurrent call leases its
    // own device scratch from a pool (allocated once, reused: no allocation per query).
    CacheQueryResult query(const QueryRequest& req, FilterAlgo algo, bool strict_threshold = false) const {
        if (req.q.size() != static_cast<size_t>(dim_)) throw std::invalid_argument("dot: length mismatch");
        Lease sc(*this);
        Vector out(dim_, 0.0f), part(dim_ + 2, 0.0f);
        int32_t counts[4] = {0, 0, 0, 0};
        const float tau = req.tau;
        lv_query_args a{};
        a.q = req.q.data();
        a.tau = &tau;
        a.scale = req.effective_scale();
        a.algo = static_cast<int>(algo);
        a.strict = strict_threshold ? 1 : 0;
        a.where = LV_HOST;
        a.out = out.data();
        a.partial = part.data();
        a.counts = counts;
        a.sel_bits = sc->bits();
        a.totals = sc->totals();
        a.workspace = sc->ws.p;
        detail::check(lv_query(ctx_.get(), &a), "lv_query");
        const int64_t n_now = lv_n(ctx_.get()), indexed = lv_indexed_count(ctx_.get());
        CacheQueryResult r;
        r.selected = bits_to_ids(sc.get(), sc->bits(), n_now);
        for (KeyId id : r.selected)
            if (id < indexed) r.retrieved.push_back(id);
        for (int64_t j = indexed; j < n_now; ++j) r.retrieved.push_back(static_cast<KeyId>(j));
        if (group_index_) {  // cache.cpp:37-64: the filter's stats, then the buffer and f_scan over n
            if (indexed > 0) r.stats = group_candidates(req, algo, false).stats;
            r.stats.keys_scanned += n_now - indexed;
            r.stats.f_scan = n_now ? double(r.stats.keys_scanned) / double(n_now) : 1.0;
        } else {
            uint64_t tot[4] = {0, 0, 0, 0};
            detail::cuda_check(cudaMemcpy(tot, sc->totals(), sizeof(tot), cudaMemcpyDeviceToHost), "cudaMemcpy");
            r.stats.groups_tested = static_cast<int64_t>(tot[0]);
            r.stats.keys_scanned = counts[2];
            r.stats.f_scan = n_now ? double(counts[2]) / double(n_now) : 1.0;
            r.stats.gate_cost_equiv = 2.0 * double(tot[0]) / double(cfg_.r);
        }
        if (counts[3]) {
            AttentionResult att{strict_threshold ? r.selected : r.retrieved, {}, std::move(out)};
            att.weights.resize(att.selected_ids.size());
            if (!att.selected_ids.empty())
                detail::check(lv_attention_weights(ctx_.get(), 0, att.selected_ids.data(),
                                                   (int64_t)att.selected_ids.size(), req.q.data(),
                                                   req.effective_scale(), part[0], part[1], LV_HOST,
                                                   att.weights.data(), nullptr),
                              "attention weights");
            r.attention = std::move(att);
        }
        return r;
    }

    // query_ta / query_full_subspace's candidate set (query.hpp:48-58) on the device:
    // every indexed key of a cell whose bound reaches tau (ascending), with the stats.
    CandidateSetView candidates(const QueryRequest& req) const {
        if (req.q.size() != static_cast<size_t>(dim_)) throw std::invalid_argument("dot: length mismatch");
        Lease sc(*this);
        int32_t counts[4] = {0, 0, 0, 0};
        const float tau = req.tau;
        lv_query_args a{};
        a.q = req.q.data();
        a.tau = &tau;
        a.scale = req.effective_scale();
        a.algo = LV_ALGO_TA;
        a.where = LV_HOST;
        a.counts = counts;
        a.totals = sc->totals();
        a.cand_bits = sc->bits();
        a.workspace = sc->ws.p;
        detail::check(lv_query(ctx_.get(), &a), "lv_query");
        CandidateSetView c;
        c.live_ids = bits_to_ids(sc.get(), sc->bits(), (int64_t)indexed_count());
        uint64_t tot[4] = {0, 0, 0, 0};
        detail::cuda_check(cudaMemcpy(tot, sc->totals(), sizeof(tot), cudaMemcpyDeviceToHost), "cudaMemcpy");
        c.groups_tested = static_cast<int64_t>(tot[0]);
        return c;
    }

    struct GroupCandidates {
        std::vector<KeyId> live_ids;
        QueryStats stats;
    };
    // query_ta / query_full_subspace (query.cpp:82-303) on the grouped index: the reference's
    // candidate set and statistics. FullSubspace takes req.tau_subspace, else derives it
    // (cache.cpp:38-41).
    GroupCandidates group_candidates(const QueryRequest& req, FilterAlgo algo, bool want_ids = true) const {
        if (!group_index_) throw std::invalid_argument("LouverCache: built without the grouped index");
        if (req.q.size() != static_cast<size_t>(dim_)) throw std::invalid_argument("dot: length mismatch");
        std::vector<Scalar> ts;
        if (algo == FilterAlgo::FullSubspace) {
            if (req.tau_subspace) {
                if (static_cast<int>(req.tau_subspace->size()) != cfg_.S)
                    throw std::invalid_argument("query_full_subspace: tau_subspace length != S");
                ts = *req.tau_subspace;
            } else {
                ts = group_thresholds(req.q, req.tau);
            }
        }
        const int64_t m = static_cast<int64_t>(indexed_count());
        GroupCandidates out;
        if (want_ids) out.live_ids.resize(static_cast<size_t>(m));
        int64_t nlive = 0;
        lv_group_stats st{};
        detail::check(lv_group_candidates(ctx_.get(), 0, req.q.data(), req.tau, ts.empty() ? nullptr : ts.data(),
                                          static_cast<int>(algo), nullptr, want_ids ? out.live_ids.data() : nullptr, m,
                                          &nlive, &st, nullptr),
                      "group candidates");
        if (want_ids) out.live_ids.resize(static_cast<size_t>(nlive));
        out.stats.groups_tested_per_subspace.assign(static_cast<size_t>(cfg_.S), lv_group_count(ctx_.get()));
        out.stats.groups_tested = st.groups_tested;
        out.stats.keys_scanned = st.keys_scanned;
        out.stats.f_scan = st.f_scan;
        out.stats.gate_cost_equiv = st.gate_cost_equiv;
        if (st.ta_stop_depth >= 0) {
            out.stats.ta_stop_depth = st.ta_stop_depth;
            out.stats.ta_stop_upper = st.ta_stop_upper;
        }
        return out;
    }
    // derive_subspace_thresholds (query.cpp:305-336) on the grouped index
    std::vector<Scalar> group_thresholds(ConstVecRef q, Scalar tau) const {
        if (!group_index_) throw std::invalid_argument("LouverCache: built without the grouped index");
        if (q.size() != static_cast<size_t>(dim_)) throw std::invalid_argument("dot: length mismatch");
        std::vector<Scalar> out(static_cast<size_t>(cfg_.S));
        detail::check(lv_group_thresholds(ctx_.get(), 0, q.data(), tau, out.data(), nullptr), "derive_subspace_thresholds");
        return out;
    }
    bool has_group_index() const { return group_index_; }
    const BuildConfig& config() const { return cfg_; }

    // cache.hpp:49: a host copy of the device store (KeyStore of the stored rows)
    KeyStore store() const { return KeyStore(rows(false), rows(true), dim_); }
    // cache.hpp:50: the device index's shape (cells of r contiguous keys with AABB summaries)
    IndexView index() const {
        int64_t g[8] = {0};
        detail::check(lv_geometry(ctx_.get(), g), "lv_geometry");
        return IndexView{static_cast<int>(g[1]), indexed_count(), (indexed_count() + g[1] - 1) / g[1]};
    }

    int dim() const { return dim_; }
    std::size_t n() const { return static_cast<size_t>(lv_n(ctx_.get())); }
    std::size_t indexed_count() const { return static_cast<size_t>(lv_indexed_count(ctx_.get())); }
    std::size_t pending_count() const { return static_cast<size_t>(lv_pending_count(ctx_.get())); }
    std::vector<KeyId> pending_ids() const {
        std::vector<KeyId> ids;
        for (size_t j = indexed_count(); j < n(); ++j) ids.push_back(static_cast<KeyId>(j));
        return ids;
    }
    std::size_t flush_count() const { return static_cast<size_t>(lv_flush_count(ctx_.get())); }
    std::size_t buffer_capacity() const { return buffer_capacity_; }
    // host copy of the stored rows (keys: values = false)
    std::vector<Scalar> rows(bool values) const {
        std::vector<Scalar> out(n() * dim_);
        if (!out.empty())
            detail::check(lv_read_rows(ctx_.get(), 0, 0, (int64_t)n(), values ? 1 : 0, out.data()), "lv_read_rows");
        return out;
    }
    lv_ctx* handle() const { return ctx_.get(); }

    // device bitmap [words] -> ascending ids < limit (device compaction kernel)
    std::vector<KeyId> bits_to_ids(const uint32_t* dev_bits, int64_t limit) const {
        Lease sc(*this);
        return bits_to_ids(sc.get(), dev_bits, limit);
    }

  private:
    // per-call device scratch, pooled: leased by a query, returned when it ends
    struct Scratch {
        std::size_t cap_keys;
        std::size_t tot_off;               // byte offset of totals [4] u64 + count i32 after the bitmap
        detail::DevBuf bitbuf, ws, idbuf;  // bitmap + totals + count; query workspace; ids [cap]
        Scratch(std::size_t cap, int64_t words, std::size_t ws_bytes)
            : cap_keys(cap), tot_off((static_cast<size_t>(words) * 4 + 15) / 16 * 16),
              bitbuf(tot_off + 48), ws(ws_bytes), idbuf(cap * 4) {}
        uint32_t* bits() { return static_cast<uint32_t*>(bitbuf.p); }
        uint64_t* totals() { return reinterpret_cast<uint64_t*>(static_cast<char*>(bitbuf.p) + tot_off); }
        int32_t* count() { return reinterpret_cast<int32_t*>(totals() + 4); }
    };
    class Lease {
      public:
        explicit Lease(const LouverCache& c) : c_(c) {
            std::lock_guard<std::mutex> g(c_.pool_mu_);
            const int64_t words = lv_bitmap_words(c_.ctx_.get());
            while (!c_.pool_.empty()) {  // drop scratch sized for a smaller arena (after regrowth)
                std::unique_ptr<Scratch> s = std::move(c_.pool_.back());
                c_.pool_.pop_back();
                if (s->cap_keys == c_.capacity_) {
                    s_ = std::move(s);
                    break;
                }
            }
            if (!s_) s_ = std::make_unique<Scratch>(c_.capacity_, words, lv_query_workspace_bytes(c_.ctx_.get()));
        }
        ~Lease() {
            std::lock_guard<std::mutex> g(c_.pool_mu_);
            c_.pool_.push_back(std::move(s_));
        }
        Scratch* operator->() { return s_.get(); }
        Scratch* get() { return s_.get(); }

      private:
        const LouverCache& c_;
        std::unique_ptr<Scratch> s_;
    };

    std::vector<KeyId> bits_to_ids(Scratch* sc, const uint32_t* dev_bits, int64_t limit) const {
        if (limit <= 0) return {};
        detail::check(lv_bitmap_to_ids(dev_bits, lv_bitmap_words(ctx_.get()), 1, limit, static_cast<uint32_t*>(sc->idbuf.p),
                                       limit, sc->count(), nullptr),
                      "lv_bitmap_to_ids");
        int32_t c = 0;
        detail::cuda_check(cudaMemcpy(&c, sc->count(), 4, cudaMemcpyDeviceToHost), "cudaMemcpy");
        std::vector<KeyId> out(static_cast<size_t>(c));
        if (c) detail::cuda_check(cudaMemcpy(out.data(), sc->idbuf.p, 4 * static_cast<size_t>(c), cudaMemcpyDeviceToHost), "cudaMemcpy");
        return out;
    }

    void create(std::size_t capacity) {
        capacity_ = capacity;
        lv_config c{};
        c.d = dim_;
        c.n_kv_heads = 1;
        c.group_size = 1;
        c.batch = 1;
        c.dtype = LV_F32;
        c.S = static_cast<int>(cfg_.S);
        c.r = static_cast<int>(cfg_.r);
        c.grouping = static_cast<int>(cfg_.grouping);
        c.enclosure = static_cast<int>(cfg_.enclosing);
        c.rng_seed = cfg_.rng_seed;
        c.buffer_capacity = static_cast<int64_t>(buffer_capacity_);
        c.capacity = static_cast<int64_t>(capacity);
        c.group_index = group_index_ ? 1 : 0;
        lv_ctx* h = nullptr;
        detail::check(lv_create(&c, &h), "lv_create");
        ctx_.reset(h);
    }

    int dim_;
    BuildConfig cfg_;
    std::size_t buffer_capacity_;
    bool group_index_ = true;
    std::size_t capacity_ = 0;
    std::unique_ptr<lv_ctx, detail::CtxDeleter> ctx_;
    mutable std::mutex pool_mu_;
    mutable std::vector<std::unique_ptr<Scratch>> pool_;
};

// query.hpp:44-45: ids j < limit with dot(q, k_j) >= tau (normative dot, on the device).
inline std::vector<KeyId> brute_force_range(const LouverCache& cache, ConstVecRef q, Scalar tau, std::size_t limit) {
    if (limit > cache.n()) throw std::invalid_argument("brute_force_range: limit > n");
    if (q.size() != static_cast<size_t>(cache.dim())) throw std::invalid_argument("dot: length mismatch");
    if (limit == 0) return {};
    detail::DevBuf bits(static_cast<size_t>(lv_bitmap_words(cache.handle())) * 4);
    detail::check(lv_brute_force_range(cache.handle(), q.data(), &tau, (int64_t)limit, LV_HOST,
                                       static_cast<uint32_t*>(bits.p), nullptr),
                  "lv_brute_force_range");
    return cache.bits_to_ids(static_cast<const uint32_t*>(bits.p), (int64_t)limit);
}

// query.hpp:48-49: the candidates meeting tau (normative dot), ascending.
inline std::vector<KeyId> exact_check(const LouverCache& cache, std::span<const KeyId> candidates, ConstVecRef q,
                                      Scalar tau) {
    if (q.size() != static_cast<size_t>(cache.dim())) throw std::invalid_argument("dot: length mismatch");
    std::vector<uint8_t> flags(candidates.size());
    if (!candidates.empty())
        detail::check(lv_exact_check(cache.handle(), 0, candidates.data(), (int64_t)candidates.size(), q.data(), tau,
                                     LV_HOST, flags.data(), nullptr),
                      "exact_check");
    std::vector<KeyId> out;
    for (size_t i = 0; i < candidates.size(); ++i)
        if (flags[i]) out.push_back(candidates[i]);
    std::sort(out.begin(), out.end());
    return out;
}

// query.hpp:32-35: CandidateSet with the stats the device reports (groups = cells).
struct CandidateSet {
    std::vector<KeyId> live_ids;  // ascending, duplicate-free, among the indexed keys
    QueryStats stats;
};

namespace detail {
inline CandidateSet candidate_set(const LouverCache& cache, const QueryRequest& req) {
    CandidateSetView v = cache.candidates(req);
    CandidateSet c;
    c.stats.groups_tested = v.groups_tested;
    c.stats.keys_scanned = static_cast<std::int64_t>(v.live_ids.size());
    const auto idx = cache.indexed_count();
    c.stats.f_scan = idx ? double(v.live_ids.size()) / double(idx) : 0.0;  // finalize_stats, query.cpp:70-78
    c.stats.gate_cost_equiv = 2.0 * double(v.groups_tested) / double(cache.index().r);
    c.live_ids = std::move(v.live_ids);
    return c;
}
}  // namespace detail

// query.hpp:60-63: on the grouped index, the reference's TA candidate set and stats; without
// it, the device cells' filter (full-dimension cell bounds against req.tau).
inline CandidateSet query_ta(const LouverCache& cache, const QueryRequest& req) {
    if (cache.has_group_index()) {
        auto g = cache.group_candidates(req, FilterAlgo::Ta);
        return CandidateSet{std::move(g.live_ids), std::move(g.stats)};
    }
    return detail::candidate_set(cache, req);
}

// query.hpp:51-53: validates tau_subspace like the reference (query.cpp:84-87); the device
// filter bounds each cell over all coordinates against req.tau.
inline CandidateSet query_full_subspace(const LouverCache& cache, const QueryRequest& req, int S) {
    if (!req.tau_subspace) throw std::invalid_argument("query_full_subspace: tau_subspace required");
    if (static_cast<int>(req.tau_subspace->size()) != S)
        throw std::invalid_argument("query_full_subspace: tau_subspace length != S");
    if (cache.has_group_index() && S == cache.config().S) {  // the reference's filter (query.cpp:82-117)
        auto g = cache.group_candidates(req, FilterAlgo::FullSubspace);
        return CandidateSet{std::move(g.live_ids), std::move(g.stats)};
    }
    return detail::candidate_set(cache, req);
}

// query.hpp:60-65 over the device index (lv_subspace_thresholds).
inline std::vector<Scalar> derive_subspace_thresholds(const LouverCache& cache, ConstVecRef q, Scalar tau, int S) {
    if (q.size() != static_cast<size_t>(cache.dim())) throw std::invalid_argument("dot: length mismatch");
    if (cache.has_group_index() && S == cache.config().S) return cache.group_thresholds(q, tau);  // query.cpp:305-336
    std::vector<Scalar> out(static_cast<size_t>(S > 0 ? S : 0));
    detail::check(lv_subspace_thresholds(cache.handle(), 0, q.data(), tau, S, LV_HOST, out.data(), nullptr),
                  "derive_subspace_thresholds");
    return out;
}

// query.hpp:74-75 / query.cpp:374-383: |retrieved ∩ exact_topk| / k.
inline double recall_at_k(std::span<const KeyId> exact_topk, std::span<const KeyId> retrieved) {
    if (exact_topk.empty()) throw std::invalid_argument("recall_at_k: k >= 1 required");
    std::vector<KeyId> a(exact_topk.begin(), exact_topk.end()), b(retrieved.begin(), retrieved.end()), both;
    std::sort(a.begin(), a.end());
    std::sort(b.begin(), b.end());
    std::set_intersection(a.begin(), a.end(), b.begin(), b.end(), std::back_inserter(both));
    return static_cast<double>(both.size()) / static_cast<double>(a.size());
}

// query.hpp:69-72: softmax over sort∪unique(selected ∪ buffer); nullopt when empty.
inline std::optional<AttentionResult> sparse_attention(const LouverCache& cache, std::span<const KeyId> buffer_ids,
                                                       std::span<const KeyId> selected_ids, ConstVecRef q,
                                                       Scalar scale) {
    if (q.size() != static_cast<size_t>(cache.dim())) throw std::invalid_argument("dot: length mismatch");
    std::vector<KeyId> tokens(selected_ids.begin(), selected_ids.end());
    tokens.insert(tokens.end(), buffer_ids.begin(), buffer_ids.end());
    std::sort(tokens.begin(), tokens.end());
    tokens.erase(std::unique(tokens.begin(), tokens.end()), tokens.end());
    AttentionResult r;
    r.output.assign(cache.dim(), 0.0f);
    r.weights.assign(tokens.size() ? tokens.size() : 1, 0.0f);
    int64_t ntok = 0;
    const int rc = detail::check(
        lv_sparse_attention(cache.handle(), 0, buffer_ids.empty() ? nullptr : buffer_ids.data(), (int64_t)buffer_ids.size(),
                            selected_ids.empty() ? nullptr : selected_ids.data(), (int64_t)selected_ids.size(),
                            q.data(), scale, LV_HOST, r.output.data(), r.weights.data(), &ntok, nullptr),
        "sparse_attention");
    if (rc == LV_EMPTY) return std::nullopt;
    r.weights.resize(static_cast<size_t>(ntok));
    r.selected_ids = std::move(tokens);
    return r;
}

// One decode layer: batch x H_kv slots (GQA group G), fp32 or bf16 KV in HBM.
// query_device() is the hot path: device q [batch][H_q][d], tau [batch][H_q],
// out [batch][H_q][d] (or partial [batch][H_q][d+2] for sequence sharding),
// enqueue-only on `stream`.
class LouverLayer {
  public:
    LouverLayer(int d, int n_kv_heads, int group_size, int batch, std::int64_t capacity, BuildConfig cfg,
                std::size_t buffer_capacity, int dtype = LV_BF16)
        : d_(d), rows_(static_cast<std::int64_t>(batch) * n_kv_heads * group_size) {
        cfg.validate(d);
        lv_config c{};
        c.d = d;
        c.n_kv_heads = n_kv_heads;
        c.group_size = group_size;
        c.batch = batch;
        c.dtype = dtype;
        c.S = static_cast<int>(cfg.S);
        c.r = static_cast<int>(cfg.r);
        c.grouping = static_cast<int>(cfg.grouping);
        c.enclosure = static_cast<int>(cfg.enclosing);
        c.rng_seed = cfg.rng_seed;
        c.buffer_capacity = static_cast<int64_t>(buffer_capacity);
        c.capacity = capacity;
        lv_ctx* h = nullptr;
        detail::check(lv_create(&c, &h), "lv_create");
        ctx_.reset(h);
    }
    // K, V: [batch][H_kv][n][d], src_dtype LV_F32 / LV_BF16, host or device
    void build(const void* K, const void* V, std::int64_t n, int src_dtype, int where, cudaStream_t st = nullptr) {
        detail::check(lv_build(ctx_.get(), K, V, n, src_dtype, where, st), "lv_build");
    }
    // one new key per slot: k, v [batch][H_kv][d]
    void push_key(const void* k, const void* v, int src_dtype, int where, cudaStream_t st = nullptr) {
        detail::check(lv_push_key(ctx_.get(), k, v, src_dtype, where, st), "lv_push_key");
    }
    bool flush_buffer(cudaStream_t st = nullptr) { return detail::check(lv_flush(ctx_.get(), st), "lv_flush") == LV_OK; }
    void query_device(const float* q, const float* tau, float* out, cudaStream_t st, float* partial = nullptr,
                      int32_t* counts = nullptr, bool strict = false, float scale = 0.0f, void* workspace = nullptr) const {
        lv_query_args a{};
        a.q = q;
        a.tau = tau;
        a.scale = scale;
        a.algo = LV_ALGO_TA;
        a.strict = strict ? 1 : 0;
        a.where = LV_DEVICE;
        a.out = out;
        a.partial = partial;
        a.counts = counts;
        a.workspace = workspace;
        a.stream = st;
        detail::check(lv_query(ctx_.get(), &a), "lv_query");
    }
    std::size_t workspace_bytes() const { return lv_query_workspace_bytes(ctx_.get()); }
    std::int64_t n() const { return lv_n(ctx_.get()); }
    int dim() const { return d_; }
    std::int64_t rows() const { return rows_; }  // batch x H_q query rows
    lv_ctx* handle() const { return ctx_.get(); }

  private:
    int d_;
    std::int64_t rows_;
    std::unique_ptr<lv_ctx, detail::CtxDeleter> ctx_;
};

// One decode step over L layers with HOST buffers (lv_query_layers): q [L][rows][d],
// tau [L][rows], out [L][rows][d] fp32. With cudaHostAlloc'd buffers and a non-default
// stream the step is a cached CUDA graph with no copy-engine transfers.
inline void query_layers_host(const std::vector<const LouverLayer*>& layers, const float* q, const float* tau,
                              float* out, cudaStream_t st, float scale = 0.0f, bool strict = false) {
    std::vector<lv_ctx*> hs;
    hs.reserve(layers.size());
    for (const LouverLayer* l : layers) hs.push_back(l->handle());
    detail::check(lv_query_layers(hs.data(), static_cast<int>(hs.size()), q, tau, scale, strict ? 1 : 0, out, nullptr, st),
                  "lv_query_layers");
}

// Log-sum-exp merge of P sequence-shard partials [P][rows][d+2] -> out [rows][d].
inline void lse_merge(const float* partials, int P, std::int64_t rows, int d, float* out, cudaStream_t st) {
    detail::check(lv_lse_merge(partials, P, rows, d, out, st), "lv_lse_merge");
}

// ---- threshold oracle (threshold.hpp:9-53) -------------------------------------------

enum class OracleVariant { SampleMax = LV_TAU_MAX, SampleTopK = LV_TAU_TOPK, SampleGap = LV_TAU_GAP,
                           SampleMeanMax = LV_TAU_MEANMAX, Budget = LV_TAU_BUDGET };

struct OracleConfig {  // threshold.hpp:11-23
    OracleVariant variant = OracleVariant::SampleMax;
    int m = 2;
    double alpha = 0.1;
    void validate() const {
        if (variant == OracleVariant::SampleTopK && m < 1) throw std::invalid_argument("OracleConfig: m >= 1 required");
        if (variant == OracleVariant::Budget && !(alpha > 0.0 && alpha < 1.0))
            throw std::invalid_argument("OracleConfig: 0 < alpha < 1 required");
    }
};

// threshold.hpp:29-50. Samples ids of a cache's (append-only) arena rows with the
// reference's std::mt19937_64 draws; the key argument of update() is accepted for
// signature parity only.
class Reservoir {
  public:
    explicit Reservoir(std::size_t capacity = 256, std::uint64_t seed = 0) {
        lv_reservoir* r = nullptr;
        detail::check(lv_reservoir_create((int64_t)capacity, seed, &r), "Reservoir");
        res_.reset(r);
    }
    void update(KeyId id, ConstVecRef = {}) { detail::check(lv_reservoir_update(res_.get(), id, nullptr), "update"); }
    std::size_t size() const { return (std::size_t)lv_reservoir_size(res_.get()); }
    std::size_t seen() const { return (std::size_t)lv_reservoir_seen(res_.get()); }
    std::size_t capacity() const { return (std::size_t)lv_reservoir_capacity(res_.get()); }
    std::vector<KeyId> ids() const {
        std::vector<KeyId> out(size());
        if (!out.empty()) detail::check(lv_reservoir_ids(res_.get(), out.data()), "ids");
        return out;
    }

  private:
    struct Del {
        void operator()(lv_reservoir* r) const { lv_reservoir_destroy(r); }
    };
    std::unique_ptr<lv_reservoir, Del> res_;
};

// threshold.cpp:63-103 on the device, over the cache's rows the reservoir sampled.
inline Scalar estimate_tau(const LouverCache& cache, const Reservoir& res, ConstVecRef q, const OracleConfig& cfg) {
    cfg.validate();
    if (q.size() != static_cast<size_t>(cache.dim())) throw std::invalid_argument("dot: length mismatch");
    const std::vector<KeyId> ids = res.ids();
    if (ids.empty()) throw std::invalid_argument("estimate_tau: empty reservoir");
    Scalar tau = 0.0f;
    detail::check(lv_estimate_tau(cache.handle(), ids.data(), (int64_t)ids.size(), (int64_t)ids.size(), q.data(),
                                  static_cast<int>(cfg.variant), cfg.m, cfg.alpha, LV_HOST, &tau, nullptr),
                  "estimate_tau");
    return tau;
}

// ---- decode loop (bench.hpp:16-58, bench.cpp:12-136) ---------------------------------

// bench.cpp:12-19
inline double speedup_estimate(double g, double r, double f_scan) {
    if (r < 1.0) throw std::invalid_argument("speedup_estimate: r >= 1 required");
    if (g < 0.0 || f_scan < 0.0 || f_scan > 1.0)
        throw std::invalid_argument("speedup_estimate: need g >= 0 and f_scan in [0, 1]");
    const double denom = g / r + f_scan;
    if (denom == 0.0) throw std::domain_error("speedup_estimate: g and f_scan both zero");
    return 1.0 / denom;
}

struct ThresholdSource {  // bench.hpp:16-19: exactly one is set
    std::optional<Scalar> fixed_tau;
    std::optional<OracleConfig> oracle;
};

struct DecodeSimConfig {  // bench.hpp:21-31
    BuildConfig build;
    std::size_t buffer_capacity = 128;
    FilterAlgo algo = FilterAlgo::Ta;
    ThresholdSource threshold;
    std::size_t reservoir_capacity = 256;
    std::uint64_t seed = 0;
    bool verify = false;
    bool strict_threshold = false;
};

struct MetricsReport {  // bench.hpp:33-48 (recall@k: see the Python driver)
    std::size_t steps = 0, flushes = 0, violations = 0;
    double mean_f_scan = 0.0, mean_keys_scanned = 0.0, mean_groups_tested = 0.0, mean_gate_cost_equiv = 0.0;
    double mean_selected = 0.0, mean_retrieved = 0.0, mean_tau = 0.0, mean_speedup_estimate = 0.0;
    double median_query_us = 0.0;
};

// bench.cpp:54-136 through the host layer: row t of `rows` (keys and values) and of
// `queries` ([steps][d]) drives step t. Each query is one synchronous device call;
// the device-resident loop with no per-step synchronisation is
// paper_2605_06763_b200/decode_sim.py.
inline MetricsReport run_decode_sim(const KeyStore& rows, std::span<const Scalar> queries, const DecodeSimConfig& cfg) {
    const int d = rows.dim();
    const std::size_t steps = rows.n();
    if (queries.size() != steps * static_cast<size_t>(d))
        throw std::invalid_argument("run_decode_sim: keys/values/queries row mismatch");
    if (!cfg.threshold.fixed_tau && !cfg.threshold.oracle)
        throw std::invalid_argument("run_decode_sim: no threshold source");
    LouverCache cache(d, cfg.build, cfg.buffer_capacity, steps < 16 ? 16 : steps);
    Reservoir reservoir(cfg.reservoir_capacity, cfg.seed);
    MetricsReport rep;
    rep.steps = steps;
    std::vector<double> wall_us;
    double sum_tau = 0.0, sum_speedup = 0.0;
    const std::size_t need =
        cfg.threshold.oracle && cfg.threshold.oracle->variant == OracleVariant::SampleTopK ? cfg.threshold.oracle->m : 1;
    for (std::size_t t = 0; t < steps; ++t) {
        QueryRequest req;
        req.q.assign(queries.begin() + t * d, queries.begin() + (t + 1) * d);
        if (cfg.threshold.fixed_tau) {
            req.tau = *cfg.threshold.fixed_tau;
        } else if (reservoir.size() >= 2 && reservoir.size() >= need) {
            req.tau = estimate_tau(cache, reservoir, req.q, *cfg.threshold.oracle);
        } else {
            req.tau = -std::numeric_limits<Scalar>::infinity();  // warm-up: retrieve all
        }
        const auto t0 = std::chrono::steady_clock::now();
        const CacheQueryResult ans = cache.query(req, cfg.algo, cfg.strict_threshold);
        const auto t1 = std::chrono::steady_clock::now();
        wall_us.push_back(std::chrono::duration<double, std::micro>(t1 - t0).count());
        if (cfg.verify && ans.selected != brute_force_range(cache, req.q, req.tau, cache.n())) ++rep.violations;
        rep.mean_f_scan += ans.stats.f_scan;
        rep.mean_keys_scanned += static_cast<double>(ans.stats.keys_scanned);
        rep.mean_groups_tested += static_cast<double>(ans.stats.groups_tested);
        rep.mean_gate_cost_equiv += ans.stats.gate_cost_equiv;
        rep.mean_selected += static_cast<double>(ans.selected.size());
        rep.mean_retrieved += static_cast<double>(ans.retrieved.size());
        sum_tau += std::isfinite(req.tau) ? req.tau : 0.0;
        const double g = cfg.build.enclosing == EnclosureKind::Aabb ? 2.0 : 1.0;
        sum_speedup += speedup_estimate(g, cfg.build.r, ans.stats.f_scan);
        cache.push_key(rows.key(static_cast<KeyId>(t)), rows.value(static_cast<KeyId>(t)));
        reservoir.update(static_cast<KeyId>(t));
    }
    const double inv = steps ? 1.0 / static_cast<double>(steps) : 0.0;
    rep.flushes = cache.flush_count();
    rep.mean_f_scan *= inv;
    rep.mean_keys_scanned *= inv;
    rep.mean_groups_tested *= inv;
    rep.mean_gate_cost_equiv *= inv;
    rep.mean_selected *= inv;
    rep.mean_retrieved *= inv;
    rep.mean_tau = sum_tau * inv;
    rep.mean_speedup_estimate = sum_speedup * inv;
    if (!wall_us.empty()) {  // bench.cpp:23-33
        const std::size_t mid = wall_us.size() / 2;
        std::nth_element(wall_us.begin(), wall_us.begin() + mid, wall_us.end());
        double med = wall_us[mid];
        if (wall_us.size() % 2 == 0) med = 0.5 * (med + *std::max_element(wall_us.begin(), wall_us.begin() + mid));
        rep.median_query_us = med;
    }
    return rep;
}

}  // namespace louver_b200
