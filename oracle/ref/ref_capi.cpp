// TEST INFRASTRUCTURE — NOT PRODUCT CODE.
//
// The reference library ITSELF (the unmodified sources /root/reference/proj/src/*.cpp,
// compiled against the Eigen shim in oracle/ref/Eigen) behind the same C ABI as the
// restatement (oracle/louver_oracle.h), so oracle/pyoracle.py can load either build:
// oracle/liblouver_oracle.so (restatement, travels everywhere) or
// oracle/_ref/liblouver_ref.so (the reference, built here from /root/reference by
// oracle/Makefile; git-ignored). tests/test_oracle_vs_reference.py checks one
// against the other; bench.py --impl reference times this build when present.
#include <algorithm>
#include <cstring>
#include <functional>
#include <memory>
#include <stdexcept>
#include <string>
#include <vector>

#include "../louver_oracle.h"
#include "louver/bench.hpp"
#include "louver/cache.hpp"
#include "louver/index.hpp"
#include "louver/io.hpp"
#include "louver/query.hpp"
#include "louver/threshold.hpp"

using namespace louver;

namespace {

thread_local std::string g_err;

int guarded(const std::function<int()>& f) {
    try {
        return f();
    } catch (const std::out_of_range& e) {
        g_err = e.what();
        return LVO_ERANGE;
    } catch (const std::exception& e) {
        g_err = e.what();
        return LVO_EINVAL;
    }
}

Matrix rows_of(const float* p, int64_t n, int d) {
    Matrix m(n, d);
    if (n) std::memcpy(m.data(), p, sizeof(float) * size_t(n) * d);
    return m;
}

Vector vec_of(const float* p, int d) {
    Vector v(d);
    std::memcpy(v.data(), p, sizeof(float) * d);
    return v;
}

KeyStore store_of(const float* keys, const float* values, int64_t n, int d) {
    Matrix k = rows_of(keys, n, d);
    Matrix v = values ? rows_of(values, n, d) : Matrix(n, d);
    return KeyStore(std::move(k), std::move(v));
}

BuildConfig config_of(const lvo_build_config* c) {
    BuildConfig b;
    b.S = c->S;
    b.r = c->r;
    b.grouping = static_cast<GroupingStrategy>(c->grouping);
    b.enclosing = static_cast<EnclosureKind>(c->enclosure);
    b.rng_seed = c->rng_seed;
    return b;
}

void copy_ids(const std::vector<KeyId>& ids, uint32_t* out, int64_t cap, int64_t* count) {
    if (count) *count = (int64_t)ids.size();
    if (out && !ids.empty()) std::memcpy(out, ids.data(), sizeof(uint32_t) * std::min<size_t>(ids.size(), cap));
}

}  // namespace

struct lvo_cache {
    std::unique_ptr<LouverCache> c;
};

struct lvo_reservoir {
    Reservoir r;
    lvo_reservoir(int64_t cap, uint64_t seed) : r((size_t)cap, seed) {}
};

extern "C" {

const char* lvo_last_error(void) { return g_err.c_str(); }

float lvo_dot(const float* a, const float* b, int64_t len) { return dot(a, b, len); }

int lvo_brute_force_range(const float* keys, int64_t n, int d, const float* q, float tau, int64_t limit,
                          uint32_t* out_ids, int64_t cap, int64_t* count) {
    return guarded([&] {
        const KeyStore st = store_of(keys, nullptr, n, d);
        const Vector qv = vec_of(q, d);
        copy_ids(brute_force_range(st, qv, tau, (size_t)limit), out_ids, cap, count);
        return LVO_OK;
    });
}

int lvo_exact_check(const float* keys, int64_t n, int d, const uint32_t* cand, int64_t ncand, const float* q,
                    float tau, uint32_t* out_ids, int64_t* count) {
    return guarded([&] {
        const KeyStore st = store_of(keys, nullptr, n, d);
        const Vector qv = vec_of(q, d);
        const auto ids = exact_check(st, std::span<const KeyId>(cand, (size_t)ncand), qv, tau);
        copy_ids(ids, out_ids, (int64_t)ids.size(), count);
        return LVO_OK;
    });
}

int lvo_layout(int d, int S, int* offsets) {
    return guarded([&] {
        const SubspaceLayout l(d, S);
        std::copy(l.offsets.begin(), l.offsets.end(), offsets);
        return LVO_OK;
    });
}

int lvo_scores(const float* keys, int64_t n, int d, const float* q, float* out) {
    for (int64_t j = 0; j < n; ++j) out[j] = dot(q, keys + j * d, d);
    return LVO_OK;
}

float lvo_kth_score(const float* keys, int64_t n, int d, const float* q, int64_t k) {
    std::vector<float> s((size_t)n);
    lvo_scores(keys, n, d, q, s.data());
    std::nth_element(s.begin(), s.begin() + (k - 1), s.end(), std::greater<float>());
    return s[(size_t)(k - 1)];
}

int lvo_sparse_attention(const float* keys, const float* values, int64_t n, int d, const uint32_t* buffer_ids,
                         int64_t nbuf, const uint32_t* sel_ids, int64_t nsel, const float* q, float scale,
                         float* out, float* weights, int64_t* ntok) {
    return guarded([&] {
        const KeyStore st = store_of(keys, values, n, d);
        const Vector qv = vec_of(q, d);
        for (int64_t i = 0; i < nbuf; ++i)
            if (buffer_ids[i] >= n) throw std::out_of_range("sparse_attention: id out of range");
        for (int64_t i = 0; i < nsel; ++i)
            if (sel_ids[i] >= n) throw std::out_of_range("sparse_attention: id out of range");
        const auto res = sparse_attention(st, std::span<const KeyId>(buffer_ids, (size_t)nbuf),
                                          std::span<const KeyId>(sel_ids, (size_t)nsel), qv, scale);
        if (!res) {
            if (ntok) *ntok = 0;
            return LVO_EMPTY;
        }
        if (ntok) *ntok = (int64_t)res->selected_ids.size();
        std::memcpy(out, res->output.data(), sizeof(float) * d);
        if (weights) std::memcpy(weights, res->weights.data(), sizeof(float) * res->weights.size());
        return LVO_OK;
    });
}

int lvo_cache_create(int d, const lvo_build_config* cfg, int64_t buffer_capacity, lvo_cache** out) {
    return guarded([&] {
        auto* c = new lvo_cache;
        try {
            c->c = std::make_unique<LouverCache>(d, config_of(cfg), (size_t)buffer_capacity);
        } catch (...) {
            delete c;
            throw;
        }
        *out = c;
        return LVO_OK;
    });
}

int lvo_cache_adopt(const float* keys, const float* values, int64_t n, int d, const lvo_build_config* cfg,
                    int64_t buffer_capacity, lvo_cache** out) {
    return guarded([&] {
        auto* c = new lvo_cache;
        try {
            c->c = std::make_unique<LouverCache>(store_of(keys, values, n, d), config_of(cfg), (size_t)buffer_capacity);
        } catch (...) {
            delete c;
            throw;
        }
        *out = c;
        return LVO_OK;
    });
}

void lvo_cache_destroy(lvo_cache* c) { delete c; }

int lvo_cache_push_key(lvo_cache* c, const float* k, const float* v) {
    return guarded([&] {
        const int d = c->c->store().dim();
        c->c->push_key(vec_of(k, d), vec_of(v, d));
        return LVO_OK;
    });
}

int lvo_cache_flush(lvo_cache* c) {
    return guarded([&] { return c->c->flush_buffer() ? LVO_OK : LVO_EMPTY; });
}

int64_t lvo_cache_n(const lvo_cache* c) { return (int64_t)c->c->store().n(); }
int64_t lvo_cache_indexed_count(const lvo_cache* c) { return (int64_t)c->c->indexed_count(); }
int64_t lvo_cache_flush_count(const lvo_cache* c) { return (int64_t)c->c->flush_count(); }

int64_t lvo_cache_groups(const lvo_cache* c, int s) {
    const auto& idx = c->c->index();
    if (s < 0 || s >= (int)idx.per_subspace.size()) return 0;
    return (int64_t)idx.per_subspace[s].groups.size();
}

int64_t lvo_cache_group_members(const lvo_cache* c, int s, int64_t g, uint32_t* out, int64_t cap) {
    const auto& idx = c->c->index();
    if (s < 0 || s >= (int)idx.per_subspace.size()) return 0;
    const auto& m = idx.per_subspace[s].groups[(size_t)g].members;
    std::memcpy(out, m.data(), sizeof(uint32_t) * std::min<size_t>(m.size(), (size_t)cap));
    return (int64_t)m.size();
}

int lvo_cache_query(const lvo_cache* c, const float* q, float tau, float scale, int algo, int strict,
                    uint32_t* selected, int64_t* nsel, uint32_t* retrieved, int64_t* nret, int64_t cap,
                    float* attn_out, int* has_attn, lvo_stats* stats) {
    return guarded([&] {
        const int d = c->c->store().dim();
        QueryRequest req;
        req.q = vec_of(q, d);
        req.tau = tau;
        req.scale = scale;
        const auto res = c->c->query(req, algo == 0 ? FilterAlgo::FullSubspace : FilterAlgo::Ta, strict != 0);
        copy_ids(res.selected, selected, cap, nsel);
        copy_ids(res.retrieved, retrieved, cap, nret);
        if (has_attn) *has_attn = res.attention ? 1 : 0;
        if (res.attention && attn_out) std::memcpy(attn_out, res.attention->output.data(), sizeof(float) * d);
        if (stats) {
            stats->groups_tested = res.stats.groups_tested;
            stats->keys_scanned = res.stats.keys_scanned;
            stats->f_scan = res.stats.f_scan;
            stats->gate_cost_equiv = res.stats.gate_cost_equiv;
            stats->ta_stop_depth = res.stats.ta_stop_depth ? *res.stats.ta_stop_depth : -1;
            stats->ta_stop_upper = res.stats.ta_stop_upper ? *res.stats.ta_stop_upper : 0.0;
        }
        return LVO_OK;
    });
}

int lvo_cache_candidates(const lvo_cache* c, const float* q, float tau, const float* tau_s, int algo,
                         uint32_t* ids, int64_t cap, int64_t* n, lvo_stats* stats) {
    return guarded([&] {
        const auto& idx = c->c->index();
        const int d = c->c->store().dim();
        QueryRequest req;
        req.q = vec_of(q, d);
        req.tau = tau;
        if (tau_s) req.tau_subspace = std::vector<Scalar>(tau_s, tau_s + idx.layout.S);
        const CandidateSet cs = algo == 0 ? query_full_subspace(idx, c->c->store(), req)
                                          : query_ta(idx, c->c->store(), req);
        copy_ids(cs.live_ids, ids, cap, n);
        if (stats) {
            stats->groups_tested = cs.stats.groups_tested;
            stats->keys_scanned = cs.stats.keys_scanned;
            stats->f_scan = cs.stats.f_scan;
            stats->gate_cost_equiv = cs.stats.gate_cost_equiv;
            stats->ta_stop_depth = cs.stats.ta_stop_depth ? *cs.stats.ta_stop_depth : -1;
            stats->ta_stop_upper = cs.stats.ta_stop_upper ? *cs.stats.ta_stop_upper : 0.0;
        }
        return LVO_OK;
    });
}

int lvo_cache_thresholds(const lvo_cache* c, const float* q, float tau, float* out) {
    return guarded([&] {
        const int d = c->c->store().dim();
        const auto t = derive_subspace_thresholds(c->c->index(), vec_of(q, d), tau);
        std::memcpy(out, t.data(), sizeof(float) * t.size());
        return LVO_OK;
    });
}

int lvo_cache_subspace(const lvo_cache* c, int s, uint32_t* assign, uint32_t* moff, uint32_t* mids, float* a,
                       float* b, float* radii, double* norm_bound) {
    return guarded([&] {
        const auto& idx = c->c->index();
        if (s < 0 || s >= (int)idx.per_subspace.size()) throw std::out_of_range("subspace");
        const auto& sb = idx.per_subspace[s];
        const std::size_t K = sb.groups.size();
        if (assign) std::memcpy(assign, sb.assignments.data(), sizeof(uint32_t) * sb.assignments.size());
        if (moff) std::memcpy(moff, sb.member_offsets.data(), sizeof(uint32_t) * sb.member_offsets.size());
        if (mids) std::memcpy(mids, sb.member_ids.data(), sizeof(uint32_t) * sb.member_ids.size());
        const bool box = idx.config.enclosing == EnclosureKind::Aabb;
        const auto& A = box ? sb.gate_lo : sb.gate_centers;
        for (std::size_t i = 0; a && i < A.size(); ++i) std::memcpy(a + i * K, A[i].data(), sizeof(float) * K);
        for (std::size_t i = 0; b && box && i < sb.gate_hi.size(); ++i)
            std::memcpy(b + i * K, sb.gate_hi[i].data(), sizeof(float) * K);
        if (radii && !box) std::memcpy(radii, sb.gate_radii.data(), sizeof(float) * K);
        if (norm_bound) *norm_bound = sb.norm_bound;
        return LVO_OK;
    });
}

int lvr_cache_save_index(const lvo_cache* c, const char* path) {
    return guarded([&] {
        save_index(path, c->c->index());
        return LVO_OK;
    });
}

int lvo_balanced_pca_tree(const float* points, int64_t m, int w, int r, uint32_t* out) {
    return guarded([&] {
        const Matrix p = rows_of(points, m, w);
        const auto a = balanced_pca_tree(p, r);
        std::memcpy(out, a.data(), sizeof(uint32_t) * a.size());
        return LVO_OK;
    });
}

int lvo_assign_groups(const float* points, int64_t m, int w, const lvo_build_config* cfg, int subspace,
                      uint32_t base_id, uint32_t* out) {
    return guarded([&] {
        const Matrix p = rows_of(points, m, w);
        const auto a = assign_groups(p, config_of(cfg), subspace, base_id);
        std::memcpy(out, a.data(), sizeof(uint32_t) * a.size());
        return LVO_OK;
    });
}

int lvo_enclose_group(const float* points, int64_t m, int w, int kind, float* center, float* radius, float* lo,
                      float* hi) {
    return guarded([&] {
        const Matrix p = rows_of(points, m, w);
        const Enclosure e = enclose_group(p, static_cast<EnclosureKind>(kind));
        if (e.kind == EnclosureKind::Aabb) {
            std::memcpy(lo, e.lo.data(), sizeof(float) * w);
            std::memcpy(hi, e.hi.data(), sizeof(float) * w);
        } else {
            std::memcpy(center, e.center.data(), sizeof(float) * w);
            *radius = e.radius;
        }
        return LVO_OK;
    });
}

lvo_reservoir* lvo_reservoir_create(int64_t capacity, uint64_t seed) {
    try {
        return new lvo_reservoir(capacity, seed);
    } catch (const std::exception& e) {
        g_err = e.what();
        return nullptr;
    }
}
void lvo_reservoir_destroy(lvo_reservoir* r) { delete r; }

int64_t lvo_reservoir_update(lvo_reservoir* r, uint32_t id) {
    // the reference samples (id, key); keys do not change which slot is written
    const std::vector<KeyId> before = r->r.ids();
    Vector k(1);
    k[0] = 0.0f;
    r->r.update(id, k);
    const auto& after = r->r.ids();
    if (after.size() > before.size()) return (int64_t)after.size() - 1;
    for (size_t s = 0; s < after.size(); ++s)
        if (after[s] != before[s]) return (int64_t)s;
    return -1;  // not admitted (ids are distinct in every caller, so a write always shows)
}
int64_t lvo_reservoir_size(const lvo_reservoir* r) { return (int64_t)r->r.size(); }
int64_t lvo_reservoir_seen(const lvo_reservoir* r) { return (int64_t)r->r.seen(); }
void lvo_reservoir_ids(const lvo_reservoir* r, uint32_t* out) {
    std::memcpy(out, r->r.ids().data(), sizeof(uint32_t) * r->r.size());
}

int lvo_estimate_tau(const float* keys, int64_t n, int d, const float* q, int variant, int m, double alpha,
                     float* tau) {
    return guarded([&] {
        Reservoir res(std::max<size_t>(1, (size_t)n), 0);
        for (int64_t j = 0; j < n; ++j) res.update((KeyId)j, vec_of(keys + j * d, d));
        OracleConfig cfg;
        cfg.variant = static_cast<OracleVariant>(variant);
        cfg.m = m;
        cfg.alpha = alpha;
        *tau = estimate_tau(res, vec_of(q, d), cfg);
        return LVO_OK;
    });
}

// io.cpp:145-206 generators (gaussian law), to pin the repo's synth streams.
int lvr_gen_synthetic(int64_t n, int d, uint64_t seed, int queries, float* out) {
    return guarded([&] {
        DistributionSpec spec;
        const Matrix m = queries ? gen_synthetic_queries((size_t)n, d, spec, seed) : gen_synthetic((size_t)n, d, spec, seed);
        std::memcpy(out, m.data(), sizeof(float) * size_t(n) * d);
        return LVO_OK;
    });
}

}  // extern "C"
