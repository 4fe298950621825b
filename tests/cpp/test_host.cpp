// C++ host-layer parity test: include/louver_b200.hpp (the reference-shaped API)
// against the CPU oracle (oracle/louver_oracle.h, test infrastructure) on seeded
// synthetic streams with the reference laws (io.cpp:89-206).
//
// Mirrors the reference's own C++ tests: test_cache.cpp:102-144 (query vs
// brute force, strict toggle, flush-at-B), test_query.cpp:178-196 (attention
// known answers / nullopt), and test_core.cpp error behaviour.
// usage: test_host [--compile-only]
#include <algorithm>
#include <cmath>
#include <cstdio>
#include <cstring>
#include <string>
#include <vector>

#include "louver_b200.hpp"
#include "louver_oracle.h"

using namespace louver_b200;

static int failures = 0;
#define EXPECT(cond, ...)                                   \
    do {                                                    \
        if (!(cond)) {                                      \
            ++failures;                                     \
            std::printf("FAIL %s:%d: ", __FILE__, __LINE__); \
            std::printf(__VA_ARGS__);                       \
            std::printf("\n");                              \
        }                                                   \
    } while (0)

static float bf16_round(float x) {  // round to nearest even, as the device conversion
    uint32_t u;
    std::memcpy(&u, &x, 4);
    u = (u + 0x7fffu + ((u >> 16) & 1u)) & 0xffff0000u;
    std::memcpy(&x, &u, 4);
    return x;
}

static std::vector<uint32_t> oracle_range(const std::vector<float>& K, int64_t n, int d, const float* q, float tau) {
    std::vector<uint32_t> ids(static_cast<size_t>(n ? n : 1));
    int64_t cnt = 0;
    lvo_brute_force_range(K.data(), n, d, q, tau, n, ids.data(), n, &cnt);
    ids.resize(static_cast<size_t>(cnt));
    return ids;
}

static double rel_err(const float* a, const float* b, int d) {
    double num = 0, den = 0;
    for (int i = 0; i < d; ++i) {
        num += (double(a[i]) - b[i]) * (double(a[i]) - b[i]);
        den += double(b[i]) * b[i];
    }
    return std::sqrt(num) / std::max(std::sqrt(den), 1e-30);
}

static void test_cache_fp32() {
    const int d = 64;
    const int64_t n0 = 3000, extra = 200;
    std::vector<float> K((n0 + extra) * d), V((n0 + extra) * d), Q(4 * d);
    lv_synth_keys(n0 + extra, d, 11, K.data());
    lv_synth_keys(n0 + extra, d, 12, V.data());
    lv_synth_queries(4, d, 13, Q.data());
    KeyStore store(std::vector<float>(K.begin(), K.begin() + n0 * d), std::vector<float>(V.begin(), V.begin() + n0 * d), d);
    BuildConfig cfg;
    cfg.S = 4;
    cfg.r = 16;
    LouverCache cache(store, cfg, 64);
    EXPECT(cache.n() == (size_t)n0 && cache.indexed_count() == (size_t)n0, "adopt indexes everything");
    EXPECT(!cache.flush_buffer(), "empty flush returns false (cache.cpp:14)");
    for (int64_t j = n0; j < n0 + extra; ++j)
        cache.push_key({K.data() + j * d, (size_t)d}, {V.data() + j * d, (size_t)d});
    EXPECT(cache.flush_count() == (size_t)(extra / 64), "flush-at-B: %zu flushes", cache.flush_count());
    EXPECT(cache.pending_count() == (size_t)(extra % 64), "pending %zu", cache.pending_count());
    const int64_t n = n0 + extra;
    for (int qi = 0; qi < 4; ++qi) {
        const float* q = Q.data() + qi * d;
        const float tau = lvo_kth_score(K.data(), n, d, q, (n + 19) / 20);
        QueryRequest req;
        req.q.assign(q, q + d);
        req.tau = tau;
        for (int strict = 0; strict < 2; ++strict) {
            CacheQueryResult r = cache.query(req, FilterAlgo::Ta, strict != 0);
            const auto want = oracle_range(K, n, d, q, tau);
            EXPECT(r.selected == want, "q%d selected: %zu vs oracle %zu", qi, r.selected.size(), want.size());
            std::vector<uint32_t> ret;
            for (uint32_t id : want)
                if (id < cache.indexed_count()) ret.push_back(id);
            for (size_t j = cache.indexed_count(); j < (size_t)n; ++j) ret.push_back((uint32_t)j);
            EXPECT(r.retrieved == ret, "q%d retrieved", qi);
            const auto& att = strict ? r.selected : r.retrieved;
            std::vector<float> o(d);
            int64_t ntok = 0;
            const int rc = lvo_sparse_attention(K.data(), V.data(), n, d, nullptr, 0, att.data(), (int64_t)att.size(), q,
                                                req.effective_scale(), o.data(), nullptr, &ntok);
            EXPECT((rc == LVO_EMPTY) == !r.attention.has_value(), "q%d attention presence", qi);
            if (r.attention) EXPECT(rel_err(r.attention->output.data(), o.data(), d) <= 1e-4, "q%d attention", qi);
            if (r.attention) {  // AttentionResult::weights aligned with the attended ids (query.cpp:359-365)
                std::vector<float> w(att.size() ? att.size() : 1);
                lvo_sparse_attention(K.data(), V.data(), n, d, nullptr, 0, att.data(), (int64_t)att.size(), q,
                                     req.effective_scale(), o.data(), w.data(), &ntok);
                EXPECT(r.attention->weights.size() == att.size(), "q%d weights size", qi);
                double worst = 0.0;
                for (size_t i = 0; i < att.size() && i < r.attention->weights.size(); ++i)
                    worst = std::max(worst, std::fabs(double(r.attention->weights[i]) - w[i]) / (std::fabs(w[i]) + 1e-30));
                EXPECT(worst <= 1e-4, "q%d weights rel err %g", qi, worst);
            }
        }
        // exact_check (query.cpp:22-31): every stored id as the candidate list, reversed
        std::vector<KeyId> all(n);
        for (int64_t j = 0; j < n; ++j) all[j] = (KeyId)(n - 1 - j);
        EXPECT(exact_check(cache, all, {q, (size_t)d}, tau) == oracle_range(K, n, d, q, tau), "exact_check q%d", qi);
        // query_ta's candidate set on the grouped index: the oracle cache's, id for id, with its stats
        {
            lvo_build_config oc{4, 16, 3, 0, 0};  // S=4, r=16, PCA tree, ball
            lvo_cache* oca = nullptr;
            lvo_cache_adopt(K.data(), V.data(), n0, d, &oc, 64, &oca);
            for (int64_t j = n0; j < n; ++j) lvo_cache_push_key(oca, K.data() + j * d, V.data() + j * d);
            std::vector<uint32_t> ids(n);
            int64_t cnt = 0;
            lvo_stats ost{};
            lvo_cache_candidates(oca, q, tau, nullptr, 1, ids.data(), n, &cnt, &ost);
            ids.resize(cnt);
            const CandidateSet g = query_ta(cache, req);
            EXPECT(g.live_ids == ids && g.stats.keys_scanned == ost.keys_scanned &&
                       g.stats.ta_stop_depth.value_or(-1) == ost.ta_stop_depth,
                   "query_ta on the grouped index q%d: %zu vs oracle %zu", qi, g.live_ids.size(), ids.size());
            std::vector<float> ots(4);
            lvo_cache_thresholds(oca, q, tau, ots.data());
            EXPECT(derive_subspace_thresholds(cache, {q, (size_t)d}, tau, 4) == ots, "grouped thresholds q%d", qi);
            QueryRequest rq = req;
            rq.tau_subspace = ots;
            ids.assign(n, 0);
            lvo_cache_candidates(oca, q, tau, ots.data(), 0, ids.data(), n, &cnt, &ost);
            ids.resize(cnt);
            EXPECT(query_full_subspace(cache, rq, 4).live_ids == ids, "query_full_subspace on the grouped index q%d", qi);
            lvo_cache_destroy(oca);
        }
        // the device cells' candidate set: a superset of the indexed selected keys, within [0, indexed)
        const CandidateSet cs = detail::candidate_set(cache, req);
        const auto sel_all = oracle_range(K, n, d, q, tau);
        bool sup = true, inside = true;
        for (KeyId id : sel_all)
            if (id < cache.indexed_count() && !std::binary_search(cs.live_ids.begin(), cs.live_ids.end(), id)) sup = false;
        for (KeyId id : cs.live_ids)
            if (id >= cache.indexed_count()) inside = false;
        EXPECT(sup && inside && std::is_sorted(cs.live_ids.begin(), cs.live_ids.end()), "query_ta candidates q%d", qi);
        EXPECT(cs.stats.keys_scanned == (int64_t)cs.live_ids.size() && cs.stats.groups_tested > 0, "candidate stats");
        // derive_subspace_thresholds over the device cells (S other than the grouped index's):
        // S = 1 gives tau itself; S = 4 thresholds are safe for every selected key
        EXPECT(derive_subspace_thresholds(cache, {q, (size_t)d}, tau, 1)[0] == tau, "S=1 threshold");
        const auto ts = derive_subspace_thresholds(cache, {q, (size_t)d}, tau, 4);
        bool safe = ts.size() == 4;
        for (KeyId id : sel_all) {
            if (id >= cache.indexed_count()) continue;
            for (int s = 0; s < 4 && safe; ++s) {
                float part = 0.0f;  // the subspace's partial dot in the reference's order
                for (int c = s * (d / 4); c < (s + 1) * (d / 4); ++c) part += q[c] * K[(size_t)id * d + c];
                if (part < ts[s]) safe = false;
            }
        }
        EXPECT(safe, "derive_subspace_thresholds safe q%d", qi);
        const auto bf = brute_force_range(cache, {q, (size_t)d}, tau, (size_t)n);
        EXPECT(bf == oracle_range(K, n, d, q, tau), "brute_force_range q%d", qi);
    }
    // sparse_attention: nullopt on an empty set, weights sum to 1 otherwise (query.cpp:338-371)
    EXPECT(!sparse_attention(cache, {}, {}, {Q.data(), (size_t)d}, 0.125f).has_value(), "empty -> nullopt");
    std::vector<KeyId> sel = {5, 1, 5, 900};
    std::vector<KeyId> buf = {3100};
    auto a = sparse_attention(cache, buf, sel, {Q.data(), (size_t)d}, 0.125f);
    EXPECT(a && a->selected_ids == std::vector<KeyId>({1, 5, 900, 3100}), "sort-unique token set");
    if (a) {
        double s = 0;
        for (float w : a->weights) s += w;
        EXPECT(std::fabs(s - 1.0) < 1e-5, "weights sum %f", s);
    }
    // recall_at_k (query.cpp:374-383), store() (cache.hpp:49)
    EXPECT(recall_at_k(std::vector<KeyId>{4, 1, 2, 3}, std::vector<KeyId>{9, 4, 2}) == 0.5, "recall_at_k");
    bool threw_r = false;
    try {
        recall_at_k({}, std::vector<KeyId>{1});
    } catch (const std::invalid_argument&) {
        threw_r = true;
    }
    EXPECT(threw_r, "recall_at_k: k >= 1 required");
    const KeyStore st = cache.store();
    EXPECT(st.n() == (size_t)(n0 + extra) && std::memcmp(st.key_data(), K.data(), sizeof(float) * K.size()) == 0 &&
               std::memcmp(st.value_data(), V.data(), sizeof(float) * V.size()) == 0,
           "store() holds the stored rows");
    EXPECT(cache.index().r == 16 && cache.index().indexed_count == cache.indexed_count(), "index() view");
    bool threw_fs = false;
    try {
        QueryRequest rq;
        rq.q.assign(Q.begin(), Q.begin() + d);
        query_full_subspace(cache, rq, 4);
    } catch (const std::invalid_argument&) {
        threw_fs = true;
    }
    EXPECT(threw_fs, "query_full_subspace: tau_subspace required");
    // reference error behaviour
    bool threw = false;
    try {
        cache.push_key({K.data(), (size_t)(d - 1)}, {V.data(), (size_t)d});
    } catch (const std::invalid_argument&) {
        threw = true;
    }
    EXPECT(threw, "dimension mismatch -> std::invalid_argument");
    threw = false;
    try {
        QueryRequest bad;
        bad.q.assign(d + 1, 0.0f);
        cache.query(bad, FilterAlgo::Ta);
    } catch (const std::invalid_argument&) {
        threw = true;
    }
    EXPECT(threw, "query length mismatch -> std::invalid_argument");
    threw = false;
    try {
        BuildConfig c0;
        c0.S = 0;
        LouverCache bad(d, c0, 8);
    } catch (const std::invalid_argument&) {
        threw = true;
    }
    EXPECT(threw, "BuildConfig::validate -> std::invalid_argument");
}

static void test_layer_bf16() {
    const int d = 128, H = 2, G = 4, B = 1;
    const int64_t n = 4096;
    std::vector<float> K(H * n * d), V(H * n * d), Q(H * G * d);
    for (int h = 0; h < H; ++h) {
        lv_synth_keys(n, d, 100 + h, K.data() + h * n * d);
        lv_synth_keys(n, d, 200 + h, V.data() + h * n * d);
    }
    lv_synth_queries(H * G, d, 300, Q.data());
    for (auto* v : {&K, &V, &Q})
        for (float& x : *v) x = bf16_round(x);
    std::vector<float> tau(H * G);
    for (int hq = 0; hq < H * G; ++hq)
        tau[hq] = lvo_kth_score(K.data() + (hq / G) * n * d, n, d, Q.data() + hq * d, n / 20);
    BuildConfig cfg;
    cfg.S = 1;
    cfg.r = 16;
    cfg.grouping = GroupingStrategy::Contiguous;
    cfg.enclosing = EnclosureKind::Aabb;
    LouverLayer layer(d, H, G, B, n, cfg, 128, LV_BF16);
    layer.build(K.data(), V.data(), n, LV_F32, LV_HOST);
    float *dq, *dt, *dout;
    int32_t* dcnt;
    cudaMalloc(&dq, Q.size() * 4);
    cudaMalloc(&dt, tau.size() * 4);
    cudaMalloc(&dout, Q.size() * 4);
    cudaMalloc(&dcnt, H * G * 16);
    cudaMemset(dcnt, 0, H * G * 16);
    cudaMemcpy(dq, Q.data(), Q.size() * 4, cudaMemcpyHostToDevice);
    cudaMemcpy(dt, tau.data(), tau.size() * 4, cudaMemcpyHostToDevice);
    layer.query_device(dq, dt, dout, nullptr, nullptr, dcnt);
    std::vector<float> out(Q.size());
    std::vector<int32_t> cnt(H * G * 4);
    cudaMemcpy(out.data(), dout, out.size() * 4, cudaMemcpyDeviceToHost);
    cudaMemcpy(cnt.data(), dcnt, cnt.size() * 4, cudaMemcpyDeviceToHost);
    for (int hq = 0; hq < H * G; ++hq) {
        const float* Kh = K.data() + (hq / G) * n * d;
        const float* Vh = V.data() + (hq / G) * n * d;
        std::vector<uint32_t> ids(n);
        int64_t c = 0;
        lvo_brute_force_range(Kh, n, d, Q.data() + hq * d, tau[hq], n, ids.data(), n, &c);
        EXPECT(cnt[hq * 4 + 0] == c, "head %d selected count %d vs oracle %lld", hq, cnt[hq * 4], (long long)c);
        std::vector<float> o(d);
        int64_t ntok = 0;
        lvo_sparse_attention(Kh, Vh, n, d, nullptr, 0, ids.data(), c, Q.data() + hq * d,
                             (float)(1.0 / std::sqrt((double)d)), o.data(), nullptr, &ntok);
        EXPECT(rel_err(out.data() + hq * d, o.data(), d) <= 1e-4, "head %d attention rel err %g", hq,
               rel_err(out.data() + hq * d, o.data(), d));
    }
    // the host-buffer decode step (lv_query_layers) with mapped pinned buffers on a
    // non-default stream: the cached graph, called twice (capture, replay)
    float *hq, *ht, *ho;
    cudaHostAlloc(reinterpret_cast<void**>(&hq), Q.size() * 4, cudaHostAllocDefault);
    cudaHostAlloc(reinterpret_cast<void**>(&ht), tau.size() * 4, cudaHostAllocDefault);
    cudaHostAlloc(reinterpret_cast<void**>(&ho), Q.size() * 4, cudaHostAllocDefault);
    std::copy(Q.begin(), Q.end(), hq);
    std::copy(tau.begin(), tau.end(), ht);
    cudaStream_t st;
    cudaStreamCreateWithFlags(&st, cudaStreamNonBlocking);
    for (int rep = 0; rep < 2; ++rep) {
        std::fill(ho, ho + Q.size(), 0.0f);
        query_layers_host({&layer}, hq, ht, ho, st);
        double worst = 0.0, scale = 0.0;
        for (size_t i = 0; i < out.size(); ++i) {
            worst = std::max(worst, (double)std::fabs(ho[i] - out[i]));
            scale = std::max(scale, (double)std::fabs(out[i]));
        }
        EXPECT(worst <= 1e-5 * scale, "query_layers_host (call %d) vs query_device: max diff %g", rep, worst);
    }
    cudaStreamDestroy(st);
    cudaFreeHost(hq);
    cudaFreeHost(ht);
    cudaFreeHost(ho);
    cudaFree(dq);
    cudaFree(dt);
    cudaFree(dout);
    cudaFree(dcnt);
}

// threshold.hpp through the host layer: the reservoir's draws equal the oracle's,
// and the device estimate equals the oracle's for every variant (bit-exact).
static void test_threshold() {
    const int d = 64, n = 3000;
    std::vector<float> K((size_t)n * d);
    for (size_t i = 0; i < K.size(); ++i) K[i] = std::sin(0.37f * (float)i) + 0.01f * (float)(i % 97);
    KeyStore store(d);
    for (int j = 0; j < n; ++j) store.append({K.data() + (size_t)j * d, (size_t)d}, {K.data() + (size_t)j * d, (size_t)d});
    LouverCache cache(store, BuildConfig{1, 16, GroupingStrategy::Contiguous, EnclosureKind::Aabb, 0}, 128);
    Reservoir res(256, 42);
    lvo_reservoir* ref = lvo_reservoir_create(256, 42);
    for (int j = 0; j < n; ++j) {
        res.update((KeyId)j);
        lvo_reservoir_update(ref, (uint32_t)j);
    }
    std::vector<uint32_t> rid(256);
    lvo_reservoir_ids(ref, rid.data());
    EXPECT(res.ids() == rid, "reservoir draws equal the oracle's");
    std::vector<float> sample;
    for (uint32_t id : rid) sample.insert(sample.end(), K.begin() + (size_t)id * d, K.begin() + (size_t)(id + 1) * d);
    std::vector<float> q(d);
    for (int c = 0; c < d; ++c) q[c] = std::cos(0.11f * (float)c);
    const OracleConfig cfgs[] = {{OracleVariant::SampleMax, 2, 0.1}, {OracleVariant::SampleTopK, 7, 0.1},
                                 {OracleVariant::SampleGap, 2, 0.1}, {OracleVariant::SampleMeanMax, 2, 0.1},
                                 {OracleVariant::Budget, 2, 0.05}};
    for (const auto& cfg : cfgs) {
        float want = 0.0f;
        lvo_estimate_tau(sample.data(), 256, d, q.data(), (int)cfg.variant, cfg.m, cfg.alpha, &want);
        const float got = estimate_tau(cache, res, {q.data(), (size_t)d}, cfg);
        EXPECT(got == want, "estimate_tau variant %d: %g vs oracle %g", (int)cfg.variant, got, want);
    }
    bool threw = false;
    try {
        estimate_tau(cache, res, {q.data(), (size_t)d}, OracleConfig{OracleVariant::Budget, 2, 1.5});
    } catch (const std::invalid_argument&) {
        threw = true;
    }
    EXPECT(threw, "OracleConfig::validate -> std::invalid_argument");
    lvo_reservoir_destroy(ref);
}

// bench.hpp run_decode_sim through the host layer against the oracle's own loop
// (LouverCache::query + Reservoir + estimate_tau restated on the CPU).
static void test_decode_sim() {
    const int d = 16;
    const std::size_t steps = 300;
    std::vector<float> K(steps * d), V(steps * d), Q(steps * d);
    for (size_t i = 0; i < K.size(); ++i) {
        K[i] = std::sin(0.731f * (float)i) + 0.05f * std::cos(0.017f * (float)i);
        V[i] = std::cos(0.29f * (float)i);
        Q[i] = std::sin(1.37f * (float)i + 0.5f);
    }
    KeyStore rows(K, V, d);
    DecodeSimConfig cfg;
    cfg.build = BuildConfig{1, 16, GroupingStrategy::Contiguous, EnclosureKind::Aabb, 0};
    cfg.buffer_capacity = 32;
    cfg.threshold.oracle = OracleConfig{OracleVariant::Budget, 0, 0.2};
    cfg.reservoir_capacity = 64;
    cfg.seed = 3;
    cfg.verify = true;
    const MetricsReport rep = run_decode_sim(rows, {Q.data(), Q.size()}, cfg);
    EXPECT(rep.steps == steps && rep.violations == 0, "decode sim: %zu violations", rep.violations);
    EXPECT(rep.flushes == steps / 32, "decode sim flushes %zu", rep.flushes);
    // the oracle's loop (bench.cpp:71-120)
    lvo_build_config oc{1, 16, 0, 1, 0};
    lvo_cache* c = nullptr;
    lvo_cache_create(d, &oc, 32, &c);
    lvo_reservoir* res = lvo_reservoir_create(64, 3);
    double sel = 0, ret = 0, tau_sum = 0;
    std::vector<uint32_t> sb(steps + 1), rb(steps + 1), ids(64);
    std::vector<float> sample, attn(d);
    for (std::size_t t = 0; t < steps; ++t) {
        float tau = -INFINITY;
        const int64_t sz = lvo_reservoir_size(res);
        if (sz >= 2) {
            lvo_reservoir_ids(res, ids.data());
            sample.clear();
            for (int64_t i = 0; i < sz; ++i) sample.insert(sample.end(), K.begin() + ids[i] * d, K.begin() + (ids[i] + 1) * d);
            lvo_estimate_tau(sample.data(), sz, d, Q.data() + t * d, 4, 0, 0.2, &tau);
        }
        int64_t ns = 0, nr = 0;
        int has = 0;
        lvo_stats st{};
        lvo_cache_query(c, Q.data() + t * d, tau, 0.0f, 1, 0, sb.data(), &ns, rb.data(), &nr, (int64_t)sb.size(),
                        attn.data(), &has, &st);
        sel += (double)ns;
        ret += (double)nr;
        tau_sum += std::isfinite(tau) ? tau : 0.0;
        lvo_cache_push_key(c, K.data() + t * d, V.data() + t * d);
        lvo_reservoir_update(res, (uint32_t)t);
    }
    EXPECT(std::fabs(rep.mean_selected - sel / steps) < 1e-9, "mean selected %f vs oracle %f", rep.mean_selected,
           sel / steps);
    EXPECT(std::fabs(rep.mean_retrieved - ret / steps) < 1e-9, "mean retrieved %f vs oracle %f", rep.mean_retrieved,
           ret / steps);
    EXPECT(std::fabs(rep.mean_tau - tau_sum / steps) < 1e-9, "mean tau %f vs oracle %f", rep.mean_tau, tau_sum / steps);
    lvo_reservoir_destroy(res);
    lvo_cache_destroy(c);
}

int main(int argc, char** argv) {
    if (argc > 1 && std::strcmp(argv[1], "--compile-only") == 0) {
        std::printf("%s\n", lv_build_info());
        return 0;
    }
    try {
        test_cache_fp32();
        test_layer_bf16();
        test_threshold();
        test_decode_sim();
    } catch (const std::exception& e) {
        std::printf("FAIL exception: %s\n", e.what());
        return 2;
    }
    if (failures) {
        std::printf("%d failure(s)\n", failures);
        return 1;
    }
    std::printf("OK\n");
    return 0;
}
