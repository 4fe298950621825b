/*
 * TEST INFRASTRUCTURE — NOT PRODUCT CODE.
 *
 * CPU oracle for the Louver decode hot path: a plain C++17 restatement (no
 * Eigen) of the reference library's L0-L3 layers, exported through a C ABI so
 * that pytest (ctypes) and bench.py's cpu_baseline / --impl reference legs can
 * drive it. Only tests/, __graft_entry__.smoke() and bench.py's CPU legs may
 * load this library; the product path (liblouver_b200.so) never links it.
 *
 * Every function cites the reference file:line it restates (paths relative to
 * /root/reference/proj). Parity is pinned by the reference's own known-answer
 * tests (tests/test_oracle_kat.py, each test citing the reference test it
 * ports); see DESIGN.md "Oracle".
 *
 * Conventions: row-major float32 [n][d] key/value matrices; ids are uint32
 * ascending; functions return 0 on success, LVO_EMPTY (1) when the
 * reference would return nullopt/false, and negative on argument errors
 * (message via lvo_last_error()).
 */
#ifndef LOUVER_ORACLE_H
#define LOUVER_ORACLE_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define LVO_OK 0
#define LVO_EMPTY 1
#define LVO_EINVAL (-1)
#define LVO_ERANGE (-2)

/* grouping: 0 contiguous, 1 interleaved, 2 random, 3 pca_tree  (types.hpp:16-21)
 * enclosure: 0 ball, 1 aabb, 2 span_ball                       (types.hpp:23-27) */
typedef struct {
    int S;
    int r;
    int grouping;
    int enclosure;
    uint64_t rng_seed;
} lvo_build_config;

typedef struct {
    int64_t groups_tested;
    int64_t keys_scanned;
    double f_scan;
    double gate_cost_equiv;
    int ta_stop_depth; /* -1 when the TA scan never halted early */
    double ta_stop_upper;
} lvo_stats;

const char* lvo_last_error(void);

/* core.hpp:17-21 normative dot */
float lvo_dot(const float* a, const float* b, int64_t len);

/* query.cpp:11-20; writes up to `cap` ids, returns the count via *count */
int lvo_brute_force_range(const float* keys, int64_t n, int d, const float* q, float tau,
                          int64_t limit, uint32_t* out_ids, int64_t cap, int64_t* count);

/* query.cpp:22-31: candidates filtered by dot >= tau, sorted ascending. */
int lvo_exact_check(const float* keys, int64_t n, int d, const uint32_t* cand, int64_t ncand,
                    const float* q, float tau, uint32_t* out_ids, int64_t* count);

/* core.hpp:35-54: offsets[S+1] of the subspace layout. */
int lvo_layout(int d, int S, int* offsets);

/* All normative scores dot(q, k_j), j in [0, n). Convenience for τ selection. */
int lvo_scores(const float* keys, int64_t n, int d, const float* q, float* out);

/* query.cpp:338-371 (selected ∪ buffer, sorted, deduplicated). out[d], weights[ntok]
 * (weights may be NULL). Returns LVO_EMPTY for an empty token set. */
int lvo_sparse_attention(const float* keys, const float* values, int64_t n, int d,
                         const uint32_t* buffer_ids, int64_t nbuf, const uint32_t* sel_ids,
                         int64_t nsel, const float* q, float scale, float* out,
                         float* weights, int64_t* ntok);

/* --- LouverCache (cache.hpp:21-63, cache.cpp:7-70) ------------------------ */
typedef struct lvo_cache lvo_cache;

int lvo_cache_create(int d, const lvo_build_config* cfg, int64_t buffer_capacity,
                     lvo_cache** out);
/* Adopting constructor (cache.hpp:31-36): index all n keys immediately. */
int lvo_cache_adopt(const float* keys, const float* values, int64_t n, int d,
                    const lvo_build_config* cfg, int64_t buffer_capacity, lvo_cache** out);
void lvo_cache_destroy(lvo_cache* c);
int lvo_cache_push_key(lvo_cache* c, const float* k, const float* v);
/* returns LVO_EMPTY when nothing was pending (cache.cpp:14) */
int lvo_cache_flush(lvo_cache* c);
int64_t lvo_cache_n(const lvo_cache* c);
int64_t lvo_cache_indexed_count(const lvo_cache* c);
int64_t lvo_cache_flush_count(const lvo_cache* c);
/* Group count of subspace s (0 when no index yet). */
int64_t lvo_cache_groups(const lvo_cache* c, int s);
/* Copy the members of group g of subspace s; returns count. */
int64_t lvo_cache_group_members(const lvo_cache* c, int s, int64_t g, uint32_t* out, int64_t cap);

/* algo: 0 FullSubspace, 1 Ta (cache.hpp:7). selected/retrieved are written up
 * to `cap` ids each; attention output (d floats) is written when has_attn. */
int lvo_cache_query(const lvo_cache* c, const float* q, float tau, float scale, int algo,
                    int strict, uint32_t* selected, int64_t* nsel, uint32_t* retrieved,
                    int64_t* nret, int64_t cap, float* attn_out, int* has_attn,
                    lvo_stats* stats);

/* The cache's index directly (cache.hpp:49-50 index()): the candidate set of
 * query_full_subspace (algo 0; tau_s[S] required) or query_ta (algo 1) with its stats
 * (query.cpp:82-303), derive_subspace_thresholds (query.cpp:305-336, out[S]), and one
 * subspace's arrays (index.hpp:29-52): assignments[indexed], member offsets[K + 1],
 * member ids[indexed], gate arrays [w][K] (a: centers or lo, b: hi), radii[K], norm_bound.
 * Any output pointer may be NULL. */
int lvo_cache_candidates(const lvo_cache* c, const float* q, float tau, const float* tau_s, int algo,
                         uint32_t* ids, int64_t cap, int64_t* n, lvo_stats* stats);
int lvo_cache_thresholds(const lvo_cache* c, const float* q, float tau, float* out);
int lvo_cache_subspace(const lvo_cache* c, int s, uint32_t* assign, uint32_t* moff, uint32_t* mids,
                       float* a, float* b, float* radii, double* norm_bound);

/* --- Index-level entry points used by tests ------------------------------- */
/* index.cpp:15-68; points [m][w]; out assignments[m] */
int lvo_balanced_pca_tree(const float* points, int64_t m, int w, int r, uint32_t* out);
/* index.cpp:70-102 */
int lvo_assign_groups(const float* points, int64_t m, int w, const lvo_build_config* cfg,
                      int subspace, uint32_t base_id, uint32_t* out);
/* index.cpp:104-137: kind 0 ball / 2 span: center[w], radius; kind 1: lo[w], hi[w] */
int lvo_enclose_group(const float* points, int64_t m, int w, int kind, float* center,
                      float* radius, float* lo, float* hi);

/* --- Threshold oracle (threshold.hpp:9-53, threshold.cpp:40-103). The bench
 *     itself passes a fixed τ = exact k-th largest normative score. ---------- */
/* Reservoir (threshold.hpp:29-50) over ids; update = threshold.cpp:40-55.
 * lvo_reservoir_update returns the position written, or -1. */
typedef struct lvo_reservoir lvo_reservoir;
lvo_reservoir* lvo_reservoir_create(int64_t capacity, uint64_t seed);
void lvo_reservoir_destroy(lvo_reservoir* r);
int64_t lvo_reservoir_update(lvo_reservoir* r, uint32_t id);
int64_t lvo_reservoir_size(const lvo_reservoir* r);
int64_t lvo_reservoir_seen(const lvo_reservoir* r);
void lvo_reservoir_ids(const lvo_reservoir* r, uint32_t* out);
/* estimate_tau (threshold.cpp:63-103) over the n sampled keys [n][d];
 * variant as OracleVariant (threshold.hpp:9): 0 max, 1 topk, 2 gap, 3 meanmax,
 * 4 budget. Returns LVO_EINVAL for the reference's invalid_argument cases. */
int lvo_estimate_tau(const float* keys, int64_t n, int d, const float* q, int variant, int m,
                     double alpha, float* tau);
/* k-th largest normative score (1-based k) over keys [0, n). */
float lvo_kth_score(const float* keys, int64_t n, int d, const float* q, int64_t k);

#ifdef __cplusplus
}
#endif
#endif
