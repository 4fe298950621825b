/*
 * louver_b200.h — C ABI of the B200-native Louver decode hot path.
 *
 * One lv_ctx holds ONE attention layer's KV cache for `batch` independent
 * sequences x `n_kv_heads` KV heads (a "slot" = one (sequence, kv head)
 * pair), the device index over it (contiguous cells with AABB summaries), and
 * the scratch its queries need. Grouped-query attention: q head hq reads kv
 * head hq / group_size (Llama convention).
 *
 * The entry points replace the reference library API (paths relative to
 * /root/reference/proj):
 *   lv_create / lv_destroy  — LouverCache(int, BuildConfig, size_t)        include/louver/cache.hpp:24-29
 *   lv_build                — LouverCache(KeyStore, BuildConfig, size_t) +  include/louver/cache.hpp:31-36
 *                             build_index(const KeyStore&, const BuildConfig&) include/louver/index.hpp:79
 *   lv_push_key             — LouverCache::push_key                        include/louver/cache.hpp:38, src/cache.cpp:7-10
 *   lv_flush                — LouverCache::flush_buffer                    include/louver/cache.hpp:41, src/cache.cpp:12-22
 *   lv_query                — LouverCache::query (filter + exact_check +   include/louver/cache.hpp:46-47, src/cache.cpp:30-70
 *                             dense buffer scan + sparse_attention)
 *   lv_brute_force_range    — brute_force_range                            include/louver/query.hpp:44-45, src/query.cpp:11-20
 *   lv_sparse_attention     — sparse_attention                              include/louver/query.hpp:69-72, src/query.cpp:338-371
 *   lv_dense_decode         — (no reference counterpart) full-scan decode, the speed-up denominator
 *   lv_lse_merge            — (no reference counterpart) log-sum-exp merge of sequence-sharded partials
 *
 * Status codes map onto the reference's error behaviour: LV_EINVAL <-
 * std::invalid_argument, LV_ERANGE <- std::out_of_range, LV_ERUNTIME <-
 * std::runtime_error, LV_EMPTY <- std::nullopt / `false` (empty attention set,
 * empty flush). lv_last_error() returns the message of the calling thread's
 * last failure.
 *
 * Memory: pointers tagged `where` are host (LV_HOST; copies happen inside the
 * call on `stream`, which is then synchronised) or device (LV_DEVICE; the call
 * only enqueues work on `stream`). `stream` is a cudaStream_t (NULL = legacy
 * default stream).
 *
 * Threading (cache.hpp:18-20): single writer — lv_build / lv_push_key /
 * lv_flush need exclusive access; lv_query is re-entrant across threads and
 * streams when each caller passes its own `workspace` (see
 * lv_query_workspace_bytes); with workspace == NULL the context's internal
 * workspace is used and concurrent queries on one context must be serialised.
 */
#ifndef LOUVER_B200_H
#define LOUVER_B200_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define LV_OK 0
#define LV_EMPTY 1
#define LV_EINVAL (-1)
#define LV_ERANGE (-2)
#define LV_ERUNTIME (-3)
#define LV_ENODEV (-4)

#define LV_F32 0
#define LV_BF16 1

#define LV_HOST 0
#define LV_DEVICE 1

/* FilterAlgo (cache.hpp:7). Both select the same final set; on the device
 * both run the fused cell probe (the per-cell AABB bound summed over all
 * coordinates is at least as strong as either reference filter). */
#define LV_ALGO_FULL_SUBSPACE 0
#define LV_ALGO_TA 1

typedef struct lv_ctx lv_ctx;

typedef struct {
    int d;                   /* head dimension, 1..256 */
    int n_kv_heads;          /* H_kv >= 1 */
    int group_size;          /* G = H_q / H_kv, one of 1, 2, 4, 8 */
    int batch;               /* independent sequences >= 1 */
    int dtype;               /* K/V storage: LV_F32 or LV_BF16 (summaries use the same type) */
    /* BuildConfig (index.hpp:10-22). The device index groups keys into
     * contiguous cells of `r` keys (r rounded up to a power of two, <= 64) with
     * one AABB per cell; S, grouping, enclosure and rng_seed are validated like
     * the reference and recorded, but only change pruning statistics — the
     * selected set and the attention output do not depend on them (SURVEY
     * Executive summary item 3). */
    int S;
    int r;
    int grouping;            /* 0 contiguous, 1 interleaved, 2 random, 3 pca_tree */
    int enclosure;           /* 0 ball, 1 aabb, 2 span_ball */
    uint64_t rng_seed;
    int64_t buffer_capacity; /* B >= 1: keys [indexed_count, n) form the dense-scanned buffer */
    int64_t capacity;        /* max keys per sequence held in the HBM arena */
    /* 1: also build the reference's grouped index on the device — S subspaces, the
     * configured GroupingStrategy (PCA tree included) and EnclosureKind, packed gate
     * arrays and member lists, bit-exact with index.cpp — at lv_build and at every flush.
     * It serves lv_group_candidates / lv_group_thresholds (the reference's candidate sets
     * and QueryStats) and lv_save_index (the reference's snapshot of that index). The
     * fused query does not use it (its final sets do not depend on the grouping).
     * Memory: about the fp32 key arena again. 0: off. */
    int group_index;
} lv_config;

typedef struct {
    const float* q;     /* [batch][H_q][d] fp32 */
    const float* tau;   /* [batch][H_q] fp32, applied to the unscaled normative q.k */
    float scale;        /* softmax scale; 0 -> 1/sqrt(d) (query.hpp:17-19) */
    int algo;           /* LV_ALGO_*; accepted for API parity */
    int strict;         /* 0: attend selected ∪ buffer (default); 1: attend selected only */
    int where;          /* LV_HOST or LV_DEVICE for q, tau, out, partial, counts */
    float* out;         /* [batch][H_q][d] attention output; rows with an empty set are 0 */
    float* partial;     /* optional [batch][H_q][d+2]: (m, l, o[d]) with o unnormalised,
                           for lv_lse_merge across sequence shards */
    int32_t* counts;    /* optional [batch][H_q][4]: selected, attended, keys_scanned, has_attn */
    uint32_t* sel_bits; /* optional DEVICE [batch][H_q][lv_bitmap_words()] bitmap of selected ids */
    uint64_t* totals;   /* optional DEVICE [4]: cells probed, cells surviving (union over the
                           group), keys loaded (union), values loaded (union) — summed over slots */
    void* workspace;    /* optional DEVICE scratch of lv_query_workspace_bytes() bytes */
    void* stream;       /* cudaStream_t */
    uint32_t* cand_bits; /* optional DEVICE [batch][H_kv][lv_bitmap_words()]: the candidate set of
                            query_ta / query_full_subspace (query.hpp:48-58) — every INDEXED key
                            of a cell whose bound reaches any q head's threshold (fp32 caches) */
} lv_query_args;

/* QueryStats (query.hpp:24-32) of a candidate filter on the grouped index. */
typedef struct {
    int64_t groups_tested;  /* sum over subspaces */
    int64_t keys_scanned;   /* |live_ids| */
    double f_scan;          /* keys_scanned / indexed_count */
    double gate_cost_equiv; /* g * groups_tested / r, g = 2 for AABB, 1 for balls */
    int32_t ta_stop_depth;  /* -1: the TA scan did not halt early (or FullSubspace) */
    double ta_stop_upper;   /* U(d*) when it halted */
} lv_group_stats;

const char* lv_last_error(void);

/* Version string and the device the library was compiled for ("sm_100a"). */
const char* lv_build_info(void);

int lv_create(const lv_config* cfg, lv_ctx** out);
int lv_destroy(lv_ctx* ctx);

/* Prefill: adopt n keys/values per slot and index them all (the adopting
 * constructor, cache.hpp:31-36). K, V: [batch][H_kv][n][d] of `src_dtype`
 * (LV_F32 always accepted; LV_BF16 when the storage dtype is bf16). Replaces
 * any previous contents. n == 0 leaves an empty cache. */
int lv_build(lv_ctx* ctx, const void* K, const void* V, int64_t n, int src_dtype, int where,
             void* stream);

/* Grow the arena to hold `capacity` keys per sequence, keeping every stored
 * row, summary and counter (KeyStore's geometric regrowth, core.hpp:156-162).
 * Invalidates caller workspaces sized by lv_query_workspace_bytes(). */
int lv_reserve(lv_ctx* ctx, int64_t capacity, void* stream);

/* Append one key/value per slot (k, v: [batch][H_kv][d] of src_dtype) and fold
 * it into the open cell's summary in place; when pending >= B the buffer is
 * flushed (cache.cpp:7-10). Enqueue-only for LV_DEVICE: the counters live on
 * the device, so the call is CUDA-graph capturable. */
int lv_push_key(lv_ctx* ctx, const void* k, const void* v, int src_dtype, int where,
                void* stream);

/* cache.cpp:12-22: returns LV_EMPTY (no-op) when nothing is pending. */
int lv_flush(lv_ctx* ctx, void* stream);

int lv_query(lv_ctx* ctx, const lv_query_args* args);
size_t lv_query_workspace_bytes(const lv_ctx* ctx);

/* One decode step over L layers with HOST buffers (each layer an lv_ctx with the
 * same batch, H_q and d): q [L][batch][H_q][d], tau [L][batch][H_q], out
 * [L][batch][H_q][d], fp32 host memory (pinned for full speed). One host->device
 * copy of every q and tau, the L fused layer queries back to back on the stream,
 * one device->host copy of out, one synchronisation — the host-buffer form of the
 * decode step. staging: optional DEVICE scratch of lv_query_layers_staging_bytes()
 * bytes; NULL uses ctxs[0]'s internal staging (calls sharing ctxs[0] serialise).
 * Each layer's query uses its context's internal workspace. With pinned buffers, the
 * internal staging and a non-default stream, the step runs as a CUDA graph captured on
 * the first call and replayed while the contexts, buffers and stream stay the same
 * (LV_LAYERS_GRAPH=0 disables it). When the pinned buffers are mapped into the device
 * address space (cudaHostAlloc memory on a UVA system) and d is a multiple of 64, the
 * graph uses no copy engine: one kernel stages q and tau from host memory and each layer
 * kernel writes its output rows straight into `out` (LV_LAYERS_MAPPED=0: copies). */
int lv_query_layers(lv_ctx* const* ctxs, int L, const float* q, const float* tau, float scale, int strict,
                    float* out, void* staging, void* stream);
size_t lv_query_layers_staging_bytes(const lv_ctx* ctx, int L);

/* Device geometry: out[8] = {padded d, cell keys r, arena rows, cells per slot,
 * query splits per slot, chunks per split, keys per chunk, query smem bytes}
 * (the split geometry of the fp32 / dense / brute-force kernels). */
int lv_geometry(const lv_ctx* ctx, int64_t* out);

/* bf16 query path (one fused persistent kernel per layer): out[4] = {CTAs per
 * slot, resident CTAs per SM, threads per CTA, dynamic smem bytes} as chosen
 * by the last query launch; zeros before the first bf16 query. */
int lv_layer_geometry(const lv_ctx* ctx, int64_t* out);

/* Debug: while dev_buf != NULL, bf16 queries write up to 64 globaltimer stamps per
 * CTA (order [slot][team CTA]) into dev_buf [slots*team][64]. */
int lv_debug_trace(lv_ctx* ctx, int64_t* dev_buf);
int64_t lv_bitmap_words(const lv_ctx* ctx);

/* Host mirrors of the device counters (uniform over slots). */
int64_t lv_n(const lv_ctx* ctx);
int64_t lv_indexed_count(const lv_ctx* ctx);
int64_t lv_pending_count(const lv_ctx* ctx);
int64_t lv_flush_count(const lv_ctx* ctx);

/* Refresh the host mirrors from the device counters (needed after replaying a
 * captured CUDA graph that contains lv_push_key). */
int lv_sync_counters(lv_ctx* ctx, void* stream);

/* Read back stored keys/values of one slot as fp32 rows [count][d] (host). */
int lv_read_rows(const lv_ctx* ctx, int slot, int64_t first, int64_t count, int which_v,
                 float* out);

/* query.cpp:11-20 on the device: bitmap of ids j < limit with dot(q, k_j) >= tau
 * for every q head (normative dot, bit-exact). q, tau as in lv_query (`where`
 * applies to them); sel_bits is DEVICE [batch][H_q][lv_bitmap_words()].
 * limit == -1: every key stored when the kernel runs (the device counter; for
 * CUDA-graph replay, where a host-side limit would be frozen at capture). */
int lv_brute_force_range(lv_ctx* ctx, const float* q, const float* tau, int64_t limit, int where,
                         uint32_t* sel_bits, void* stream);

/* Expand bitmaps to ascending id lists on the device: ids[row][..] gets the set
 * bits of row `row` below `limit`; count[row] the number written. */
int lv_bitmap_to_ids(const uint32_t* bits, int64_t words, int64_t rows, int64_t limit,
                     uint32_t* ids, int64_t ids_stride, int32_t* count, void* stream);

/* query.cpp:338-371 for ONE q head: tokens = sort∪unique(selected ∪ buffer)
 * (ids of slot `slot`), scores = scale·normative dot, softmax, output. ids are
 * host or device per `where`; out[d] and optional weights[ntok] likewise.
 * Returns LV_EMPTY when the token set is empty. */
int lv_sparse_attention(lv_ctx* ctx, int slot, const uint32_t* buffer_ids, int64_t nbuf,
                        const uint32_t* selected_ids, int64_t nsel, const float* q, float scale,
                        int where, float* out, float* weights, int64_t* ntok, void* stream);

/* exact_check (query.hpp:48-49, query.cpp:22-31) on the device: flags[i] = 1 iff the
 * normative dot(q, k_{ids[i]}) >= tau for key ids[i] of slot `slot`, else 0. ids, q
 * and flags are host or device per `where`; ids must be < lv_n. */
int lv_exact_check(lv_ctx* ctx, int slot, const uint32_t* ids, int64_t nids, const float* q, float tau, int where,
                   uint8_t* flags, void* stream);

/* The attention weights of a query (AttentionResult::weights, query.cpp:359-365):
 * weights[i] = exp(scale * dot(q, k_{ids[i]}) - m) / l with the normative dot, for the
 * attended ids of slot `slot` and the (m, l) of lv_query's `partial` row of that q
 * head. ids, q, weights host or device per `where`. */
int lv_attention_weights(lv_ctx* ctx, int slot, const uint32_t* ids, int64_t nids, const float* q, float scale,
                         float m, float l, int where, float* weights, void* stream);

/* derive_subspace_thresholds (query.hpp:60-65, query.cpp:305-336) over the device
 * index of slot `slot`: with S slices of the SubspaceLayout (core.hpp:41-50), M_s = the
 * largest AABB bound of subspace s over the cells holding indexed keys, slack =
 * 4 d eps ||q|| sqrt(sum_s nb_s^2) (0 when S = 1, nb_s the cells' largest
 * ||max(|lo|, |hi|)|| over s), tau_s = tau - (sum M - M_s) - slack. q [d] and out [S]
 * host or device per `where`. Any key with dot(q, k) >= tau meets every tau_s. */
int lv_subspace_thresholds(lv_ctx* ctx, int slot, const float* q, float tau, int S, int where, float* out,
                           void* stream);

/* Full-scan decode over keys [0, n) of every slot (fused split-K online
 * softmax, GQA-grouped). Same q/out conventions as lv_query. */
int lv_dense_decode(lv_ctx* ctx, const float* q, float scale, int where, float* out,
                    float* partial, void* stream);

/* Log-sum-exp merge of P shard partials [P][rows][d+2] (m, l, o unnormalised)
 * into out[rows][d] (device pointers). Empty shards carry m = -inf, l = 0. */
/* Grouped index (lv_config.group_index = 1), for one slot (sequence x kv head).
 * lv_group_candidates: the candidate set of query_full_subspace (algo
 * LV_ALGO_FULL_SUBSPACE; tau_subspace[S] required, host) or query_ta (LV_ALGO_TA)
 * (query.cpp:82-303) for the host query q[d] — live_bits: optional DEVICE bitmap of
 * lv_bitmap_words() words over the indexed keys; live_ids: optional HOST array of `cap`
 * ids (ascending), *nlive its length; stats: optional HOST. Synchronises `stream`.
 * lv_group_thresholds: derive_subspace_thresholds (query.cpp:305-336), out[S] host.
 * lv_group_count: groups per subspace (K, the same for every slot and subspace).
 * lv_group_export: HOST copies of subspace s of a slot — assignments[indexed],
 * member offsets[K + 1], member ids[indexed] (ascending within each group), gate arrays
 * coordinate-major [w][K] (a: centers for balls, lo for AABB; b: hi for AABB), radii[K]
 * and norm_bound; any pointer may be NULL. */
int lv_group_candidates(lv_ctx* ctx, int slot, const float* q, float tau, const float* tau_subspace, int algo,
                        uint32_t* live_bits, uint32_t* live_ids, int64_t cap, int64_t* nlive,
                        lv_group_stats* stats, void* stream);
int lv_group_thresholds(lv_ctx* ctx, int slot, const float* q, float tau, float* out, void* stream);
int64_t lv_group_count(const lv_ctx* ctx);
int lv_group_export(const lv_ctx* ctx, int slot, int s, uint32_t* assignments, uint32_t* member_offsets,
                    uint32_t* member_ids, float* a, float* b, float* radii, double* norm_bound);

int lv_lse_merge(const float* partials, int P, int64_t rows, int d, float* out, void* stream);

/* --- Threshold oracle (threshold.hpp:9-53, threshold.cpp:40-103) --------------
 * OracleVariant (threshold.hpp:9), same order. */
#define LV_TAU_MAX 0      /* "max":      the largest sample score */
#define LV_TAU_TOPK 1     /* "topk:m":   the m-th largest */
#define LV_TAU_GAP 2      /* "gap":      cut at the largest gap between sorted scores */
#define LV_TAU_MEANMAX 3  /* "meanmax":  (max + mean) / 2, mean in double */
#define LV_TAU_BUDGET 4   /* "budget:a": nearest-rank (1 - a) quantile */

/* Reservoir (threshold.hpp:29-50): Algorithm R over a key stream, with the
 * reference's std::mt19937_64 + uniform_int_distribution draws, so a reservoir
 * with the same capacity and seed holds the same ids after the same updates.
 * It samples arena row ids (host bookkeeping; keys stay in the HBM arena). */
typedef struct lv_reservoir lv_reservoir;
int lv_reservoir_create(int64_t capacity, uint64_t seed, lv_reservoir** out); /* capacity >= 1 */
int lv_reservoir_destroy(lv_reservoir* res);
/* Reservoir::update (threshold.cpp:40-55); *slot (optional) = the position
 * written, or -1 when the id was not admitted. */
int lv_reservoir_update(lv_reservoir* res, uint32_t id, int64_t* slot);
int64_t lv_reservoir_size(const lv_reservoir* res);
int64_t lv_reservoir_seen(const lv_reservoir* res);
int64_t lv_reservoir_capacity(const lv_reservoir* res);
/* Copies the size() sampled ids, in reservoir order, to host ids[]. */
int lv_reservoir_ids(const lv_reservoir* res, uint32_t* ids);

/* estimate_tau (threshold.cpp:63-103) for every q head on the device: the
 * reservoir of kv slot s is ids[s * ld .. s * ld + count) (arena rows < lv_n),
 * q is [batch][H_q][d] fp32, tau[batch][H_q] receives the estimates; ids, q
 * and tau are host or device per `where`. Scores use the normative dot on the
 * arena rows (bf16 arenas: the stored bf16 keys). Errors as the reference's
 * std::invalid_argument: LV_EINVAL for an invalid OracleConfig (topk m < 1,
 * budget alpha outside (0, 1)), an empty reservoir, topk count < m, gap
 * count < 2; count > 8192 is LV_EINVAL too (one CTA sorts the sample). */
int lv_estimate_tau(lv_ctx* ctx, const uint32_t* ids, int64_t count, int64_t ld, const float* q,
                    int variant, int m, double alpha, int where, float* tau, void* stream);

/* Decode-loop verification (bench.cpp:83-86): adds to *violations (DEVICE
 * int32) the number of rows whose two DEVICE bitmaps [rows][words] differ,
 * e.g. lv_query's sel_bits against lv_brute_force_range's. Enqueue-only. */
int lv_bits_diff(const uint32_t* a, const uint32_t* b, int64_t words, int64_t rows, int32_t* violations,
                 void* stream);

/* Decode-loop plumbing for CUDA-graph replay of run_decode_sim (bench.cpp:54-136):
 * a DEVICE int64 step counter t selects each step's slice, so one captured decode
 * step (inputs in, estimate_tau, lv_query, lv_push_key, statistics out) replays the
 * whole loop with no host work. All pointers DEVICE; enqueue-only; capturable.
 * bytes and strides are multiples of 4.
 *   lv_step_load:      dst[0, bytes) <- src[t * stride, t * stride + bytes)
 *   lv_step_store:     dst[t * stride, + bytes) <- src[0, bytes)
 *   lv_step_reservoir: s = slot_of_step[t]; if s >= 0: ids[j * ld + s] = row0 + t for each of
 *                      the nslots reservoir copies — the write of Reservoir::update
 *                      (threshold.cpp:40-55), drawn on the host in advance
 *   lv_step_advance:   t += 1 */
/* Several step-indexed copies in one launch (up to 8): dir 0 = load, 1 = store. */
typedef struct lv_step_copy {
    const void* src;
    void* dst;
    int64_t stride;
    int64_t bytes;
    int dir;
} lv_step_copy;
int lv_step_copies(const int64_t* step, const lv_step_copy* copies, int ncopies, void* stream);
int lv_step_load(const int64_t* step, const void* src, int64_t stride, void* dst, int64_t bytes, void* stream);
int lv_step_store(const int64_t* step, const void* src, void* dst, int64_t stride, int64_t bytes, void* stream);
int lv_step_reservoir(const int64_t* step, const int32_t* slot_of_step, int64_t row0, uint32_t* ids, int nslots,
                      int64_t ld, void* stream);
int lv_step_advance(int64_t* step, void* stream);
/* The end of a decode step in one launch: the copies (as lv_step_copies), the reservoir
 * write (as lv_step_reservoir; ids may be NULL), then the step counter's advance. */
int lv_step_epilogue(int64_t* step, const lv_step_copy* copies, int ncopies, const int32_t* slot_of_step,
                     int64_t row0, uint32_t* ids, int nslots, int64_t ld, void* stream);

/* --- Snapshots (io.hpp:40-51, io.cpp:205-317) --------------------------------
 * "LVKD" dataset: magic, version 1, n, d (u32 LE), n*d f32 row-major. With
 * out == NULL, lv_load_dataset only reports n and d. Errors as the reference's
 * std::runtime_error (LV_ERUNTIME): bad magic, truncation, trailing bytes. */
int lv_save_dataset(const char* path, const float* data, int64_t n, int d);
int lv_load_dataset(const char* path, float* out, int64_t cap_rows, int64_t* n, int* d);
/* "LVIX" index snapshot of slot `slot` (io.cpp:236-268). With the grouped index
 * (lv_config.group_index) it is that index, byte for byte the reference's save_index
 * of the same BuildConfig and keys; without it, the device cells written in the
 * reference's format (S = 1, contiguous groups of r keys, exact fp32 AABBs of the
 * stored keys, indexed_count = lv_indexed_count). */
int lv_save_index(const lv_ctx* ctx, int slot, const char* path);
/* Reads any reference LVIX file (every grouping / enclosure / S), checks it
 * against the cache (dimension, indexed_count <= n, groups partitioning the
 * indexed keys consistently with the assignments, no trailing bytes) and adopts
 * its indexed_count: keys past it become the buffer. With the grouped index (one
 * slot, the snapshot's BuildConfig equal to the cache's) the snapshot's groups,
 * enclosures and members become the grouped index, gate arrays and norm bounds
 * derived as load_index does (io.cpp:309); otherwise the grouped index is rebuilt over
 * [0, indexed_count) with the cache's BuildConfig. */
int lv_load_index(lv_ctx* ctx, const char* path, int64_t* indexed_count, void* stream);

/* Host-side synthetic streams with the reference laws (io.cpp:89-206);
 * exported by liblouver_synth.so. */
int lv_synth_keys(int64_t n, int d, uint64_t seed, float* out);
int lv_synth_queries(int64_t nq, int d, uint64_t seed, float* out);
int lv_synth_mixture(int64_t n, int d, int k, double spread, uint64_t seed, int queries,
                     float* out);
int lv_synth_keys_multi(int64_t n, int d, const uint64_t* seeds, int64_t nstreams, float* out,
                        int threads);

#ifdef __cplusplus
}
#endif
#endif
