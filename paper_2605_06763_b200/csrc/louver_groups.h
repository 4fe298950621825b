// Grouped index on the device: the reference's LouverIndex (S subspaces, each a set of
// groups from the configured GroupingStrategy, each group an Enclosure, packed gate
// arrays, member lists) built from the keys in the HBM arena, and the two candidate
// filters over it (query_full_subspace, query_ta) plus derive_subspace_thresholds.
//
// The fused query kernel never needs it: its contiguous-cell AABB summaries select the
// same final sets. This index reproduces the reference's own grouping, enclosures,
// candidate sets and statistics (keys_scanned, f_scan, gate_cost_equiv, TA stop depth)
// for a BuildConfig, and serialises as the reference's LVIX snapshot.
//
//   balanced_pca_tree / pca_split   index.cpp:15-68    level-synchronous median splits
//   assign_groups                   index.cpp:70-102
//   enclose_group                   index.cpp:104-137
//   append_gate_entry               index.cpp:139-168
//   index_range / append_to_index   index.cpp:172-232
//   gate_bounds                     query.cpp:47-68
//   query_full_subspace             query.cpp:82-117
//   query_ta                        query.cpp:204-303
//   derive_subspace_thresholds      query.cpp:305-336
#pragma once

#include <cstdint>
#include <vector>

#include <cuda_runtime.h>

namespace lvg {

struct ArenaView {            // the cache's key arena
    const void* K = nullptr;  // [slots][cap][DP], fp32 or bf16
    bool bf16 = false;
    int DP = 0;
    long long cap = 0;
};

struct GroupIndex {
    int S = 1, d = 0, r = 1, grouping = 0, enclosure = 0, slots = 0;
    unsigned long long seed = 0;
    std::vector<int> off;     // SubspaceLayout offsets [S + 1]
    int wmax = 0;
    long long cap = 0;        // keys per slot (arena rows)
    long long kcap = 0;       // groups per (slot, subspace)
    long long indexed = 0;    // keys indexed (host mirror; the same for every slot)
    long long K = 0;          // groups per (slot, subspace): the grouping's shape depends only
                              // on the block sizes, so it is the same everywhere
    // device arrays, pair p = slot * S + s
    unsigned* assign = nullptr;        // [P][cap]
    unsigned* moff = nullptr;          // [P][kcap + 1]
    unsigned* mids = nullptr;          // [P][cap]
    float* ga = nullptr;               // [P][wmax][kcap] centers (ball kinds) or lo (AABB)
    float* gb = nullptr;               // [P][wmax][kcap] hi (AABB)
    float* grad = nullptr;             // [P][kcap] radii (ball kinds)
    unsigned long long* nbound = nullptr;  // [P] norm_bound as the bits of a double >= 0
};

struct Stats {
    long long groups_tested = 0, keys_scanned = 0;
    double f_scan = 0.0, gate_cost_equiv = 0.0;
    int ta_stop_depth = -1;
    double ta_stop_upper = 0.0;
};

// allocation; layout/config validated by the caller
cudaError_t create(GroupIndex& gi, int d, int S, int r, int grouping, int enclosure, unsigned long long seed,
                   int slots, long long cap);
void destroy(GroupIndex& gi);
// capacity growth: arrays move to the new row capacity, contents kept
cudaError_t reserve(GroupIndex& gi, long long cap, cudaStream_t st);
// index_range (index.cpp:195-209) over keys [first, first + count) of every slot;
// first must equal gi.indexed (append_to_index's precondition)
cudaError_t index_range(GroupIndex& gi, const ArenaView& a, long long first, long long count, cudaStream_t st);
// candidate set of query_full_subspace (algo 0, tau_s[S] host, required) or query_ta
// (algo 1) for one slot and one query q[d] (host); live ids as a DEVICE bitmap over
// [0, indexed) (words = ceil(indexed / 32)) and the statistics (host). Synchronises.
cudaError_t candidates(const GroupIndex& gi, int slot, const float* q, float tau, const float* tau_s, int algo,
                       unsigned* live_bits, Stats* stats, cudaStream_t st);
// derive_subspace_thresholds for one slot (host q, host out[S]). Synchronises.
cudaError_t thresholds(const GroupIndex& gi, int slot, const float* q, float tau, float* out, cudaStream_t st);
// host copies of one (slot, subspace): assignments [indexed], member offsets [K + 1],
// member ids [indexed], gate arrays [w][K] (a: centers or lo, b: hi), radii [K], norm_bound
cudaError_t export_subspace(const GroupIndex& gi, int slot, int s, unsigned* assign, unsigned* moff,
                            unsigned* mids, float* a, float* b, float* radii, double* norm_bound);
// the inverse (LVIX snapshot load): groups of one (slot, subspace) given on the host,
// gate arrays and norm bounds derived as append_gate_entry does (index.cpp:139-168)
cudaError_t import_subspace(GroupIndex& gi, int slot, int s, long long indexed, long long K, const unsigned* assign,
                            const unsigned* moff, const unsigned* mids, const float* a, const float* b,
                            const float* radii, double norm_bound);

}  // namespace lvg
