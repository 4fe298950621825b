// louver_b200_nccl.hpp — sequence-sharded decode layer over NCCL, the C++
// host side of the multi-GPU path (one process per GPU, one communicator per node).
//
// Membership q.k >= tau is independent per key, so a contiguous partition of the context
// gives per-shard selected sets whose union is the global set. Each rank queries its shard
// into per-q-head partials (m, l, o[d]) with o unnormalised (lv_query's `partial`), one
// ncclAllGather moves [world][rows][d+2] fp32 partials over NVLink, and lv_lse_merge (an
// sm_100a kernel) combines them: m = max m_p, l = sum l_p e^{m_p - m}, o = sum o_p e^{m_p - m} / l.
// An empty shard carries m = -inf, l = 0. Decode-step keys go to the tail shard, which owns
// the update buffer, so flush-at-B and the buffer semantics (cache.cpp:7-70) are those of
// one cache. Thresholds are global (the caller's tau per q head over the whole context).
//
// Link with -lnccl. Everything is enqueued on the caller's stream; no host synchronisation.
#pragma once

#include <nccl.h>

#include <stdexcept>
#include <string>
#include <utility>

#include "louver_b200.hpp"

namespace louver_b200 {

// (first, count) of rank's contiguous slice of [0, n_total); sizes differ by at most 1.
inline std::pair<std::int64_t, std::int64_t> shard_range(std::int64_t n_total, int world, int rank) {
    if (world < 1 || rank < 0 || rank >= world) throw std::invalid_argument("shard_range: 0 <= rank < world required");
    if (n_total < 0) throw std::invalid_argument("shard_range: n_total >= 0 required");
    const std::int64_t base = n_total / world, extra = n_total % world;
    return {rank * base + std::min<std::int64_t>(rank, extra), base + (rank < extra ? 1 : 0)};
}

// The rank that appends decode-step keys: the tail shard, holder of the update buffer.
inline int insert_owner(int world) { return world - 1; }

namespace detail {
inline void nccl_check(ncclResult_t r, const char* what) {
    if (r != ncclSuccess) throw std::runtime_error(std::string(what) + ": " + ncclGetErrorString(r));
}
}  // namespace detail

class ShardedLayer {
  public:
    // `shard` is this rank's LouverLayer over keys shard_range(n_total, world, rank).
    ShardedLayer(LouverLayer& shard, ncclComm_t comm)
        : layer_(shard), comm_(comm), w_(static_cast<std::size_t>(shard.rows()) * (shard.dim() + 2)) {
        detail::nccl_check(ncclCommCount(comm, &world_), "ncclCommCount");
        detail::nccl_check(ncclCommUserRank(comm, &rank_), "ncclCommUserRank");
        detail::cuda_check(cudaMalloc(&partial_, sizeof(float) * w_ * (1 + world_)), "cudaMalloc");
        gathered_ = partial_ + w_;
    }
    ~ShardedLayer() { cudaFree(partial_); }
    ShardedLayer(const ShardedLayer&) = delete;
    ShardedLayer& operator=(const ShardedLayer&) = delete;

    int rank() const { return rank_; }
    int world() const { return world_; }

    // One decode step's key/value per slot (k, v [batch][H_kv][d]): the tail shard appends.
    void push_key(const void* k, const void* v, int src_dtype, int where, cudaStream_t st = nullptr) {
        if (rank_ == insert_owner(world_)) layer_.push_key(k, v, src_dtype, where, st);
    }

    // q [batch][H_q][d], tau [batch][H_q], out [batch][H_q][d]: device pointers, enqueue-only.
    void query(const float* q, const float* tau, float* out, cudaStream_t st, bool strict = false, float scale = 0.0f) {
        layer_.query_device(q, tau, nullptr, st, partial_, nullptr, strict, scale);
        detail::nccl_check(ncclAllGather(partial_, gathered_, w_, ncclFloat, comm_, st), "ncclAllGather");
        lse_merge(gathered_, world_, layer_.rows(), layer_.dim(), out, st);
    }

  private:
    LouverLayer& layer_;
    ncclComm_t comm_;
    int world_ = 1, rank_ = 0;
    std::size_t w_;             // floats per rank's partials: rows x (d + 2)
    float* partial_ = nullptr;  // [rows][d+2]
    float* gathered_ = nullptr; // [world][rows][d+2]
};

}  // namespace louver_b200
