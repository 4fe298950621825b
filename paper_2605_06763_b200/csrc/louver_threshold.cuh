// Threshold oracle on the device: estimate_tau of
// proj/src/threshold.cpp:63-103 over a reservoir sample of arena rows.
//
// The reference keeps copies of the sampled keys (threshold.hpp:29-50); here the
// reservoir holds arena row ids (rows are append-only, so key(id) never changes)
// and the kernel gathers the rows. One CTA per q head:
//   1. scores s_i = dot(q, k_{id_i}) with the normative operation order of
//      core.hpp:17-21 (fp32 multiply, then add, sequential over the coordinates);
//   2. a bitonic sort of the scores, descending (threshold.cpp:71), padded with -inf;
//   3. the variant's pick (threshold.cpp:73-101). Ranks that depend only on the
//      sample size (max, topk:m, budget:alpha) arrive precomputed from the host,
//      with the reference's own index formula, so they are bit-identical.
// Bound: latency (a few KB per q head); the d-long dependent add chain per score
// sets the time, as in the reference.
#pragma once
#include <cuda_bf16.h>
#include <cuda_runtime.h>
#include <stdint.h>

namespace lvkt {

enum : int { kPick = 0, kGap = 1, kMeanMax = 2 };

// rows staged per round: 64 KB of keys (plus one 16-byte pad per row: the dot
// loop reads one row per thread, 16 bytes at a time, without bank conflicts)
constexpr int kStageBytes = 65536;

template <typename T>
__host__ __device__ constexpr int stage_rows(int DP) {
    return kStageBytes / (DP * (int)sizeof(T)) > 0 ? kStageBytes / (DP * (int)sizeof(T)) : 1;
}

__device__ __forceinline__ void unpack8(const uint4& u, float* f, float) {
    f[0] = __uint_as_float(u.x);
    f[1] = __uint_as_float(u.y);
    f[2] = __uint_as_float(u.z);
    f[3] = __uint_as_float(u.w);
}
__device__ __forceinline__ void unpack8(const uint4& u, float* f, __nv_bfloat16) {
    const unsigned w[4] = {u.x, u.y, u.z, u.w};
#pragma unroll
    for (int i = 0; i < 4; ++i) {
        f[2 * i] = __uint_as_float(w[i] << 16);
        f[2 * i + 1] = __uint_as_float(w[i] & 0xffff0000u);
    }
}

template <typename T>
__global__ void estimate_tau_kernel(const T* __restrict__ K, long long cap, int DP, int d, int G,
                                    const uint32_t* __restrict__ ids, long long ld, int cnt,
                                    const float* __restrict__ q, int mode, int pick, int np2,
                                    float* __restrict__ tau) {
    // The kernel after this one (the layer query, launched with programmatic stream
    // serialisation) may be dispatched onto the SMs this small grid leaves idle and start its
    // pre-wait prologue now; it reads tau only after its griddepcontrol.wait.
    asm volatile("griddepcontrol.launch_dependents;\n" ::: "memory");
    extern __shared__ __align__(16) float sh[];
    constexpr int EPV = 16 / sizeof(T);  // elements per 16-byte vector
    const int vpr = DP / EPV, rstride = vpr + 1;  // vectors per row, staged row stride (padded)
    const int rpc = stage_rows<T>(DP);
    uint4* stg = reinterpret_cast<uint4*>(sh);  // [rpc][rstride]
    float* qs = sh + (size_t)rpc * rstride * 4;  // [DP], zero past d
    float* sc = qs + DP;                         // [np2]
    uint32_t* sid = reinterpret_cast<uint32_t*>(sc + np2);  // [cnt] sampled row ids
    const int row = blockIdx.x, slot = row / G;
    for (int c = threadIdx.x; c < DP; c += blockDim.x) qs[c] = c < d ? q[(size_t)row * DP + c] : 0.0f;
    const uint32_t* rid = ids + (size_t)slot * ld;
    for (int i = threadIdx.x; i < cnt; i += blockDim.x) sid[i] = __ldg(rid + i);
    const uint4* Kv = reinterpret_cast<const uint4*>(K + (size_t)slot * cap * DP);
    for (int i = cnt + threadIdx.x; i < np2; i += blockDim.x) sc[i] = -INFINITY;  // sorts behind every score
    const unsigned stg_s = (unsigned)__cvta_generic_to_shared(stg);
    for (int base = 0; base < cnt; base += rpc) {
        const int nr = cnt - base < rpc ? cnt - base : rpc;
        __syncthreads();  // previous round's rows consumed (ids and qs written)
        // every row of the round in flight at once (asynchronous copies, one wait)
        for (int i = threadIdx.x; i < nr * vpr; i += blockDim.x) {
            const int r = i / vpr, c = i - r * vpr;
            asm volatile("cp.async.cg.shared.global [%0], [%1], 16;\n" ::"r"(stg_s + (unsigned)(r * rstride + c) * 16u),
                         "l"(Kv + (size_t)sid[base + r] * vpr + c)
                         : "memory");
        }
        asm volatile("cp.async.commit_group;\ncp.async.wait_group 0;\n" ::: "memory");
        __syncthreads();
        for (int r = threadIdx.x; r < nr; r += blockDim.x) {
            // normative order (core.hpp:17-21): fp32 multiply, then add, coordinate by coordinate
            float s = 0.0f;
            const int nv = (d + EPV - 1) / EPV;
            for (int v = 0; v < nv; ++v) {
                float kf[8];
                unpack8(stg[r * rstride + v], kf, T());
#pragma unroll
                for (int e = 0; e < EPV; ++e)
                    if (v * EPV + e < d) s = __fadd_rn(s, __fmul_rn(qs[v * EPV + e], kf[e]));
            }
            sc[base + r] = s;
        }
    }
    __syncthreads();
    // bitonic sort, descending overall
    if (np2 == (int)blockDim.x) {
        // one score per thread: partners closer than a warp swap through shuffles, only
        // the log2(np2) - 5 widest distances of each merge go through shared memory.
        // On equal scores each side keeps its own value, so the multiset is preserved.
        const int i = threadIdx.x;
        float v = sc[i];
        for (int k = 2; k <= np2; k <<= 1) {
            for (int j = k >> 1; j > 0; j >>= 1) {
                float o;
                if (j >= 32) {
                    __syncthreads();
                    sc[i] = v;
                    __syncthreads();
                    o = sc[i ^ j];
                } else {
                    o = __shfl_xor_sync(0xffffffffu, v, j);
                }
                const bool take_max = ((i & j) == 0) == ((i & k) == 0);
                v = take_max ? (o > v ? o : v) : (o < v ? o : v);
            }
        }
        __syncthreads();
        sc[i] = v;
        __syncthreads();
    } else {
        for (int k = 2; k <= np2; k <<= 1) {
            for (int j = k >> 1; j > 0; j >>= 1) {
                for (int i = threadIdx.x; i < np2; i += blockDim.x) {
                    const int p = i ^ j;
                    if (p > i) {
                        const float a = sc[i], b = sc[p];
                        const bool desc = (i & k) == 0;
                        if (desc ? a < b : a > b) {
                            sc[i] = b;
                            sc[p] = a;
                        }
                    }
                }
                __syncthreads();
            }
        }
    }
    if (threadIdx.x != 0) return;
    float r;
    if (mode == kPick) {
        r = sc[pick];
    } else if (mode == kGap) {  // threshold.cpp:78-91: first largest gap wins ties
        int best = 0;
        float best_gap = __fsub_rn(sc[0], sc[1]);
        for (int i = 1; i + 1 < cnt; ++i) {
            const float g = __fsub_rn(sc[i], sc[i + 1]);
            if (g > best_gap) {
                best_gap = g;
                best = i;
            }
        }
        r = sc[best];
    } else {  // threshold.cpp:92-97: mean in double over the sorted scores, in order
        double mean = 0.0;
        for (int i = 0; i < cnt; ++i) mean = __dadd_rn(mean, (double)sc[i]);
        mean = __ddiv_rn(mean, (double)cnt);
        r = (float)__ddiv_rn(__dadd_rn((double)sc[0], mean), 2.0);
    }
    tau[row] = r;
}

// decode-loop verification (bench.cpp:83-86 on the device): one block per row adds
// one violation when the row's two id bitmaps differ anywhere
__global__ void bits_diff_kernel(const uint32_t* __restrict__ a, const uint32_t* __restrict__ b, long long words,
                                 int* __restrict__ violations) {
    const long long base = (long long)blockIdx.x * words;
    int diff = 0;
    for (long long i = threadIdx.x; i < words; i += blockDim.x) diff |= a[base + i] != b[base + i];
    diff = __syncthreads_or(diff);
    if (diff && threadIdx.x == 0) atomicAdd(violations, 1);
}

// ---- decode-loop plumbing for CUDA-graph replay (bench.cpp:71-120): a device step counter
// selects each step's inputs, so one captured step replays the whole loop with no host work

// dir 0: dst[0, words) <- src[t * stride ..];  dir 1: dst[t * stride ..] <- src[0, words)
__global__ void step_copy_kernel(const long long* __restrict__ step, const uint32_t* __restrict__ src,
                                 uint32_t* __restrict__ dst, long long stride_words, long long words, int dir) {
    const long long off = *step * stride_words;
    const uint32_t* s = dir == 0 ? src + off : src;
    uint32_t* d = dir == 0 ? dst : dst + off;
    for (long long i = (long long)blockIdx.x * blockDim.x + threadIdx.x; i < words; i += (long long)gridDim.x * blockDim.x)
        d[i] = s[i];
}

struct StepCopy {
    const uint32_t* src;
    uint32_t* dst;
    long long stride_words;
    long long words;
    int dir;  // 0: dst <- src[t * stride]; 1: dst[t * stride] <- src
};
struct StepCopies {
    StepCopy c[8];
    int n;
};

// every copy of a step in one launch (blockIdx.y = copy)
__global__ void step_copies_kernel(const long long* __restrict__ step, const __grid_constant__ StepCopies cs) {
    if ((int)blockIdx.y >= cs.n) return;
    const StepCopy& c = cs.c[blockIdx.y];
    const long long off = *step * c.stride_words;
    const uint32_t* s = c.dir == 0 ? c.src + off : c.src;
    uint32_t* d = c.dir == 0 ? c.dst : c.dst + off;
    for (long long i = (long long)blockIdx.x * blockDim.x + threadIdx.x; i < c.words; i += (long long)gridDim.x * blockDim.x)
        d[i] = s[i];
}

// Reservoir::update's write (threshold.cpp:40-55), drawn on the host in advance: the step's
// admitted slot (or -1) receives the step's arena row
__global__ void step_reservoir_kernel(const long long* __restrict__ step, const int* __restrict__ slot_of_step,
                                      long long row0, uint32_t* __restrict__ ids, int nslots, long long ld) {
    const long long t = *step;
    const int slot = slot_of_step[t];
    if (slot >= 0 && (int)threadIdx.x < nslots) ids[threadIdx.x * ld + slot] = (uint32_t)(row0 + t);
}

__global__ void step_advance_kernel(long long* step) { *step += 1; }

// The end of a decode step in one launch (one block): the step's log stores, the
// reservoir's write for the step's row, then the counter advance (after every read of it)
__global__ void step_epilogue_kernel(long long* step, const __grid_constant__ StepCopies cs,
                                     const int* __restrict__ slot_of_step, long long row0, uint32_t* __restrict__ ids,
                                     int nslots, long long ld) {
    const long long t = *step;
    for (int k = 0; k < cs.n; ++k) {
        const StepCopy& c = cs.c[k];
        const long long off = t * c.stride_words;
        const uint32_t* s = c.dir == 0 ? c.src + off : c.src;
        uint32_t* d = c.dir == 0 ? c.dst : c.dst + off;
        for (long long i = threadIdx.x; i < c.words; i += blockDim.x) d[i] = s[i];
    }
    if (ids) {
        const int slot = slot_of_step[t];
        for (int i = threadIdx.x; slot >= 0 && i < nslots; i += blockDim.x) ids[i * ld + slot] = (uint32_t)(row0 + t);
    }
    __syncthreads();
    if (threadIdx.x == 0) *step = t + 1;
}

}  // namespace lvkt
