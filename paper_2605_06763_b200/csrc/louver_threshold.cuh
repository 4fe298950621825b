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

__device__ __forceinline__ float to_f(float x) { return x; }
__device__ __forceinline__ float to_f(__nv_bfloat16 x) { return __bfloat162float(x); }

template <typename T>
__global__ void estimate_tau_kernel(const T* __restrict__ K, long long cap, int DP, int d, int G,
                                    const uint32_t* __restrict__ ids, long long ld, int cnt,
                                    const float* __restrict__ q, int mode, int pick, int np2,
                                    float* __restrict__ tau) {
    extern __shared__ float sh[];
    float* qs = sh;         // [d]
    float* sc = sh + DP;    // [np2]
    const int row = blockIdx.x, slot = row / G;
    for (int c = threadIdx.x; c < d; c += blockDim.x) qs[c] = q[(size_t)row * DP + c];
    __syncthreads();
    const uint32_t* rid = ids + (size_t)slot * ld;
    for (int i = threadIdx.x; i < np2; i += blockDim.x) {
        float s = -INFINITY;  // padding sorts behind every finite score
        if (i < cnt) {
            const T* k = K + ((size_t)slot * cap + rid[i]) * DP;
            s = 0.0f;
#pragma unroll 8
            for (int c = 0; c < d; ++c) s = __fadd_rn(s, __fmul_rn(qs[c], to_f(k[c])));
        }
        sc[i] = s;
    }
    __syncthreads();
    // bitonic sort, descending overall
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

}  // namespace lvkt
