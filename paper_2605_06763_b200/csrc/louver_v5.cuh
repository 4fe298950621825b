// Louver bf16 query path, flat warp-level form (sm_100a).
//
// Every warp works independently on 16-row tiles, with tensor-core A
// fragments loaded straight from HBM into registers: within each 32-element
// k-pair, lane q = lane%4 of row i loads the 16 bytes [32p+8q, 32p+8q+8) of
// that row, and the k order of both operands is permuted accordingly (logical
// k-step 2p+h, element j -> physical 32p + 8(j/2 % 4)... see a_frags()), so one
// LDG.128 per lane per row per 32 dims feeds two mma k-steps with fully used
// 32-byte sectors. No shared-memory staging, no CTA barriers in the hot loops:
// the SM overlaps the load -> mma -> gather chains of ~16 warps.
//
// K1 louver_probe_v5  grid (nbp, slots): warps stride over 16-cell tiles of the
//     cell-major summaries (row per cell = [hi | lo], 2*DP bf16). bound_g =
//     [hi|lo].[q+|q-] with q split into 2 bf16 parts; a cell survives when any
//     q head's bound reaches tau - 2^-12 S_g (or it holds buffer keys).
//     Output: one 16-bit survivor mask per tile, cmask[slot][tile].
// K2 louver_exact_v5  grid (nb, slots): the slot's surviving rows (prefix over
//     popc(cmask) * r) are split evenly over its CTAs and, inside, round-robin
//     over warps in 16-row tasks. Fast scores with q split into 3 bf16 parts;
//     pairs within 2^-13 S_g of tau get the normative sequential fp32 dot
//     (core.hpp:17-21) so membership is bit-exact. Attended pairs (selected ∪
//     buffer, cache.cpp:48-68) gather their V rows (8 bytes per lane) into a
//     per-warp online softmax; warps, then CTAs (two-level ticket tree), merge.
#pragma once

#include <cstdio>

#include "louver_v2.cuh"

namespace lvk5 {

using lvk::Counters;
using lvk::QueryParams;
using lvk2::bf_bits;
using lvk2::bf_val;
using lvk2::mma16816;

constexpr int kT = 256;
constexpr int kW = kT / 32;
constexpr int kMG = 16;  // K2 partials per merge group

struct V5Params {
    QueryParams p;
    const __nv_bfloat16* sum;  // [slot][cap_cells][2*DP] cell rows [hi | lo]
    unsigned short* cmask;     // [slot][tiles] survivor bit per cell of each 16-cell tile
    int tiles;                 // 16-cell tiles per slot (cap_cells / 16)
    int nbp;                   // K1 CTAs per slot
    int nb;                    // K2 CTAs per slot
    float* gpart;              // [slots][ngroups][G][DP+2]
    int* gtickets;             // [slots][ngroups]
    int* stickets;             // [slots]
    int ngroups;
    int* gmax;                 // optional [slot][G]: reset to the encoding of -inf by K1
    int slots;                 // v9: slots of the layer (the grid may loop over them)
    unsigned short* glist;     // v9: survivor lists in global scratch when they outgrow smem (else null)
    int list_cap;              // v9: entries per CTA list
    long long sealed;          // v9: cells complete when the query was enqueued (immutable summaries)
    int dbg;                   // v9: timing experiments only (LV_DBG; output invalid): 1 no merge,
                               //     2 no CTA partial and no merge, 4 ticket without the merge body
};

// physical element of logical (k-step t, fragment element e in 0..3) for lane q:
// e = 0,1 -> b0/a0 pair, e = 2,3 -> b1/a2 pair.
__device__ __forceinline__ int perm_dim(int t, int q, int e) { return 32 * (t >> 1) + 8 * q + 4 * (t & 1) + e; }

// B fragment of a k-way split matrix whose column n is part (n / G) of q_g,
// g = n % G; `val(k, g)` gives the fp32 value at physical k.
template <int G, int PARTS, typename Val>
__device__ __forceinline__ uint2 b_frag(int t, int nt, int lane, Val val) {
    const int col = nt * 8 + lane / 4, q = lane & 3;
    unsigned short v[4] = {0, 0, 0, 0};
    if (col < PARTS * G) {
        const int part = col / G, g = col % G;
#pragma unroll
        for (int e = 0; e < 4; ++e) {
            float x = val(perm_dim(t, q, e), g);
            unsigned short b = bf_bits(x);
            for (int k = 0; k < part; ++k) {
                x = x - bf_val(b);
                b = bf_bits(x);
            }
            v[e] = b;
        }
    }
    return make_uint2((unsigned)v[0] | ((unsigned)v[1] << 16), (unsigned)v[2] | ((unsigned)v[3] << 16));
}

__device__ __forceinline__ uint4 ldg16(const void* p) {
    uint4 r;
    asm volatile("ld.global.nc.L1::no_allocate.v4.u32 {%0,%1,%2,%3}, [%4];\n"
                 : "=r"(r.x), "=r"(r.y), "=r"(r.z), "=r"(r.w)
                 : "l"(p));
    return r;
}
__device__ __forceinline__ uint2 ldg8(const void* p) {
    uint2 r;
    asm volatile("ld.global.nc.L1::no_allocate.v2.u32 {%0,%1}, [%2];\n" : "=r"(r.x), "=r"(r.y) : "l"(p));
    return r;
}

// VPL consecutive bf16 of a V row (VPL = DP/32 in {2,4,8}) -> uint4 container
template <int VPL>
__device__ __forceinline__ uint4 ldg_v(const unsigned char* p) {
    if constexpr (VPL == 8) {
        return ldg16(p);
    } else if constexpr (VPL == 4) {
        const uint2 a = ldg8(p);
        return make_uint4(a.x, a.y, 0u, 0u);
    } else {
        unsigned a;
        asm volatile("ld.global.nc.L1::no_allocate.u32 %0, [%1];\n" : "=r"(a) : "l"(p));
        return make_uint4(a, 0u, 0u, 0u);
    }
}

// S_g = sum_c |q_gc| colmax_c rounded up; q rows copied to qf[G][DP+4].
template <int DP, int G>
__device__ __forceinline__ void setup_q(const float* qsrc, const float* colmax, float* qf, float* red, float* S) {
    const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
    float s[G];
#pragma unroll
    for (int g = 0; g < G; ++g) s[g] = 0.0f;
    for (int i = tid; i < G * DP; i += kT) {
        const int g = i / DP, c = i % DP;
        const float x = qsrc[i];
        qf[g * (DP + 4) + c] = x;
        const float t = __fmul_ru(fabsf(x), colmax[c]);
#pragma unroll
        for (int h = 0; h < G; ++h)
            if (h == g) s[h] = __fadd_ru(s[h], t);
    }
#pragma unroll
    for (int g = 0; g < G; ++g) {
        float v = s[g];
#pragma unroll
        for (int o = 16; o > 0; o >>= 1) v = __fadd_ru(v, __shfl_xor_sync(0xffffffffu, v, o));
        if (lane == 0) red[warp * G + g] = v;
    }
    __syncthreads();
    if (tid < G) {
        float v = 0.0f;
        for (int w = 0; w < kW; ++w) v = __fadd_ru(v, red[w * G + tid]);
        S[tid] = v;
    }
    __syncthreads();
}

// ----------------------------------------------------------------------- K1

template <int DP, int G>
struct P5 {
    static constexpr int NT = (2 * G + 7) / 8;
    static constexpr int KS = 2 * DP / 16;  // k-steps over [hi | lo]
    static constexpr int OFF_FR = 0;                              // [KS][NT][32] uint2
    static constexpr int OFF_CT = OFF_FR + KS * NT * 32 * 8;      // [kW][16][8*NT] f32
    static constexpr int OFF_Q = OFF_CT + kW * 16 * 8 * NT * 4;   // [G][DP+4]
    static constexpr int OFF_M = OFF_Q + G * (DP + 4) * 4;        // tau_pr[G], S[G], red[kW*G]
    static constexpr int SMEM = OFF_M + (2 * G + kW * G) * 4;
};

template <int DP, int G>
__global__ void __launch_bounds__(kT, 2) louver_probe_v5(const __grid_constant__ V5Params vp) {
    using Ge = P5<DP, G>;
    const QueryParams& p = vp.p;
    extern __shared__ __align__(16) unsigned char smem[];
    uint2* fr = reinterpret_cast<uint2*>(smem + Ge::OFF_FR);
    float* qf = reinterpret_cast<float*>(smem + Ge::OFF_Q);
    float* tau_pr = reinterpret_cast<float*>(smem + Ge::OFF_M);
    float* S = tau_pr + G;
    float* red = S + G;
    const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
    const int slot = blockIdx.y;
    float* ct = reinterpret_cast<float*>(smem + Ge::OFF_CT) + warp * 16 * 8 * Ge::NT;

    // The first tile's loads depend on nothing: issue them before the setup.
    // Rows are addressed within the arena capacity; rows past n are ignored.
    const __nv_bfloat16* base = vp.sum + (size_t)slot * p.cap_cells * (2 * DP);
    const int q = lane & 3;
    constexpr int NP = 2 * DP / 32;  // k-pairs
    uint4 u0[NP], u1[NP];
    const int stride = vp.nbp * kW;
    auto load_tile = [&](int tile) {
        const long long c0 = (long long)tile << 4;
        const unsigned char* row0 =
            reinterpret_cast<const unsigned char*>(base + (size_t)(c0 + (lane >> 2)) * 2 * DP);
        const unsigned char* row1 = row0 + 8 * 2 * DP * 2;
#pragma unroll
        for (int pp = 0; pp < NP; ++pp) {
            u0[pp] = ldg16(row0 + (32 * pp + 8 * q) * 2);
            u1[pp] = ldg16(row1 + (32 * pp + 8 * q) * 2);
        }
    };
    int tile = blockIdx.x * kW + warp;
    if (tile < vp.tiles) load_tile(tile);

    const long long n = p.ctr->n;
    const long long indexed = p.ctr->indexed;
    const int rl = p.r_log2, r = 1 << rl;
    const long long ncells = (n + r - 1) >> rl;
    const int ntile = (int)((ncells + 15) >> 4);
    setup_q<DP, G>(p.q + (size_t)slot * G * DP, p.colmax + (size_t)slot * DP, qf, red, S);
    if (tid < G) tau_pr[tid] = __fsub_rd(p.tau[(size_t)slot * G + tid], __fmul_ru(S[tid], 2.44140625e-4f));
    for (int i = tid; i < Ge::KS * Ge::NT * 32; i += kT) {
        const int l = i & 31, nt = (i >> 5) % Ge::NT, t = (i >> 5) / Ge::NT;
        fr[i] = b_frag<G, 2>(t, nt, l, [&](int k, int g) {
            const float x = qf[g * (DP + 4) + (k % DP)];
            return k < DP ? fmaxf(x, 0.0f) : fminf(x, 0.0f);  // [hi | lo] . [q+ | q-]
        });
    }
    __syncthreads();
    // the exact kernel may start its own setup now (programmatic dependent launch)
    if (vp.gmax && blockIdx.x == 0 && tid < G) {
        const int ninf = __float_as_int(-INFINITY) ^ 0x7fffffff;  // order-preserving int of -inf
        vp.gmax[(size_t)slot * G + tid] = ninf;
    }
    asm volatile("griddepcontrol.launch_dependents;\n" ::: "memory");

    for (; tile < ntile; tile += stride) {
        const long long c0 = (long long)tile << 4;
        float acc[Ge::NT][4];
#pragma unroll
        for (int t = 0; t < Ge::NT; ++t) acc[t][0] = acc[t][1] = acc[t][2] = acc[t][3] = 0.0f;
#pragma unroll
        for (int pp = 0; pp < NP; ++pp) {
            const unsigned a0[4] = {u0[pp].x, u1[pp].x, u0[pp].y, u1[pp].y};
            const unsigned a1[4] = {u0[pp].z, u1[pp].z, u0[pp].w, u1[pp].w};
#pragma unroll
            for (int t = 0; t < Ge::NT; ++t) {
                const uint2 b0 = fr[((2 * pp) * Ge::NT + t) * 32 + lane];
                const uint2 b1 = fr[((2 * pp + 1) * Ge::NT + t) * 32 + lane];
                mma16816(acc[t], a0, b0.x, b0.y);
                mma16816(acc[t], a1, b1.x, b1.y);
            }
        }
        if (tile + stride < ntile) load_tile(tile + stride);  // prefetch the next tile
#pragma unroll
        for (int t = 0; t < Ge::NT; ++t) {
            const int rw = lane >> 2, col = t * 8 + 2 * q;
            ct[rw * 8 * Ge::NT + col] = acc[t][0];
            ct[rw * 8 * Ge::NT + col + 1] = acc[t][1];
            ct[(rw + 8) * 8 * Ge::NT + col] = acc[t][2];
            ct[(rw + 8) * 8 * Ge::NT + col + 1] = acc[t][3];
        }
        __syncwarp();
        unsigned gm = 0;
        int scan = 0;
        const long long cell = c0 + lane;
        if (lane < 16 && cell < ncells) {
            const long long cs = cell << rl, ce = cs + r;
            if (ce > indexed) {
                gm = (1u << G) - 1u;  // holds buffer keys: scanned densely
            } else {
#pragma unroll
                for (int g = 0; g < G; ++g) {
                    const float b = ct[lane * 8 * Ge::NT + g] + ct[lane * 8 * Ge::NT + G + g];
                    if (b >= tau_pr[g]) gm |= 1u << g;
                }
            }
            scan = (int)((ce < n ? ce : n) - cs);
        }
        __syncwarp();
        const unsigned m = __ballot_sync(0xffffffffu, gm != 0) & 0xffffu;
        if (lane == 0) vp.cmask[(size_t)slot * vp.tiles + tile] = (unsigned short)m;
        __syncwarp();
        if (p.totals) {
            const int tested = __popc(__ballot_sync(0xffffffffu, lane < 16 && cell < ncells));
            if (lane == 0) {
                atomicAdd(p.totals + 0, (unsigned long long)tested);
                atomicAdd(p.totals + 1, (unsigned long long)__popc(m));
            }
        }
        if (p.counts) {
#pragma unroll
            for (int g = 0; g < G; ++g) {
                const int v = lvk::warp_sum_int((gm >> g) & 1 ? scan : 0);
                if (lane == 0 && v) atomicAdd(p.counts + ((size_t)slot * G + g) * 4 + 2, v);
            }
        }
    }
}

// ----------------------------------------------------------------------- K2

template <int DP, int G>
struct E5 {
    static constexpr int NT = (3 * G + 7) / 8;
    static constexpr int KS = DP / 16;
    static constexpr int KL = 2048;                                   // row -> key list per segment
    static constexpr int OFF_FR = 0;                                  // [KS][NT][32] uint2
    static constexpr int OFF_Q = OFF_FR + KS * NT * 32 * 8;           // [G][DP+4]
    static constexpr int OFF_M = OFF_Q + G * (DP + 4) * 4;            // misc floats
    static constexpr int MISC = 4 * G + kW * G + 8;
    static constexpr int OFF_KL = (OFF_M + MISC * 4 + 15) / 16 * 16;  // [KL] u32 keys of the segment
    static constexpr int OFF_WS = OFF_KL + KL * 4;                    // per-warp scratch
    static constexpr int WCT = 16 * 8 * NT;                           // C tile floats
    static constexpr int WSC = 16 * G;                                // scores of the task
    static constexpr int WSZ = (WCT + WSC) * 4;
    static constexpr int SZ_WS = kW * WSZ;
    static constexpr int SZ_RED = kW * G * (DP + 2) * 4;              // final warp reduction
    static constexpr int SZ_U = SZ_WS > SZ_RED ? SZ_WS : SZ_RED;
    static constexpr int FIXED = OFF_WS + SZ_U;
    static int smem(int tiles) { return FIXED + tiles * 8; }          // cmask (u32) + prefix (u32)
};

// Merge P partials [P][G][DP+2] (stride W) into dst / out rows (kT threads).
template <int DP, int G>
__device__ void merge5(const float* src, int P, float* dst, float* out, float* part_out, int* counts,
                       float* shw) {
    // shw: [P][G] weights, then M[G], L[G]; all partial headers are loaded in
    // parallel and the o loads are batched, so a merge costs ~2 L2 round trips.
    const int tid = threadIdx.x;
    constexpr int W = G * (DP + 2);
    float* shm = shw;              // [P][G] m, then weights
    float* shl = shw + P * G;      // [P][G] l
    float* ML = shl + P * G;       // M[G], L[G]
    for (int i = tid; i < P * G; i += kT) {
        const int s = i / G, g = i % G;
        shm[i] = __ldcg(src + (size_t)s * W + g * (DP + 2));
        shl[i] = __ldcg(src + (size_t)s * W + g * (DP + 2) + 1);
    }
    __syncthreads();
    if (tid < G) {
        float m = -INFINITY;
        for (int s = 0; s < P; ++s) m = fmaxf(m, shm[s * G + tid]);
        float l = 0.0f;
        for (int s = 0; s < P; ++s) {
            const float ms = shm[s * G + tid];
            const float w = ms == -INFINITY ? 0.0f : expf(ms - m);
            shm[s * G + tid] = w;
            l += w * shl[s * G + tid];
        }
        ML[tid] = m;
        ML[G + tid] = l;
    }
    __syncthreads();
    for (int i = tid; i < G * DP; i += kT) {
        const int g = i / DP, c = i % DP;
        float acc = 0.0f;
        for (int s0 = 0; s0 < P; s0 += 8) {
            float v[8];
#pragma unroll
            for (int j = 0; j < 8; ++j)
                v[j] = s0 + j < P ? __ldcg(src + (size_t)(s0 + j) * W + g * (DP + 2) + 2 + c) : 0.0f;
#pragma unroll
            for (int j = 0; j < 8; ++j)
                if (s0 + j < P) acc = fmaf(shm[(s0 + j) * G + g], v[j], acc);
        }
        const float l = ML[G + g];
        if (dst) dst[g * (DP + 2) + 2 + c] = acc;
        if (out) out[g * DP + c] = l > 0.0f ? acc / l : 0.0f;
        if (part_out) part_out[g * (DP + 2) + 2 + c] = acc;
    }
    if (tid < G) {
        const float m = ML[tid], l = ML[G + tid];
        if (dst) {
            dst[tid * (DP + 2)] = m;
            dst[tid * (DP + 2) + 1] = l;
        }
        if (part_out) {
            part_out[tid * (DP + 2)] = m;
            part_out[tid * (DP + 2) + 1] = l;
        }
        if (counts) counts[tid * 4 + 3] = l > 0.0f ? 1 : 0;
    }
}


}  // namespace lvk5
