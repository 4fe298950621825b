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
    const int tid = threadIdx.x;
    constexpr int W = G * (DP + 2);
    if (tid < G) {
        float m = -INFINITY;
        for (int s = 0; s < P; ++s) m = fmaxf(m, __ldcg(src + (size_t)s * W + tid * (DP + 2)));
        float l = 0.0f;
        for (int s = 0; s < P; ++s) {
            const float ms = __ldcg(src + (size_t)s * W + tid * (DP + 2));
            const float w = ms == -INFINITY ? 0.0f : expf(ms - m);
            shw[s * G + tid] = w;
            l += w * __ldcg(src + (size_t)s * W + tid * (DP + 2) + 1);
        }
        shw[P * G + tid] = m;
        shw[P * G + G + tid] = l;
    }
    __syncthreads();
    for (int i = tid; i < G * DP; i += kT) {
        const int g = i / DP, c = i % DP;
        float acc = 0.0f;
        for (int s = 0; s < P; ++s) {
            const float w = shw[s * G + g];
            if (w != 0.0f) acc = fmaf(w, __ldcg(src + (size_t)s * W + g * (DP + 2) + 2 + c), acc);
        }
        const float l = shw[P * G + G + g];
        if (dst) dst[g * (DP + 2) + 2 + c] = acc;
        if (out) out[g * DP + c] = l > 0.0f ? acc / l : 0.0f;
        if (part_out) part_out[g * (DP + 2) + 2 + c] = acc;
    }
    if (tid < G) {
        const float m = shw[P * G + tid], l = shw[P * G + G + tid];
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

template <int DP, int G>
__global__ void __launch_bounds__(kT, 2) louver_exact_v5(const __grid_constant__ V5Params vp) {
    using Ge = E5<DP, G>;
    const QueryParams& p = vp.p;
    extern __shared__ __align__(16) unsigned char smem[];
    uint2* fr = reinterpret_cast<uint2*>(smem + Ge::OFF_FR);
    float* qf = reinterpret_cast<float*>(smem + Ge::OFF_Q);
    float* misc = reinterpret_cast<float*>(smem + Ge::OFF_M);
    float* tau_s = misc;         // [G]
    float* marg = misc + G;      // [G]
    float* S = misc + 2 * G;     // [G]
    float* red = misc + 4 * G;   // [kW*G]
    int* iscr = reinterpret_cast<int*>(misc + 4 * G + kW * G);  // [8]
    unsigned* klist = reinterpret_cast<unsigned*>(smem + Ge::OFF_KL);
    unsigned* ucm = reinterpret_cast<unsigned*>(smem + Ge::FIXED);  // [tiles] masks
    unsigned* upre = ucm + vp.tiles;                                // [tiles] exclusive row prefix
    const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
    const int slot = blockIdx.y, blk = blockIdx.x;
    unsigned char* ws = smem + Ge::OFF_WS + warp * Ge::WSZ;
    float* ct = reinterpret_cast<float*>(ws);
    float* wsc = ct + Ge::WCT;
    const int q = lane & 3;
    const __nv_bfloat16* Ks = reinterpret_cast<const __nv_bfloat16*>(p.K) + (size_t)slot * p.cap * DP;
    const __nv_bfloat16* Vs = reinterpret_cast<const __nv_bfloat16*>(p.V) + (size_t)slot * p.cap * DP;

    // ---- setup independent of the probe (overlaps it under programmatic launch)
    setup_q<DP, G>(p.q + (size_t)slot * G * DP, p.colmax + (size_t)slot * DP, qf, red, S);
    if (tid < G) {
        tau_s[tid] = p.tau[(size_t)slot * G + tid];
        marg[tid] = __fmul_ru(S[tid], 1.220703125e-4f);  // 2^-13 S
    }
    for (int i = tid; i < Ge::KS * Ge::NT * 32; i += kT) {
        const int l = i & 31, nt = (i >> 5) % Ge::NT, t = (i >> 5) / Ge::NT;
        fr[i] = b_frag<G, 3>(t, nt, l, [&](int k, int g) { return qf[g * (DP + 4) + k]; });
    }
    asm volatile("griddepcontrol.wait;\n" ::: "memory");  // probe results visible from here

    const long long n = p.ctr->n;
    const long long indexed = p.ctr->indexed;
    const int rl = p.r_log2, r = 1 << rl;
    const long long ncells = (n + r - 1) >> rl;
    const int ntile = (int)((ncells + 15) >> 4);
    for (int u = tid; u < ntile; u += kT) ucm[u] = vp.cmask[(size_t)slot * vp.tiles + u];
    __syncthreads();
    {
        const int per = (ntile + kT - 1) / kT;
        const int u0 = tid * per;
        int s = 0;
        for (int u = u0; u < u0 + per && u < ntile; ++u) s += __popc(ucm[u]) << rl;
        int incl = s;
#pragma unroll
        for (int o = 1; o < 32; o <<= 1) {
            const int t = __shfl_up_sync(0xffffffffu, incl, o);
            if (lane >= o) incl += t;
        }
        if (lane == 31) iscr[warp] = incl;
        __syncthreads();
        int basep = 0, total = 0;
        for (int w = 0; w < kW; ++w) {
            basep += w < warp ? iscr[w] : 0;
            total += iscr[w];
        }
        int run = basep + incl - s;
        for (int u = u0; u < u0 + per && u < ntile; ++u) {
            upre[u] = (unsigned)run;
            run += __popc(ucm[u]) << rl;
        }
        __syncthreads();
        if (tid == 0) iscr[0] = total;
        __syncthreads();
    }
    const long long total = iscr[0];
    const long long lo = total * blk / vp.nb, hi = total * (blk + 1) / vp.nb;

    // ---- per-warp online softmax state
    constexpr int VPL = DP / 32;  // V dims per lane
    float o[G][VPL], lsum[G], mrun[G];
#pragma unroll
    for (int g = 0; g < G; ++g) {
        lsum[g] = 0.0f;
        mrun[g] = -INFINITY;
#pragma unroll
        for (int e = 0; e < VPL; ++e) o[g][e] = 0.0f;
    }
    int st_sel[G], st_att[G];
#pragma unroll
    for (int g = 0; g < G; ++g) st_sel[g] = st_att[g] = 0;
    unsigned long long t_keys = 0, t_vals = 0;

    for (long long seg = lo; seg < hi; seg += Ge::KL) {
        const int nrow = (int)(hi - seg < Ge::KL ? hi - seg : Ge::KL);
        // row -> key for the whole segment, all threads (unit by binary search, cell by bit select)
        for (int i = tid; i < nrow; i += kT) {
            const long long row = seg + i;
            int a = 0, b = ntile - 1;
            while (a < b) {
                const int mid = (a + b + 1) >> 1;
                if ((long long)upre[mid] <= row) a = mid; else b = mid - 1;
            }
            const int off = (int)(row - upre[a]);
            unsigned m = ucm[a];
            for (int j = 0; j < (off >> rl); ++j) m &= m - 1;
            unsigned key = 0xffffffffu;
            if (m != 0u) {
                const long long kk = ((long long)a * 16 + (__ffs(m) - 1)) * r + (off & (r - 1));
                if (kk >= 0 && kk < n) key = (unsigned)kk;
            }
            klist[i] = key;
        }
        if (tid == 0) iscr[1] = 0;
        __syncthreads();
        const int ntask = (nrow + 15) >> 4;
        while (true) {
            int task = 0;
            if (lane == 0) task = atomicAdd(iscr + 1, 1);
            task = __shfl_sync(0xffffffffu, task, 0);
            if (task >= ntask) break;
            const int r0i = task * 16;
            const unsigned key = lane < 16 && r0i + lane < nrow ? klist[r0i + lane] : 0xffffffffu;
            const unsigned k0 = __shfl_sync(0xffffffffu, key, lane >> 2);
            const unsigned k1 = __shfl_sync(0xffffffffu, key, (lane >> 2) + 8);
            const unsigned char* row0 =
                reinterpret_cast<const unsigned char*>(Ks + (size_t)(k0 == 0xffffffffu ? 0 : k0) * DP);
            const unsigned char* row1 =
                reinterpret_cast<const unsigned char*>(Ks + (size_t)(k1 == 0xffffffffu ? 0 : k1) * DP);
            constexpr int NP = DP / 32;
            uint4 u0[NP], u1[NP];
#pragma unroll
            for (int pp = 0; pp < NP; ++pp) {
                u0[pp] = ldg16(row0 + (32 * pp + 8 * q) * 2);
                u1[pp] = ldg16(row1 + (32 * pp + 8 * q) * 2);
            }
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
#pragma unroll
            for (int t = 0; t < Ge::NT; ++t) {
                const int rw = lane >> 2, col = t * 8 + 2 * q;
                ct[rw * 8 * Ge::NT + col] = acc[t][0];
                ct[rw * 8 * Ge::NT + col + 1] = acc[t][1];
                ct[(rw + 8) * 8 * Ge::NT + col] = acc[t][2];
                ct[(rw + 8) * 8 * Ge::NT + col + 1] = acc[t][3];
            }
            __syncwarp();
            // classify (row, g): fast decides outside tau +- margin, else the normative dot
            for (int pi = lane; pi < 16 * G; pi += 32) {
                const int rw = pi / G, g = pi % G;
                const unsigned kk = r0i + rw < nrow ? klist[r0i + rw] : 0xffffffffu;
                float s = -INFINITY;
                if (kk != 0xffffffffu) {
                    const float* c = ct + rw * 8 * Ge::NT;
                    float sc = (c[g] + c[G + g]) + c[2 * G + g];
                    bool sel = sc >= tau_s[g] + marg[g];
                    if (!sel && sc >= tau_s[g] - marg[g]) {  // undecided: normative dot (core.hpp:17-21)
                        const unsigned char* kr = reinterpret_cast<const unsigned char*>(Ks + (size_t)kk * DP);
                        const float* qg = qf + g * (DP + 4);
                        float acc2 = 0.0f;
                        for (int cc = 0; cc < DP / 8; ++cc) {
                            const uint4 kv = ldg16(kr + cc * 16);
                            float kf[8];
                            lvk::unpack16<__nv_bfloat16>(kv, kf);
#pragma unroll
                            for (int e2 = 0; e2 < 8; ++e2) acc2 = __fadd_rn(acc2, __fmul_rn(qg[cc * 8 + e2], kf[e2]));
                        }
                        sc = acc2;
                        sel = acc2 >= tau_s[g];
                    }
                    const bool in_buf = (long long)kk >= indexed;
                    if (sel) {
                        ++st_sel[g];
                        if (p.bits) atomicOr(p.bits + ((size_t)slot * G + g) * p.bits_words + (kk >> 5), 1u << (kk & 31));
                    }
                    if (sel || (in_buf && !p.strict)) {
                        s = sc;
                        ++st_att[g];
                    }
                }
                wsc[pi] = s;
            }
            __syncwarp();
            // task max per q head (lane < 16 owns row lane), ILP over g
            float sv[G], mx[G];
#pragma unroll
            for (int g = 0; g < G; ++g) {
                sv[g] = lane < 16 ? wsc[lane * G + g] : -INFINITY;
                mx[g] = sv[g] == -INFINITY ? -INFINITY : p.scale * sv[g];
            }
            bool att = false;
#pragma unroll
            for (int g = 0; g < G; ++g) att |= sv[g] != -INFINITY;
            const unsigned amask = __ballot_sync(0xffffffffu, att) & 0xffffu;
            const unsigned vkeys = __ballot_sync(0xffffffffu, key != 0xffffffffu);
            if (lane == 0) t_keys += __popc(vkeys);
            __syncwarp();
            if (amask == 0) continue;
            if (lane == 0) t_vals += __popc(amask);
#pragma unroll
            for (int of = 16; of > 0; of >>= 1)
#pragma unroll
                for (int g = 0; g < G; ++g) mx[g] = fmaxf(mx[g], __shfl_xor_sync(0xffffffffu, mx[g], of));
            float pl[G], ls[G];
#pragma unroll
            for (int g = 0; g < G; ++g) {
                const float mnew = fmaxf(mrun[g], mx[g]);
                const float alpha = mrun[g] == -INFINITY ? 0.0f : __expf(mrun[g] - mnew);
                mrun[g] = mnew;
                lsum[g] *= alpha;
#pragma unroll
                for (int e = 0; e < VPL; ++e) o[g][e] *= alpha;
                pl[g] = sv[g] == -INFINITY ? 0.0f : __expf(p.scale * sv[g] - mnew);
                ls[g] = pl[g];
            }
#pragma unroll
            for (int of = 16; of > 0; of >>= 1)
#pragma unroll
                for (int g = 0; g < G; ++g) ls[g] += __shfl_xor_sync(0xffffffffu, ls[g], of);
#pragma unroll
            for (int g = 0; g < G; ++g) lsum[g] += ls[g];
            // V rows of attended keys, 8 per batch (8 bytes per lane at DP=128)
            unsigned m = amask;
            while (m) {
                uint4 vv[8];
                int rws[8];
                int cnt = 0;
#pragma unroll
                for (int i = 0; i < 8; ++i) {
                    rws[i] = -1;
                    if (m) {
                        const int rw = __ffs(m) - 1;
                        m &= m - 1;
                        rws[i] = rw;
                        const unsigned kv = __shfl_sync(0xffffffffu, key, rw);
                        vv[i] = ldg_v<VPL>(reinterpret_cast<const unsigned char*>(Vs + (size_t)kv * DP) + lane * VPL * 2);
                        ++cnt;
                    }
                }
#pragma unroll
                for (int i = 0; i < 8; ++i) {
                    if (i < cnt) {
                        float vf[8];
                        const unsigned vw[4] = {vv[i].x, vv[i].y, vv[i].z, vv[i].w};
#pragma unroll
                        for (int e = 0; e < VPL; ++e) vf[e] = (e & 1) ? lvk::bf_hi(vw[e >> 1]) : lvk::bf_lo(vw[e >> 1]);
#pragma unroll
                        for (int g = 0; g < G; ++g) {
                            const float pw = __shfl_sync(0xffffffffu, pl[g], rws[i]);
#pragma unroll
                            for (int e = 0; e < VPL; ++e) o[g][e] = fmaf(pw, vf[e], o[g][e]);
                        }
                    }
                }
            }
        }
        __syncthreads();  // klist is rewritten by the next segment
    }

    // ---- statistics
    if (p.counts) {
#pragma unroll
        for (int g = 0; g < G; ++g) {
            const int s0 = lvk::warp_sum_int(st_sel[g]);
            const int s1 = lvk::warp_sum_int(st_att[g]);
            if (lane == 0) {
                int* c = p.counts + ((size_t)slot * G + g) * 4;
                if (s0) atomicAdd(c + 0, s0);
                if (s1) atomicAdd(c + 1, s1);
            }
        }
    }
    if (p.totals && lane == 0) {
        if (t_keys) atomicAdd(p.totals + 2, t_keys);
        if (t_vals) atomicAdd(p.totals + 3, t_vals);
    }

    // ---- warp partials -> CTA partial
    __syncthreads();
    float* wred = reinterpret_cast<float*>(smem + Ge::OFF_WS);  // [kW][G][DP+2]
#pragma unroll
    for (int g = 0; g < G; ++g) {
        float* w = wred + (warp * G + g) * (DP + 2);
        if (lane == 0) {
            w[0] = mrun[g];
            w[1] = lsum[g];
        }
#pragma unroll
        for (int e = 0; e < VPL; ++e) w[2 + lane * VPL + e] = o[g][e];
    }
    __syncthreads();
    constexpr int Wd = G * (DP + 2);
    float* part = p.partial_ws + ((size_t)slot * vp.nb + blk) * Wd;
    float* shw = reinterpret_cast<float*>(smem + Ge::OFF_KL);  // the key list is no longer needed
    if (tid < G) {
        float mm = -INFINITY;
        for (int w = 0; w < kW; ++w) mm = fmaxf(mm, wred[(w * G + tid) * (DP + 2)]);
        float l = 0.0f;
        for (int w = 0; w < kW; ++w) {
            const float mw = wred[(w * G + tid) * (DP + 2)];
            const float a = mw == -INFINITY ? 0.0f : expf(mw - mm);
            shw[w * G + tid] = a;
            l += a * wred[(w * G + tid) * (DP + 2) + 1];
        }
        part[tid * (DP + 2)] = l > 0.0f ? mm : -INFINITY;
        part[tid * (DP + 2) + 1] = l;
    }
    __syncthreads();
    for (int i = tid; i < G * DP; i += kT) {
        const int g = i / DP, c = i % DP;
        float s = 0.0f;
        for (int w = 0; w < kW; ++w) s = fmaf(shw[w * G + g], wred[(w * G + g) * (DP + 2) + 2 + c], s);
        part[g * (DP + 2) + 2 + c] = s;
    }

    // ---- two-level merge
    __threadfence();
    __syncthreads();
    int* flag = iscr + 4;
    const int grp = blk / kMG;
    const int members = vp.nb - grp * kMG < kMG ? vp.nb - grp * kMG : kMG;
    if (tid == 0) *flag = atomicAdd(vp.gtickets + slot * vp.ngroups + grp, 1) == members - 1;
    __syncthreads();
    if (!*flag) return;
    __threadfence();
    merge5<DP, G>(p.partial_ws + ((size_t)slot * vp.nb + grp * kMG) * Wd, members,
                  vp.gpart + ((size_t)slot * vp.ngroups + grp) * Wd, nullptr, nullptr, nullptr, shw);
    if (tid == 0) vp.gtickets[slot * vp.ngroups + grp] = 0;
    __threadfence();
    __syncthreads();
    if (tid == 0) *flag = atomicAdd(vp.stickets + slot, 1) == vp.ngroups - 1;
    __syncthreads();
    if (!*flag) return;
    __threadfence();
    merge5<DP, G>(vp.gpart + (size_t)slot * vp.ngroups * Wd, vp.ngroups, nullptr,
                  p.out ? p.out + (size_t)slot * G * DP : nullptr,
                  p.partial_out ? p.partial_out + (size_t)slot * Wd : nullptr,
                  p.counts ? p.counts + (size_t)slot * G * 4 : nullptr, shw);
    if (tid == 0) vp.stickets[slot] = 0;
}

cudaError_t launch_query_v5(int DP, int G, const V5Params& vp, int slots, cudaStream_t st);

}  // namespace lvk5
