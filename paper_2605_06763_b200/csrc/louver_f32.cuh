// Louver fp32 query path as ONE persistent kernel per layer (sm_100a): the layer kernel's
// structure (louver_v9.cuh) for caches that keep the reference's fp32 keys and values
// (LouverCache, BASELINE C1). Scores are the normative sequential fp32 dot itself, on the
// CUDA cores: an fp32 key has 24 significant bits, which the bf16 tensor-core split of the
// bf16 path cannot hold, and a fp32 cache serves few q heads per key (G = 1 in the
// reference's cache), so the dots are cheap next to the memory traffic.
//
// Grid = (team, slots): CTA b of a slot's team owns the cells b, b + nb, b + 2 nb, ...
//   A  probe      8-cell tiles of the fp32 summary rows [hi | lo] (one 8 KiB stage per tile
//                 at d = 128); 4 lanes per cell sum max(q hi, q lo) with upward rounding, so
//                 the bound is >= the exact product; a cell survives for head g iff its bound
//                 reaches tau_g - slack_g, slack_g = 2 gamma_(DP+2) sum_c |q_c| colmax_c (the
//                 normative dot's largest deviation from the exact product), or it holds
//                 buffer keys (gate_bounds / query_ta, query.cpp:47-303).
//   B  exact      16-key tasks of the surviving cells through a per-warp 3-stage cp.async
//      + attend   ring: every (key, head) pair's normative dot (core.hpp:17-21, exact_check
//                 query.cpp:22-31) on one lane, online softmax with a lazy reference max,
//                 the attended V rows (selected ∪ buffer unless strict, cache.cpp:48-68)
//                 loaded into the block's stage and folded with fp32 FMAs
//                 (sparse_attention, query.cpp:338-371).
//   C  merge      warp partials -> CTA partial (m, l, o); the team's last CTA (acq_rel
//                 ticket) combines the nb partials.
// Stage layout: row r at r * RB, its 16-byte chunk c at chunk (c ^ (r & 15)), so a lane
// per row (scores) and a row per warp (V fold) both read without bank conflicts.
#pragma once

#include "louver_common.cuh"
#include "louver_kernels.cuh"

namespace lvkf {

using lvk::QueryParams;
using namespace lvc;

struct F32Params {
    QueryParams p;
    const float* sum;  // [slot][cap_cells][2*DP] cell rows [hi | lo]
    int* stickets;     // [slots] merge tickets (self-resetting)
    int nb;            // team CTAs per slot
    int slots;
    unsigned short* glist;  // survivor lists in global scratch when they outgrow smem (else null)
    int list_cap;
    long long sealed;  // cells complete when the query was enqueued
};

template <int DP, int G>
struct CF {
    static constexpr int RB = DP * 4;            // bytes per fp32 row
    static constexpr int STAGE = 16 * RB;        // 16 keys, or 8 summary rows [hi | lo]
    static constexpr int CPR = DP / 4;           // 16-byte chunks per row
    static constexpr int PPL = (16 * G + 31) / 32;  // (key, head) pairs per lane
    static constexpr int DPL = DP / 32;          // output dims per lane
    static constexpr int OFF_Q = 0;              // [G][DP] f32
    static constexpr int OFF_M = OFF_Q + G * DP * 4;
    static constexpr int MISC = 8 * G + 16 * G + 32;
    static constexpr int FIX = (OFF_M + MISC * 4 + 127) / 128 * 128;
    static constexpr int PERW = 3 * STAGE + 16 * G * 4;  // ring, P tile [16][G]
    static constexpr int BUDGET = 223 * 1024;
    static constexpr int NW0 = (BUDGET - FIX) / PERW;
    static constexpr int NW = NW0 > 16 ? 16 : NW0;
    static constexpr int NTHR = NW * 32;
    static constexpr int OFF_W = FIX;
    static constexpr int DYN = OFF_W + NW * PERW;
    static int smem(int list_cap) { return DYN + list_cap * 2; }
    static_assert(NW >= 2, "Louver f32: shared memory budget too small");
    static_assert(DP >= 128, "Louver f32: whole 16-byte chunks per lane in the V fold (DP 128 or 256)");
};

__device__ __forceinline__ unsigned frow(int r, int c, int RB) {  // stage byte offset of chunk c of row r
    return (unsigned)(r * RB + ((c ^ (r & 15)) << 4));
}

template <int DP, int G>
__global__ void __launch_bounds__(CF<DP, G>::NTHR, 1) louver_layer_f32(const __grid_constant__ F32Params fp) {
    using Ge = CF<DP, G>;
    constexpr int NW = Ge::NW, NTHR = Ge::NTHR, RB = Ge::RB, CPR = Ge::CPR, PPL = Ge::PPL, DPL = Ge::DPL;
    const QueryParams& p = fp.p;
    extern __shared__ __align__(128) unsigned char smem[];
    float* qf = reinterpret_cast<float*>(smem + Ge::OFF_Q);
    float* misc = reinterpret_cast<float*>(smem + Ge::OFF_M);
    float* tau_s = misc;            // [G]
    float* taup_s = misc + G;       // [G] probe threshold tau - slack
    float* red = misc + 8 * G;      // [16 G]
    int* iscr = reinterpret_cast<int*>(misc + 24 * G);  // [32]
    unsigned short* slist_s = reinterpret_cast<unsigned short*>(smem + Ge::DYN);
    const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
    const int blk = blockIdx.x, nb = fp.nb;
    unsigned char* wbase = smem + Ge::OFF_W + warp * Ge::PERW;
    const unsigned ring = smem_u32(wbase);
    float* pbuf = reinterpret_cast<float*>(wbase + 3 * Ge::STAGE);  // [16][G]

    asm volatile("griddepcontrol.launch_dependents;\n" ::: "memory");
    bool waited = false;

    for (int slot = blockIdx.y; slot < fp.slots; slot += gridDim.y) {
        const float* Ks = reinterpret_cast<const float*>(p.K) + (size_t)slot * p.cap * DP;
        const float* Vs = reinterpret_cast<const float*>(p.V) + (size_t)slot * p.cap * DP;
        const unsigned char* sumb = reinterpret_cast<const unsigned char*>(fp.sum + (size_t)slot * p.cap_cells * (2 * DP));
        unsigned short* slist = fp.glist ? fp.glist + ((size_t)slot * nb + blk) * fp.list_cap : slist_s;
        if (tid == 0) {
            iscr[2] = 0;  // survivors listed
            iscr[3] = 0;  // tasks claimed
        }
        const long long cap_cells = p.cap_cells;
        // probe tile j of this warp: cells blk + (8 (warp + j NW) + i) nb, i < 8, one stage
        auto p_issue = [&](int j, long long bound) {
            const long long c0 = blk + (long long)8 * (warp + j * NW) * nb;
            if (c0 < bound) {
                const unsigned dst = ring + (j % 3) * Ge::STAGE;
                // 8 rows of 2 DP floats = 16 half-rows of DP floats: half-row h = 2 i + (hi/lo)
                for (int ch = lane; ch < 16 * CPR; ch += 32) {
                    const int hr = ch / CPR, c = ch % CPR;
                    long long cell = c0 + (long long)(hr >> 1) * nb;
                    cell = cell < cap_cells ? cell : cap_cells - 1;  // past the arena: any row, ignored
                    cpa16(dst + frow(hr, c, RB), sumb + (size_t)cell * (8 * DP) + (size_t)(hr & 1) * RB + c * 16);
                }
            }
            cpa_commit();
        };
        bool pre = false;
        if (!waited) {  // sealed summaries depend on nothing: request them before the wait
            const long long c0 = blk + (long long)8 * warp * nb;
            pre = c0 + (long long)8 * 2 * NW * nb + 7LL * nb < fp.sealed;  // tiles 0..2 of the warp
            if (pre)
                for (int j = 0; j < 3; ++j) p_issue(j, cap_cells);
            asm volatile("griddepcontrol.wait;\n" ::: "memory");
            waited = true;
        }
        // ---- setup: q, the probe slack (upward rounding), thresholds
        const long long n = __ldcg(&p.ctr->n);
        const long long indexed = __ldcg(&p.ctr->indexed);
        for (int i = tid; i < G * DP; i += NTHR) qf[i] = __ldcg(p.q + (size_t)slot * G * DP + i);
        if (warp < G) {
            const int g = warp;
            float s = 0.0f;
            for (int c = lane; c < DP; c += 32)
                s = __fadd_ru(s, __fmul_ru(fabsf(__ldcg(p.q + ((size_t)slot * G + g) * DP + c)),
                                           __ldcg(p.colmax + (size_t)slot * DP + c)));
#pragma unroll
            for (int o = 16; o > 0; o >>= 1) s = __fadd_ru(s, __shfl_xor_sync(0xffffffffu, s, o));
            if (lane == 0) {
                const float t = __ldcg(p.tau + (size_t)slot * G + g);
                const float dd = (float)(DP + 2);
                const float gamma = __fdiv_ru(__fmul_ru(dd, 5.9604645e-08f), 1.0f - dd * 5.9604645e-08f);
                const float slack = __fmul_ru(__fmul_ru(2.0f, gamma), s);
                tau_s[g] = t;
                taup_s[g] = __fsub_rd(t, __fmul_ru(slack, 1.0009765625f));
            }
        }
        __syncthreads();
        if (!pre)
            for (int j = 0; j < 3; ++j) p_issue(j, cap_cells);
        const int rl = p.r_log2, r = 1 << rl;
        const long long ncells = (n + r - 1) >> rl;

        // ---- phase A: probe (4 lanes per cell: lane = 4 cell + quarter)
        {
            const int cl = lane >> 2, qt = lane & 3;
            for (int j = 0;; ++j) {
                const long long c0 = blk + (long long)8 * (warp + j * NW) * nb;
                if (c0 >= ncells) break;
                cpa_wait<2>();  // tile j landed (j + 1, j + 2 may pend)
                __syncwarp();
                const unsigned sb = ring + (j % 3) * Ge::STAGE;
                float bnd[G];
#pragma unroll
                for (int g = 0; g < G; ++g) bnd[g] = 0.0f;
                for (int c = qt; c < CPR; c += 4) {  // the quarter's chunks of the cell's hi and lo rows
                    const uint4 h4 = lds16(sb + frow(2 * cl, c, RB));
                    const uint4 l4 = lds16(sb + frow(2 * cl + 1, c, RB));
                    const float hv[4] = {__uint_as_float(h4.x), __uint_as_float(h4.y), __uint_as_float(h4.z), __uint_as_float(h4.w)};
                    const float lv[4] = {__uint_as_float(l4.x), __uint_as_float(l4.y), __uint_as_float(l4.z), __uint_as_float(l4.w)};
#pragma unroll
                    for (int g = 0; g < G; ++g)
#pragma unroll
                        for (int e = 0; e < 4; ++e) {
                            const float qv = qf[g * DP + 4 * c + e];
                            bnd[g] = __fadd_ru(bnd[g], fmaxf(__fmul_ru(qv, hv[e]), __fmul_ru(qv, lv[e])));
                        }
                }
#pragma unroll
                for (int g = 0; g < G; ++g) {  // the 4 quarters' sums, still rounded up
                    bnd[g] = __fadd_ru(bnd[g], __shfl_xor_sync(0xffffffffu, bnd[g], 1));
                    bnd[g] = __fadd_ru(bnd[g], __shfl_xor_sync(0xffffffffu, bnd[g], 2));
                }
                const long long cell = c0 + (long long)cl * nb;
                bool live = false;
                int scan = 0;
                unsigned gm = 0;
                if (cell < ncells) {
                    const long long cs = cell << rl, ce = cs + r;
                    if (ce > indexed) {
                        gm = (1u << G) - 1u;  // holds buffer keys: scanned densely
                    } else {
#pragma unroll
                        for (int g = 0; g < G; ++g)
                            if (bnd[g] >= taup_s[g]) gm |= 1u << g;
                    }
                    scan = (int)((ce < n ? ce : n) - cs);
                    live = true;
                }
                if (p.cand_bits && gm && qt == 0)  // the candidate set: every indexed key of a surviving cell
                    for (long long k = cell << rl; k < ((cell << rl) + r < indexed ? (cell << rl) + r : indexed); ++k)
                        atomicOr(p.cand_bits + (size_t)slot * p.bits_words + (k >> 5), 1u << (k & 31));
                const unsigned m = __ballot_sync(0xffffffffu, gm != 0 && qt == 0);  // bits 0, 4, ... 28
                if (m) {
                    int base = 0;
                    if (lane == 0) base = atomicAdd(iscr + 2, __popc(m));
                    base = __shfl_sync(0xffffffffu, base, 0);
                    if (gm && qt == 0)
                        slist[base + __popc(m & ((1u << lane) - 1u))] = (unsigned short)(8 * (warp + j * NW) + cl);
                }
                if (p.totals) {
                    const int tested = __popc(__ballot_sync(0xffffffffu, live && qt == 0));
                    if (lane == 0) {
                        atomicAdd(p.totals + 0, (unsigned long long)tested);
                        atomicAdd(p.totals + 1, (unsigned long long)__popc(m));
                    }
                }
                if (p.counts) {
#pragma unroll
                    for (int g = 0; g < G; ++g) {
                        const int v = lvk::warp_sum_int(((gm >> g) & 1) && qt == 0 ? scan : 0);
                        if (lane == 0 && v) atomicAdd(p.counts + ((size_t)slot * G + g) * 4 + 2, v);
                    }
                }
                __syncwarp();
                p_issue(j + 3, ncells);
            }
            cpa_wait<0>();
            __syncwarp();
        }
        __syncthreads();  // the CTA's survivor list is complete
        const int nsurv = iscr[2];

        // ---- phase B: exact + attend
        const float scale = p.scale * 1.4426950408889634f;  // log2 units
        const int tpc_l2 = rl - 4;
        float o[G][DPL];
#pragma unroll
        for (int g = 0; g < G; ++g)
#pragma unroll
            for (int e = 0; e < DPL; ++e) o[g][e] = 0.0f;
        float mrun[G], lsum[G];
#pragma unroll
        for (int g = 0; g < G; ++g) {
            mrun[g] = -INFINITY;
            lsum[g] = 0.0f;
        }
        int my_sel = 0, my_att = 0;
        unsigned long long t_keys = 0, t_vals = 0;
        {
            const int ntask = nsurv << tpc_l2;
            const int n32 = (int)n, idx32 = (int)indexed;
            auto key0 = [&](int t) -> int {
                const int cell = blk + (int)slist[t >> tpc_l2] * nb;
                return (cell << rl) + ((t & ((1 << tpc_l2) - 1)) << 4);
            };
            auto k_issue = [&](int t, int kb, int stage) {  // rows past n land as zeros
                if (t < ntask) {
                    const unsigned dst = ring + stage * Ge::STAGE;
                    for (int ch = lane; ch < 16 * CPR; ch += 32) {
                        const int rw = ch / CPR, c = ch % CPR;
                        cpa16z(dst + frow(rw, c, RB), Ks + (size_t)(kb + rw) * DP + 4 * c, kb + rw < n32);
                    }
                }
                cpa_commit();
            };
            int ca = 0, cb = 0;
            if (lane == 0) {
                ca = atomicAdd(iscr + 3, 1);
                cb = atomicAdd(iscr + 3, 1);
            }
            int t = __shfl_sync(0xffffffffu, ca, 0), st = 0;
            int pend_rows = 0;                // rows of the pending V block (task t - 1)
            unsigned pend_mask = 0;           // their attended-row mask
            int k0 = t < ntask ? key0(t) : 0;
            k_issue(t, k0, 0);
            cpa_commit();  // stands for V(t-1)
            while (t < ntask) {
                const int s1 = st == 2 ? 0 : st + 1;
                const int s2 = st == 0 ? 2 : st - 1;  // stage of V(t-1)
                const int tn = __shfl_sync(0xffffffffu, cb, 0);
                if (lane == 0 && tn < ntask) cb = atomicAdd(iscr + 3, 1);
                const int kn = tn < ntask ? key0(tn) : 0;
                k_issue(tn, kn, s1);
                cpa_wait<2>();  // K(t) landed
                __syncwarp();
                const unsigned sb = ring + st * Ge::STAGE;
                // -- normative scores: pair pi = lane + 32 j -> (row pi / G, head pi % G)
                float s[PPL];
                unsigned selb = 0, attb = 0;
#pragma unroll
                for (int jj = 0; jj < PPL; ++jj) {
                    const int pi = lane + 32 * jj, rw = pi / G, g = pi % G;
                    s[jj] = -INFINITY;
                    if (pi < 16 * G && k0 + rw < n32) {
                        float a = 0.0f;
                        for (int c = 0; c < CPR; ++c) {
                            const uint4 kv = lds16(sb + frow(rw, c, RB));
                            a = __fadd_rn(a, __fmul_rn(qf[g * DP + 4 * c + 0], __uint_as_float(kv.x)));
                            a = __fadd_rn(a, __fmul_rn(qf[g * DP + 4 * c + 1], __uint_as_float(kv.y)));
                            a = __fadd_rn(a, __fmul_rn(qf[g * DP + 4 * c + 2], __uint_as_float(kv.z)));
                            a = __fadd_rn(a, __fmul_rn(qf[g * DP + 4 * c + 3], __uint_as_float(kv.w)));
                        }
                        const int kk = k0 + rw;
                        const bool sel = a >= tau_s[g];
                        const bool att = sel || (!p.strict && kk >= idx32);
                        if (sel) {
                            selb |= 1u << jj;
                            ++my_sel;
                            if (p.bits)
                                atomicOr(p.bits + ((size_t)slot * G + g) * p.bits_words + (kk >> 5), 1u << (kk & 31));
                        }
                        if (att) {
                            attb |= 1u << jj;
                            ++my_att;
                            s[jj] = scale * a;
                        }
                    }
                }
                if (p.totals && lane == 0) t_keys += (k0 + 16 <= n32) ? 16 : (n32 > k0 ? n32 - k0 : 0);
                // rows with any attended head
                unsigned amask = 0;
#pragma unroll
                for (int jj = 0; jj < PPL; ++jj) {
                    const unsigned bal = __ballot_sync(0xffffffffu, (attb >> jj) & 1);
                    for (int l = 0; l < 32; ++l)
                        if ((bal >> l) & 1) amask |= 1u << ((l + 32 * jj) / G);
                }
                // online softmax per head, lazy reference max (weights stay <= 2^11.5)
                float alpha[G];
#pragma unroll
                for (int g = 0; g < G; ++g) {
                    float mloc = -INFINITY;
#pragma unroll
                    for (int jj = 0; jj < PPL; ++jj)
                        if ((lane + 32 * jj) % G == g) mloc = fmaxf(mloc, s[jj]);
#pragma unroll
                    for (int of = 16; of > 0; of >>= 1) mloc = fmaxf(mloc, __shfl_xor_sync(0xffffffffu, mloc, of));
                    alpha[g] = 1.0f;
                    if (mloc > mrun[g] + 11.541560327111707f) {
                        if (mrun[g] != -INFINITY) alpha[g] = ex2f(mrun[g] - mloc);
                        mrun[g] = mloc;
                    }
                }
                // the pending V(t-1) fold must see the old weights: fold it first (it lives in
                // stage s2, loaded one task ago), then write this task's weights
                cpa_wait<1>();  // V(t-1) landed (K(t+1) may pend)
                __syncwarp();
                if (pend_mask) {
                    const unsigned vb = ring + s2 * Ge::STAGE;
                    for (int rw = 0; rw < pend_rows; ++rw) {
                        if (!((pend_mask >> rw) & 1)) continue;
                        float vv[DPL];
#pragma unroll
                        for (int e4 = 0; e4 < DPL / 4; ++e4) {
                            const uint4 x = lds16(vb + frow(rw, lane * (DPL / 4) + e4, RB));
                            vv[4 * e4 + 0] = __uint_as_float(x.x);
                            vv[4 * e4 + 1] = __uint_as_float(x.y);
                            vv[4 * e4 + 2] = __uint_as_float(x.z);
                            vv[4 * e4 + 3] = __uint_as_float(x.w);
                        }
#pragma unroll
                        for (int g = 0; g < G; ++g) {
                            const float pw = pbuf[rw * G + g];
#pragma unroll
                            for (int e = 0; e < DPL; ++e) o[g][e] = fmaf(pw, vv[e], o[g][e]);
                        }
                    }
                }
                __syncwarp();  // pbuf reads done
#pragma unroll
                for (int g = 0; g < G; ++g) {
                    if (alpha[g] != 1.0f) {
                        lsum[g] *= alpha[g];
#pragma unroll
                        for (int e = 0; e < DPL; ++e) o[g][e] *= alpha[g];
                    }
                }
#pragma unroll
                for (int jj = 0; jj < PPL; ++jj) {
                    const int pi = lane + 32 * jj;
                    if (pi < 16 * G) {
                        const int g = pi % G;
                        const float pv = s[jj] == -INFINITY ? 0.0f : ex2f(s[jj] - mrun[g]);
                        pbuf[pi] = pv;  // [row][G]
                    }
                }
                __syncwarp();
#pragma unroll
                for (int g = 0; g < G; ++g) {  // l += this task's weights of head g
                    float lp = 0.0f;
                    for (int rw = lane; rw < 16; rw += 32) lp += pbuf[rw * G + g];
#pragma unroll
                    for (int of = 16; of > 0; of >>= 1) lp += __shfl_xor_sync(0xffffffffu, lp, of);
                    lsum[g] += lp;
                }
                // -- V(t): the attended rows into K(t)'s stage (K(t) is consumed)
                if (p.totals && lane == 0) t_vals += __popc(amask);
                if (amask) {
                    const unsigned dst = ring + st * Ge::STAGE;
                    for (int ch = lane; ch < 16 * CPR; ch += 32) {
                        const int rw = ch / CPR, c = ch % CPR;
                        if ((amask >> rw) & 1) cpa16(dst + frow(rw, c, RB), Vs + (size_t)(k0 + rw) * DP + 4 * c);
                    }
                }
                cpa_commit();
                pend_mask = amask;
                pend_rows = 16;
                st = s1;
                t = tn;
                k0 = kn;
            }
            cpa_wait<0>();
            __syncwarp();
            if (pend_mask) {  // the last task's V
                const int s2 = st == 0 ? 2 : st - 1;
                const unsigned vb = ring + s2 * Ge::STAGE;
                for (int rw = 0; rw < pend_rows; ++rw) {
                    if (!((pend_mask >> rw) & 1)) continue;
                    float vv[DPL];
#pragma unroll
                    for (int e4 = 0; e4 < DPL / 4; ++e4) {
                        const uint4 x = lds16(vb + frow(rw, lane * (DPL / 4) + e4, RB));
                        vv[4 * e4 + 0] = __uint_as_float(x.x);
                        vv[4 * e4 + 1] = __uint_as_float(x.y);
                        vv[4 * e4 + 2] = __uint_as_float(x.z);
                        vv[4 * e4 + 3] = __uint_as_float(x.w);
                    }
#pragma unroll
                    for (int g = 0; g < G; ++g) {
                        const float pw = pbuf[rw * G + g];
#pragma unroll
                        for (int e = 0; e < DPL; ++e) o[g][e] = fmaf(pw, vv[e], o[g][e]);
                    }
                }
            }
            __syncwarp();
        }

        // ---- statistics
        if (p.counts) {
            // G divides 32: every pair of a lane belongs to head lane % G
            int v0 = my_sel, v1 = my_att;
#pragma unroll
            for (int of = 16; of >= G; of >>= 1) {
                v0 += __shfl_xor_sync(0xffffffffu, v0, of);
                v1 += __shfl_xor_sync(0xffffffffu, v1, of);
            }
            if (lane < G) {
                int* c = p.counts + ((size_t)slot * G + lane) * 4;
                if (v0) atomicAdd(c + 0, v0);
                if (v1) atomicAdd(c + 1, v1);
            }
        }
        if (p.totals && lane == 0) {
            if (t_keys) atomicAdd(p.totals + 2, t_keys);
            if (t_vals) atomicAdd(p.totals + 3, t_vals);
        }

        // ---- warp partials -> CTA partial [G][DP+2] (m, l, o), then the team merge
        constexpr int Wd = G * (DP + 2);
        float* wred = reinterpret_cast<float*>(smem + Ge::OFF_W);  // [NW][Wd] over the rings
        float* shw = red;                                           // [NW][G] weights
        __syncthreads();
        {
            float* w = wred + warp * Wd;
#pragma unroll
            for (int g = 0; g < G; ++g) {
                if (lane == 0) {
                    w[g * (DP + 2)] = mrun[g] * 0.6931471805599453f;  // back to nats
                    w[g * (DP + 2) + 1] = lsum[g];
                }
#pragma unroll
                for (int e = 0; e < DPL; ++e) w[g * (DP + 2) + 2 + lane * DPL + e] = o[g][e];
            }
        }
        __syncthreads();
        float* part = p.partial_ws + ((size_t)slot * nb + blk) * Wd;
        for (int g = warp; g < G; g += NW) {
            const float mw = lane < NW ? wred[lane * Wd + g * (DP + 2)] : -INFINITY;
            const float lw = lane < NW ? wred[lane * Wd + g * (DP + 2) + 1] : 0.0f;
            float mm = mw;
#pragma unroll
            for (int o2 = 16; o2 > 0; o2 >>= 1) mm = fmaxf(mm, __shfl_xor_sync(0xffffffffu, mm, o2));
            const float a = mw == -INFINITY ? 0.0f : __expf(mw - mm);
            if (lane < NW) shw[lane * G + g] = a;
            float l = a * lw;
#pragma unroll
            for (int o2 = 16; o2 > 0; o2 >>= 1) l += __shfl_xor_sync(0xffffffffu, l, o2);
            if (lane == 0) {
                part[g * (DP + 2)] = l > 0.0f ? mm : -INFINITY;
                part[g * (DP + 2) + 1] = l;
            }
        }
        __syncthreads();
        for (int i = tid; i < G * DP; i += NTHR) {
            const int g = i / DP, c = i % DP;
            float sacc = 0.0f;
#pragma unroll 4
            for (int w = 0; w < NW; ++w) sacc = fmaf(shw[w * G + g], wred[w * Wd + g * (DP + 2) + 2 + c], sacc);
            part[g * (DP + 2) + 2 + c] = sacc;
        }
        int* ticket = fp.stickets + slot;
        __syncthreads();
        if (tid == 0) iscr[1] = atom_add_acq_rel(ticket, 1) == nb - 1;
        __syncthreads();
        if (iscr[1]) {
            const float* src = p.partial_ws + (size_t)slot * nb * Wd;
            float* M = reinterpret_cast<float*>(smem + Ge::OFF_W);
            float* L = M + G;
            float* wgt = M + 2 * G;                     // [nb][G]
            for (int g = warp; g < G; g += NW) {
                float mm = -INFINITY;
                for (int s2 = lane; s2 < nb; s2 += 32) mm = fmaxf(mm, __ldcg(src + (size_t)s2 * Wd + g * (DP + 2)));
#pragma unroll
                for (int o2 = 16; o2 > 0; o2 >>= 1) mm = fmaxf(mm, __shfl_xor_sync(0xffffffffu, mm, o2));
                float l = 0.0f;
                for (int s2 = lane; s2 < nb; s2 += 32) {
                    const float ms = __ldcg(src + (size_t)s2 * Wd + g * (DP + 2));
                    const float wv = ms == -INFINITY ? 0.0f : __expf(ms - mm);
                    wgt[s2 * G + g] = wv;
                    l += wv * __ldcg(src + (size_t)s2 * Wd + g * (DP + 2) + 1);
                }
#pragma unroll
                for (int o2 = 16; o2 > 0; o2 >>= 1) l += __shfl_xor_sync(0xffffffffu, l, o2);
                if (lane == 0) {
                    M[g] = mm;
                    L[g] = l;
                }
            }
            __syncthreads();
            for (int i = tid; i < G * DP; i += NTHR) {
                const int g = i / DP, c = i % DP;
                float a = 0.0f;
                for (int s2 = 0; s2 < nb; ++s2) a = fmaf(wgt[s2 * G + g], __ldcg(src + (size_t)s2 * Wd + g * (DP + 2) + 2 + c), a);
                const float l = L[g];
                if (p.out) p.out[((size_t)slot * G + g) * DP + c] = l > 0.0f ? a / l : 0.0f;
                if (p.partial_out) p.partial_out[(size_t)slot * Wd + g * (DP + 2) + 2 + c] = a;
            }
            if (tid < G) {
                if (p.partial_out) {
                    p.partial_out[(size_t)slot * Wd + tid * (DP + 2)] = L[tid] > 0.0f ? M[tid] : -INFINITY;
                    p.partial_out[(size_t)slot * Wd + tid * (DP + 2) + 1] = L[tid];
                }
                if (p.counts) p.counts[((size_t)slot * G + tid) * 4 + 3] = L[tid] > 0.0f ? 1 : 0;
            }
            if (tid == 0) *ticket = 0;
        }
        __syncthreads();
        __syncthreads();  // the rings served as merge scratch
    }
}

cudaError_t launch_layer_f32(int DP, int G, F32Params fp, int slots, int sms, cudaStream_t st, int* geo);

}  // namespace lvkf
