// Louver bf16 query path, exact + attend stage (K2) as a cell stream (sm_100a).
//
// The probe (K1, louver_probe_v5) leaves one survivor bit per cell. A surviving
// cell is 16*k contiguous keys, i.e. one or more 4 KB blocks of bf16 rows -- the
// shape a B200 gathers at ~6+ TB/s when each warp keeps a block in flight
// (tools/micro/gather_bw.cu). So K2 is a stream of 16-row tasks (task = 16
// consecutive rows of a surviving cell): the surviving cells of a slot are
// split evenly over its CTAs, tasks round-robin over warps, and every warp keeps
// the NEXT task's key block in flight (register ping-pong) while it scores the
// current one on the tensor cores (A fragments straight from the loaded
// registers, q split into three bf16 parts), settles pairs within 2^-13 S_g of
// tau with the normative sequential fp32 dot (core.hpp:17-21), gathers the V
// rows of attended pairs (selected ∪ buffer, cache.cpp:48-68) and folds them
// into a per-warp online softmax. Warps, then CTAs (two-level ticket tree), merge.
#pragma once

#include "louver_v5.cuh"

namespace lvk7 {

using lvk::QueryParams;
using namespace lvk5;

template <int DP, int G>
struct C7 {
    static constexpr int NT = (3 * G + 7) / 8;
    static constexpr int KS = DP / 16;
    static constexpr int NP = DP / 32;
    static constexpr int CL = 4096;                                   // surviving cells per list segment
    static constexpr int OFF_FR = 0;                                  // [KS][NT][32] uint2
    static constexpr int OFF_Q = OFF_FR + KS * NT * 32 * 8;           // [G][DP+4]
    static constexpr int OFF_M = OFF_Q + G * (DP + 4) * 4;            // misc
    static constexpr int MISC = 4 * G + kW * G + 16;
    static constexpr int OFF_CL = (OFF_M + MISC * 4 + 15) / 16 * 16;  // [CL] cell ids
    static constexpr int OFF_WS = OFF_CL + CL * 4;                    // per-warp C tile + scores
    static constexpr int WCT = 16 * 8 * NT;
    static constexpr int WSZ = (WCT + 16 * G) * 4;
    static constexpr int SZ_WS = kW * WSZ;
    static constexpr int SZ_RED = kW * G * (DP + 2) * 4;
    static constexpr int FIXED = OFF_WS + (SZ_WS > SZ_RED ? SZ_WS : SZ_RED);
    static int smem(int tiles) { return FIXED + tiles * 8; }          // masks + prefix
};

template <int DP, int G>
__global__ void __launch_bounds__(kT, 2) louver_cells_v7(const __grid_constant__ V5Params vp) {
    using Ge = C7<DP, G>;
    const QueryParams& p = vp.p;
    extern __shared__ __align__(16) unsigned char smem[];
    uint2* fr = reinterpret_cast<uint2*>(smem + Ge::OFF_FR);
    float* qf = reinterpret_cast<float*>(smem + Ge::OFF_Q);
    float* misc = reinterpret_cast<float*>(smem + Ge::OFF_M);
    float* tau_s = misc;
    float* marg = misc + G;
    float* S = misc + 2 * G;
    float* red = misc + 4 * G;
    int* iscr = reinterpret_cast<int*>(misc + 4 * G + kW * G);  // 16 ints
    unsigned* clist = reinterpret_cast<unsigned*>(smem + Ge::OFF_CL);
    unsigned* ucm = reinterpret_cast<unsigned*>(smem + Ge::FIXED);
    unsigned* upre = ucm + vp.tiles;
    const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
    const int slot = blockIdx.y, blk = blockIdx.x;
    float* ct = reinterpret_cast<float*>(smem + Ge::OFF_WS + warp * Ge::WSZ);
    float* wsc = ct + Ge::WCT;
    const int q = lane & 3;
    const __nv_bfloat16* Ks = reinterpret_cast<const __nv_bfloat16*>(p.K) + (size_t)slot * p.cap * DP;
    const __nv_bfloat16* Vs = reinterpret_cast<const __nv_bfloat16*>(p.V) + (size_t)slot * p.cap * DP;

    long long* trace = p.tot_trace ? p.tot_trace + ((size_t)slot * vp.nb + blk) * 16 : nullptr;
#define LV7_TRACE(i) \
    if (trace && tid == 0) trace[i] = lvk2::gtimer();
    LV7_TRACE(0)
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
    LV7_TRACE(1)
    asm volatile("griddepcontrol.wait;\n" ::: "memory");  // survivor masks visible
    LV7_TRACE(2)

    const long long n = p.ctr->n;
    const long long indexed = p.ctr->indexed;
    const int rl = p.r_log2, r = 1 << rl;
    const int tpc = r >> 4;  // 16-row tasks per cell
    const long long ncells = (n + r - 1) >> rl;
    const int ntile = (int)((ncells + 15) >> 4);
    {
        const unsigned short* cm = vp.cmask + (size_t)slot * vp.tiles;
        for (int u0 = 0; u0 < ntile; u0 += 4 * kT) {  // 4 independent loads in flight per thread
            unsigned v[4];
#pragma unroll
            for (int k = 0; k < 4; ++k) {
                const int u = u0 + k * kT + tid;
                v[k] = u < ntile ? (unsigned)cm[u] : 0u;
            }
#pragma unroll
            for (int k = 0; k < 4; ++k) {
                const int u = u0 + k * kT + tid;
                if (u < ntile) ucm[u] = v[k];
            }
        }
    }
    __syncthreads();
    // exclusive prefix of surviving cells per tile
    {
        const int per = (ntile + kT - 1) / kT;
        const int u0 = tid * per;
        int s = 0;
        for (int u = u0; u < u0 + per && u < ntile; ++u) s += __popc(ucm[u]);
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
            run += __popc(ucm[u]);
        }
        __syncthreads();
        if (tid == 0) iscr[8] = total;
        __syncthreads();
    }
    LV7_TRACE(3)
    const long long cs_total = iscr[8];
    const long long c_lo = cs_total * blk / vp.nb, c_hi = cs_total * (blk + 1) / vp.nb;

    constexpr int VPL = DP / 32;
    float o[G][VPL], lsum[G], mrun[G];
#pragma unroll
    for (int g = 0; g < G; ++g) {
        lsum[g] = 0.0f;
        mrun[g] = -INFINITY;
#pragma unroll
        for (int e = 0; e < VPL; ++e) o[g][e] = 0.0f;
    }
    int my_sel = 0, my_att = 0;  // pair counters of this lane's q head g = lane % G
    unsigned long long t_keys = 0, t_vals = 0;
    long long cy_mma = 0, cy_cls = 0, cy_att = 0, n_und = 0, n_task = 0;
    float tmp_unused = 0.0f;
    (void)tmp_unused;

    for (long long seg = c_lo; seg < c_hi; seg += Ge::CL) {
        const int ncell = (int)(c_hi - seg < Ge::CL ? c_hi - seg : Ge::CL);
        // surviving cell ids of the segment (tile by binary search, cell by bit select)
        for (int i = tid; i < ncell; i += kT) {
            const long long c = seg + i;
            int a = 0, b = ntile - 1;
            while (a < b) {
                const int mid = (a + b + 1) >> 1;
                if ((long long)upre[mid] <= c) a = mid; else b = mid - 1;
            }
            unsigned m = ucm[a];
            for (int j = 0; j < (int)(c - upre[a]); ++j) m &= m - 1;
            clist[i] = (unsigned)(a * 16 + __ffs(m) - 1);
        }
        __syncthreads();
        const int ntask = ncell * tpc;
        // first key of task t; rows past n are read (inside the arena) and ignored
        auto task_key0 = [&](int t) -> long long {
            return ((long long)clist[t / tpc] << rl) + (long long)(t % tpc) * 16;
        };
        constexpr int NP = Ge::NP;
        uint4 ua0[NP], ua1[NP], ub0[NP], ub1[NP];
        auto load = [&](int t, uint4 (&u0)[NP], uint4 (&u1)[NP]) {
            const long long k0 = task_key0(t);
            const unsigned char* row0 = reinterpret_cast<const unsigned char*>(Ks + (size_t)(k0 + (lane >> 2)) * DP);
            const unsigned char* row1 = row0 + 8 * DP * 2;
#pragma unroll
            for (int pp = 0; pp < NP; ++pp) {
                u0[pp] = ldg16(row0 + (32 * pp + 8 * q) * 2);
                u1[pp] = ldg16(row1 + (32 * pp + 8 * q) * 2);
            }
        };
        auto process = [&](int t, const uint4 (&u0)[NP], const uint4 (&u1)[NP]) {
            const long long k0 = task_key0(t);
            const long long cyc0 = clock64();
            ++n_task;
            float acc[2][Ge::NT][4];
#pragma unroll
            for (int h = 0; h < 2; ++h)
#pragma unroll
                for (int nt = 0; nt < Ge::NT; ++nt) acc[h][nt][0] = acc[h][nt][1] = acc[h][nt][2] = acc[h][nt][3] = 0.0f;
#pragma unroll
            for (int pp = 0; pp < NP; ++pp) {
                const unsigned a0[4] = {u0[pp].x, u1[pp].x, u0[pp].y, u1[pp].y};
                const unsigned a1[4] = {u0[pp].z, u1[pp].z, u0[pp].w, u1[pp].w};
#pragma unroll
                for (int nt = 0; nt < Ge::NT; ++nt) {
                    const uint2 b0 = fr[((2 * pp) * Ge::NT + nt) * 32 + lane];
                    const uint2 b1 = fr[((2 * pp + 1) * Ge::NT + nt) * 32 + lane];
                    mma16816(acc[0][nt], a0, b0.x, b0.y);
                    mma16816(acc[1][nt], a1, b1.x, b1.y);
                }
            }
#pragma unroll
            for (int nt = 0; nt < Ge::NT; ++nt) {
                const int rw = lane >> 2, col = nt * 8 + 2 * q;
                ct[rw * 8 * Ge::NT + col] = acc[0][nt][0] + acc[1][nt][0];
                ct[rw * 8 * Ge::NT + col + 1] = acc[0][nt][1] + acc[1][nt][1];
                ct[(rw + 8) * 8 * Ge::NT + col] = acc[0][nt][2] + acc[1][nt][2];
                ct[(rw + 8) * 8 * Ge::NT + col + 1] = acc[0][nt][3] + acc[1][nt][3];
            }
            __syncwarp();
            const long long cyc1 = clock64();
            cy_mma += cyc1 - cyc0;
            // classify: lane handles pairs (row, g = lane % G); fast score decides
            // outside tau +- margin, the normative dot inside
            const int g = lane % G;
            for (int pi = lane; pi < 16 * G; pi += 32) {
                const int rw = pi / G;
                const long long kk = k0 + rw;
                float s = -INFINITY;
                if (kk < n) {
                    const float* c = ct + rw * 8 * Ge::NT;
                    float sc = (c[g] + c[G + g]) + c[2 * G + g];
                    bool sel = sc >= tau_s[g] + marg[g];
                    if (!sel && sc >= tau_s[g] - marg[g]) {
                        ++n_und;
                        const unsigned char* kr = reinterpret_cast<const unsigned char*>(Ks + (size_t)kk * DP);
                        const float* qg = qf + g * (DP + 4);
                        float a2 = 0.0f;
                        for (int cc = 0; cc < DP / 8; ++cc) {
                            const uint4 kv = ldg16(kr + cc * 16);
                            float kf[8];
                            lvk::unpack16<__nv_bfloat16>(kv, kf);
#pragma unroll
                            for (int e2 = 0; e2 < 8; ++e2) a2 = __fadd_rn(a2, __fmul_rn(qg[cc * 8 + e2], kf[e2]));
                        }
                        sc = a2;
                        sel = a2 >= tau_s[g];
                    }
                    const bool in_buf = kk >= indexed;
                    if (sel) {
                        ++my_sel;
                        if (p.bits)
                            atomicOr(p.bits + ((size_t)slot * G + g) * p.bits_words + (kk >> 5), 1u << (kk & 31));
                    }
                    if (sel || (in_buf && !p.strict)) {
                        s = sc;
                        ++my_att;
                    }
                }
                wsc[pi] = s;
            }
            __syncwarp();
            float sv[G], mx[G];
            bool att = false;
#pragma unroll
            for (int h = 0; h < G; ++h) {
                sv[h] = lane < 16 ? wsc[lane * G + h] : -INFINITY;
                att |= sv[h] != -INFINITY;
                mx[h] = sv[h] == -INFINITY ? -INFINITY : p.scale * sv[h];
            }
            const unsigned amask = __ballot_sync(0xffffffffu, att) & 0xffffu;
            const long long cyc2 = clock64();
            cy_cls += cyc2 - cyc1;
            if (lane == 0) t_keys += (k0 + 16 <= n) ? 16 : (n > k0 ? n - k0 : 0);
            __syncwarp();
            if (amask == 0) return;
            if (lane == 0) t_vals += __popc(amask);
            // first batch of V rows of the attended keys, issued before the softmax math
            constexpr int VB = 8;
            uint4 vv[VB];
            unsigned mload = amask;
            auto load_v = [&]() {
#pragma unroll
                for (int i = 0; i < VB; ++i) {
                    if (mload) {
                        const int rw = __ffs(mload) - 1;
                        mload &= mload - 1;
                        vv[i] = ldg_v<VPL>(reinterpret_cast<const unsigned char*>(Vs + (size_t)(k0 + rw) * DP) +
                                           lane * VPL * 2);
                    }
                }
            };
            load_v();
#pragma unroll
            for (int of = 16; of > 0; of >>= 1)
#pragma unroll
                for (int h = 0; h < G; ++h) mx[h] = fmaxf(mx[h], __shfl_xor_sync(0xffffffffu, mx[h], of));
            float pl[G], ls[G];
#pragma unroll
            for (int h = 0; h < G; ++h) {
                const float mnew = fmaxf(mrun[h], mx[h]);
                const float alpha = mrun[h] == -INFINITY ? 0.0f : __expf(mrun[h] - mnew);
                mrun[h] = mnew;
                lsum[h] *= alpha;
#pragma unroll
                for (int e = 0; e < VPL; ++e) o[h][e] *= alpha;
                pl[h] = sv[h] == -INFINITY ? 0.0f : __expf(p.scale * sv[h] - mnew);
                ls[h] = pl[h];
            }
#pragma unroll
            for (int of = 16; of > 0; of >>= 1)
#pragma unroll
                for (int h = 0; h < G; ++h) ls[h] += __shfl_xor_sync(0xffffffffu, ls[h], of);
#pragma unroll
            for (int h = 0; h < G; ++h) lsum[h] += ls[h];
            unsigned m = amask;
            while (m) {
                if (m != amask) load_v();  // second batch (more than VB attended rows)
#pragma unroll
                for (int i = 0; i < VB; ++i) {
                    if (m) {
                        const int rw = __ffs(m) - 1;
                        m &= m - 1;
                        float vf[8];
                        const unsigned vw[4] = {vv[i].x, vv[i].y, vv[i].z, vv[i].w};
#pragma unroll
                        for (int e = 0; e < VPL; ++e) vf[e] = (e & 1) ? lvk::bf_hi(vw[e >> 1]) : lvk::bf_lo(vw[e >> 1]);
#pragma unroll
                        for (int h = 0; h < G; ++h) {
                            const float pw = __shfl_sync(0xffffffffu, pl[h], rw);
#pragma unroll
                            for (int e = 0; e < VPL; ++e) o[h][e] = fmaf(pw, vf[e], o[h][e]);
                        }
                    }
                }
            }
            cy_att += clock64() - cyc2;
        };
        LV7_TRACE(4)
        // ping-pong: the next task's key block is in flight while the current one is processed
        int t = warp;
        if (t < ntask) load(t, ua0, ua1);
        while (t < ntask) {
            int tn = t + kW;
            if (tn < ntask) load(tn, ub0, ub1);
            process(t, ua0, ua1);
            t = tn;
            if (t >= ntask) break;
            tn = t + kW;
            if (tn < ntask) load(tn, ua0, ua1);
            process(t, ub0, ub1);
            t = tn;
        }
        __syncthreads();  // clist is rewritten by the next segment
    }

    if (trace && lane == 0) {
        atomicMax(reinterpret_cast<unsigned long long*>(trace + 5), (unsigned long long)lvk2::gtimer());
        atomicAdd(reinterpret_cast<unsigned long long*>(trace + 8), (unsigned long long)cy_mma);
        atomicAdd(reinterpret_cast<unsigned long long*>(trace + 9), (unsigned long long)cy_cls);
        atomicAdd(reinterpret_cast<unsigned long long*>(trace + 10), (unsigned long long)cy_att);
        atomicAdd(reinterpret_cast<unsigned long long*>(trace + 12), (unsigned long long)n_task);
        atomicAdd(reinterpret_cast<unsigned long long*>(trace + 13), (unsigned long long)t_vals);
    }
    if (trace) {
        const int u = __reduce_add_sync(0xffffffffu, (unsigned)n_und);
        if (lane == 0) atomicAdd(reinterpret_cast<unsigned long long*>(trace + 11), (unsigned long long)u);
    }
    // ---- statistics: lanes with the same g = lane % G hold that head's counts
    if (p.counts) {
        int s0 = my_sel, s1 = my_att;
#pragma unroll
        for (int of = 16; of >= G; of >>= 1) {
            s0 += __shfl_xor_sync(0xffffffffu, s0, of);
            s1 += __shfl_xor_sync(0xffffffffu, s1, of);
        }
        if (lane < G) {
            int* c = p.counts + ((size_t)slot * G + lane) * 4;
            if (s0) atomicAdd(c + 0, s0);
            if (s1) atomicAdd(c + 1, s1);
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
    float* shw = reinterpret_cast<float*>(smem + Ge::OFF_CL);  // the cell list is no longer needed
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

    LV7_TRACE(6)
    // ---- two-level merge
    __threadfence();
    __syncthreads();
    int* flag = iscr + 12;
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
    LV7_TRACE(7)
#undef LV7_TRACE
}

cudaError_t launch_query_v7(int DP, int G, const V5Params& vp, int slots, cudaStream_t st);

}  // namespace lvk7
