// Louver bf16 query path, exact + attend stage (K2) as a pipelined cell stream (sm_100a).
//
// The probe (K1, louver_probe_v5) leaves one survivor bit per cell. Every
// surviving cell is r contiguous keys = r/16 tasks of 16 rows (a 4 KB block of
// bf16 keys at d=128). The surviving cells of a slot are split evenly over its
// CTAs and the tasks go round-robin over the warps. Per warp the stream is a
// three-deep software pipeline:
//
//   task t+1   key block in flight: cp.async into the warp's 2-stage smem ring
//              (swizzled so the A-fragment LDS.128 of two rows hit disjoint banks);
//   task t     scored on the tensor cores (q split into three bf16 parts, fp32
//              accumulate), classified against tau +- 2^-13 S_g, pairs inside the
//              margin settled with the normative sequential fp32 dot (core.hpp:17-21)
//              read from the staged block, softmax statistics updated and the V rows of
//              the attended keys (selected ∪ buffer, cache.cpp:48-68) issued;
//   task t-1   its V rows, loaded while task t was scored, folded into the output.
//
// No register holds an in-flight key block and no V latency sits between two
// tasks, so a warp is ready for the next block as soon as it lands. Warps, then
// CTAs (two-level ticket tree, merge5), combine their (m, l, o) partials.
#pragma once

#include "louver_v5.cuh"

namespace lvk8 {

using lvk::QueryParams;
using namespace lvk5;

__device__ __forceinline__ void cpa16(unsigned dst, const void* src) {
    asm volatile("cp.async.cg.shared.global [%0], [%1], 16;\n" ::"r"(dst), "l"(src) : "memory");
}
__device__ __forceinline__ void cpa_commit() { asm volatile("cp.async.commit_group;\n" ::: "memory"); }
__device__ __forceinline__ void cpa_wait1() { asm volatile("cp.async.wait_group 1;\n" ::: "memory"); }
__device__ __forceinline__ uint4 lds16(unsigned a) {
    uint4 r;
    asm volatile("ld.shared.v4.u32 {%0,%1,%2,%3}, [%4];\n" : "=r"(r.x), "=r"(r.y), "=r"(r.z), "=r"(r.w) : "r"(a) : "memory");
    return r;
}

template <int DP, int G>
struct C8 {
    static constexpr int NT = (3 * G + 7) / 8;          // n-tiles of the [q0|q1|q2] split
    static constexpr int KS = DP / 16;                  // k-steps
    static constexpr int NP = DP / 32;                  // k-pairs
    static constexpr int CPR = DP / 8;                  // 16-byte chunks per key row
    static constexpr int RB = DP * 2;                   // bytes per key row
    static constexpr int STAGE = 16 * RB;               // one task's key block
    static constexpr int PPL = G >= 2 ? G / 2 : 1;      // (row, head) pairs per lane
    static constexpr int VPL = DP / 32;                 // V elements per lane
    static constexpr int VB = DP <= 128 ? 16 : 8;       // deferred V rows held in registers
    static constexpr int CL = 1024;                     // surviving cells per list segment
    static constexpr int CW = 8 * NT;                   // C tile row pitch (floats)
    static constexpr int OFF_FR = 0;                                  // [KS][NT][32] uint2
    static constexpr int OFF_Q = OFF_FR + KS * NT * 32 * 8;           // [G][DP+4]
    static constexpr int OFF_M = OFF_Q + G * (DP + 4) * 4;            // misc
    static constexpr int MISC = 4 * G + kW * G + 16;
    static constexpr int OFF_CL = (OFF_M + MISC * 4 + 15) / 16 * 16;  // [CL] cell ids
    static constexpr int OFF_WS = (OFF_CL + CL * 4 + 127) / 128 * 128;
    static constexpr int WCT = 16 * CW * 4;                           // C tile bytes
    static constexpr int WSZ = 2 * STAGE + WCT;                       // key ring, C tile
    static constexpr int SZ_WS = kW * WSZ;
    static constexpr int SZ_RED = kW * G * (DP + 2) * 4;
    static constexpr int FIXED = OFF_WS + (SZ_WS > SZ_RED ? SZ_WS : SZ_RED);
    static int smem(int tiles) { return FIXED + tiles * 8; }          // masks + prefix
};

template <int DP, int G>
__global__ void __launch_bounds__(kT, 2) louver_cells_v8(const __grid_constant__ V5Params vp) {
    using Ge = C8<DP, G>;
    constexpr int NT = Ge::NT, NP = Ge::NP, CPR = Ge::CPR, RB = Ge::RB, PPL = Ge::PPL, VPL = Ge::VPL,
                  VB = Ge::VB, CW = Ge::CW;
    const QueryParams& p = vp.p;
    extern __shared__ __align__(128) unsigned char smem[];
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
    unsigned char* wbase = smem + Ge::OFF_WS + warp * Ge::WSZ;
    const unsigned ring = lvk2::smem_u32(wbase);
    float* ct = reinterpret_cast<float*>(wbase + 2 * Ge::STAGE);
    const int q4 = lane & 3;
    const __nv_bfloat16* Ks = reinterpret_cast<const __nv_bfloat16*>(p.K) + (size_t)slot * p.cap * DP;
    const __nv_bfloat16* Vs = reinterpret_cast<const __nv_bfloat16*>(p.V) + (size_t)slot * p.cap * DP;

    long long* trace = p.tot_trace ? p.tot_trace + ((size_t)slot * vp.nb + blk) * 16 : nullptr;
#define LV8_TRACE(i) \
    if (trace && tid == 0) trace[i] = lvk2::gtimer();
    LV8_TRACE(0)
    // ---- setup independent of the probe (overlaps it under programmatic launch)
    setup_q<DP, G>(p.q + (size_t)slot * G * DP, p.colmax + (size_t)slot * DP, qf, red, S);
    if (tid < G) {
        tau_s[tid] = p.tau[(size_t)slot * G + tid];
        marg[tid] = __fmul_ru(S[tid], 1.220703125e-4f);  // 2^-13 S
    }
    for (int i = tid; i < Ge::KS * NT * 32; i += kT) {
        const int l = i & 31, nt = (i >> 5) % NT, t = (i >> 5) / NT;
        fr[i] = b_frag<G, 3>(t, nt, l, [&](int k, int g) { return qf[g * (DP + 4) + k]; });
    }
    LV8_TRACE(1)
    asm volatile("griddepcontrol.wait;\n" ::: "memory");  // survivor masks visible
    LV8_TRACE(2)

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
                v[k] = u < ntile ? (unsigned)__ldcg(cm + u) : 0u;
            }
#pragma unroll
            for (int k = 0; k < 4; ++k) {
                const int u = u0 + k * kT + tid;
                if (u < ntile) ucm[u] = v[k];
            }
        }
    }
    __syncthreads();
    {  // exclusive prefix of surviving cells per tile
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
    LV8_TRACE(3)
    const long long cs_total = iscr[8];
    const long long c_lo = cs_total * blk / vp.nb, c_hi = cs_total * (blk + 1) / vp.nb;

    // per-lane state: this lane's pairs are (row, g) with g = lane % G
    const int g_me = lane % G;
    const float tau_me = tau_s[g_me], marg_me = marg[g_me];
    const float* q_me = qf + g_me * (DP + 4);
    const float scale = p.scale;
    float o[G][VPL];
#pragma unroll
    for (int g = 0; g < G; ++g)
#pragma unroll
        for (int e = 0; e < VPL; ++e) o[g][e] = 0.0f;
    float mrun = -INFINITY, lpart = 0.0f;  // head g_me: running max (warp-uniform per g), partial sum
    int my_sel = 0, my_att = 0;
    unsigned long long t_keys = 0, t_vals = 0;

    // deferred V of the previous task
    unsigned pmask = 0;
    long long pk0 = 0;
    float pp[PPL];
    uint4 vv[VB];
#pragma unroll
    for (int j = 0; j < PPL; ++j) pp[j] = 0.0f;

    // fold rows of `mask` (V in vv for the first VB, the rest loaded here) into o
    auto consume = [&]() {
        unsigned m = pmask;
        int i = 0;
        while (m) {
            if (i == VB) {  // overflow rows (DP=256 only): load the next batch now
                unsigned mm = m;
#pragma unroll
                for (int b = 0; b < VB; ++b)
                    if (mm) {
                        const int rw = __ffs(mm) - 1;
                        mm &= mm - 1;
                        vv[b] = ldg_v<VPL>(reinterpret_cast<const unsigned char*>(Vs + (size_t)(pk0 + rw) * DP) +
                                           lane * VPL * 2);
                    }
                i = 0;
            }
#pragma unroll
            for (int b = 0; b < VB; ++b) {
                if (b == i && m) {
                    const int rw = __ffs(m) - 1;
                    m &= m - 1;
                    const int pi0 = rw * G;
                    const int j = pi0 >> 5;
                    float pv = pp[0];
#pragma unroll
                    for (int jj = 1; jj < PPL; ++jj)
                        if (j == jj) pv = pp[jj];
                    float vf[VPL];
                    const unsigned vw[4] = {vv[b].x, vv[b].y, vv[b].z, vv[b].w};
#pragma unroll
                    for (int e = 0; e < VPL; ++e) vf[e] = (e & 1) ? lvk::bf_hi(vw[e >> 1]) : lvk::bf_lo(vw[e >> 1]);
#pragma unroll
                    for (int h = 0; h < G; ++h) {
                        const float pw = __shfl_sync(0xffffffffu, pv, (pi0 & 31) + h);
#pragma unroll
                        for (int e = 0; e < VPL; ++e) o[h][e] = fmaf(pw, vf[e], o[h][e]);
                    }
                    ++i;
                }
            }
        }
        pmask = 0;
    };

    for (long long seg = c_lo; seg < c_hi; seg += Ge::CL) {
        const int ncell = (int)(c_hi - seg < Ge::CL ? c_hi - seg : Ge::CL);
        for (int i = tid; i < ncell; i += kT) {  // surviving cell ids of the segment
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
        // rows past n are read (inside the arena) and ignored
        auto key0 = [&](int t) -> long long { return ((long long)clist[t / tpc] << rl) + (long long)(t % tpc) * 16; };
        auto issue = [&](int t, int stage) {
            const unsigned char* src = reinterpret_cast<const unsigned char*>(Ks + (size_t)key0(t) * DP);
            const unsigned dst = ring + stage * Ge::STAGE;
#pragma unroll
            for (int k = 0; k < CPR / 2; ++k) {  // 16 rows x CPR chunks = 32 x (CPR/2)
                const int ch = k * 32 + lane, row = ch / CPR, c = ch % CPR;
                cpa16(dst + row * RB + ((c ^ ((row & 1) << 2)) << 4), src + row * RB + c * 16);
            }
        };
        LV8_TRACE(4)
        int t = warp, st = 0;
        if (t < ntask) issue(t, 0);
        cpa_commit();
        for (; t < ntask; t += kW, st ^= 1) {
            const long long k0 = key0(t);
            if (t + kW < ntask) issue(t + kW, st ^ 1);
            cpa_commit();
            cpa_wait1();
            __syncwarp();
            // ---- scores of 16 keys x (3 parts x G heads) on the tensor cores
            const unsigned sb = ring + st * Ge::STAGE;
            float acc[NT][4];
#pragma unroll
            for (int nt = 0; nt < NT; ++nt) acc[nt][0] = acc[nt][1] = acc[nt][2] = acc[nt][3] = 0.0f;
            {
                const int rw = lane >> 2;
                const unsigned r0 = sb + rw * RB, r1 = r0 + 8 * RB;
                const int sw = (rw & 1) << 2;  // row rw and rw + 8 share the parity
#pragma unroll
                for (int pp2 = 0; pp2 < NP; ++pp2) {
                    const int c = ((4 * pp2 + q4) ^ sw) << 4;
                    const uint4 u0 = lds16(r0 + c), u1 = lds16(r1 + c);
                    const unsigned a0[4] = {u0.x, u1.x, u0.y, u1.y};
                    const unsigned a1[4] = {u0.z, u1.z, u0.w, u1.w};
#pragma unroll
                    for (int nt = 0; nt < NT; ++nt) {
                        const uint2 b0 = fr[((2 * pp2) * NT + nt) * 32 + lane];
                        const uint2 b1 = fr[((2 * pp2 + 1) * NT + nt) * 32 + lane];
                        mma16816(acc[nt], a0, b0.x, b0.y);
                        mma16816(acc[nt], a1, b1.x, b1.y);
                    }
                }
            }
#pragma unroll
            for (int nt = 0; nt < NT; ++nt) {
                const int rw = lane >> 2, col = nt * 8 + 2 * q4;
                *reinterpret_cast<float2*>(ct + rw * CW + col) = make_float2(acc[nt][0], acc[nt][1]);
                *reinterpret_cast<float2*>(ct + (rw + 8) * CW + col) = make_float2(acc[nt][2], acc[nt][3]);
            }
            __syncwarp();
            // ---- classify this lane's pairs (row = pi / G, head g_me)
            float s[PPL];
            unsigned und = 0, attb = 0;
#pragma unroll
            for (int j = 0; j < PPL; ++j) {
                const int pi = lane + 32 * j, rw = pi / G;
                const long long kk = k0 + rw;
                const float* c = ct + rw * CW;
                const float sc = (c[g_me] + c[G + g_me]) + c[2 * G + g_me];
                const bool valid = (G > 1 || lane < 16) && kk < n;
                const bool sel = valid && sc >= tau_me + marg_me;
                const bool u = valid && !sel && sc >= tau_me - marg_me;
                s[j] = sc;
                und |= (unsigned)u << j;
                attb |= (unsigned)sel << j;
            }
            if (__any_sync(0xffffffffu, und != 0)) {  // rare: settle with the normative dot
#pragma unroll
                for (int j = 0; j < PPL; ++j) {
                    if ((und >> j) & 1) {
                        const int rw = (lane + 32 * j) / G;
                        const unsigned rb = sb + rw * RB;
                        const int sw = (rw & 1) << 2;
                        float a2 = 0.0f;
#pragma unroll 1
                        for (int cc = 0; cc < CPR; ++cc) {
                            const uint4 kv = lds16(rb + ((cc ^ sw) << 4));
                            float kf[8];
                            lvk::unpack16<__nv_bfloat16>(kv, kf);
#pragma unroll
                            for (int e2 = 0; e2 < 8; ++e2) a2 = __fadd_rn(a2, __fmul_rn(q_me[cc * 8 + e2], kf[e2]));
                        }
                        s[j] = a2;
                        if (a2 >= tau_me) attb |= 1u << j;
                    }
                }
            }
            // selected pairs are reported; the buffer is attended unless strict
            unsigned amask = 0;  // rows with any attended head
#pragma unroll
            for (int j = 0; j < PPL; ++j) {
                const int pi = lane + 32 * j, rw = pi / G;
                const long long kk = k0 + rw;
                const bool valid = (G > 1 || lane < 16) && kk < n;
                const bool sel = (attb >> j) & 1;
                if (sel) {
                    ++my_sel;
                    if (p.bits)
                        atomicOr(p.bits + ((size_t)slot * G + g_me) * p.bits_words + (kk >> 5), 1u << (kk & 31));
                }
                const bool att = sel || (valid && !p.strict && kk >= indexed);
                my_att += att;
                s[j] = att ? scale * s[j] : -INFINITY;
                const unsigned b = __ballot_sync(0xffffffffu, att);
#pragma unroll
                for (int k = 0; k < 32 / G && k < 16; ++k)
                    if ((b >> (k * G)) & ((1u << G) - 1u)) amask |= 1u << (j * (32 / G) + k);
            }
            if (lane == 0) t_keys += (k0 + 16 <= n) ? 16 : (n > k0 ? n - k0 : 0);
            // ---- fold the previous task's V (loaded while this task was scored)
            if (pmask) consume();
            if (amask) {
                if (lane == 0) t_vals += __popc(amask);
                // online softmax over this lane's head: max over lanes with the same g
                float mloc = s[0];
#pragma unroll
                for (int j = 1; j < PPL; ++j) mloc = fmaxf(mloc, s[j]);
#pragma unroll
                for (int of = 16; of >= G; of >>= 1) mloc = fmaxf(mloc, __shfl_xor_sync(0xffffffffu, mloc, of));
                const float mnew = fmaxf(mrun, mloc);
                const float alpha = mrun == -INFINITY ? 0.0f : __expf(mrun - mnew);
                mrun = mnew;
                float lp = lpart * alpha;
#pragma unroll
                for (int j = 0; j < PPL; ++j) {
                    pp[j] = s[j] == -INFINITY ? 0.0f : __expf(s[j] - mnew);
                    lp += pp[j];
                }
                lpart = lp;
#pragma unroll
                for (int h = 0; h < G; ++h) {
                    const float ah = __shfl_sync(0xffffffffu, alpha, h);
#pragma unroll
                    for (int e = 0; e < VPL; ++e) o[h][e] *= ah;
                }
                // issue this task's V rows; folded after the next task is scored
                unsigned mm = amask;
#pragma unroll
                for (int b = 0; b < VB; ++b)
                    if (mm) {
                        const int rw = __ffs(mm) - 1;
                        mm &= mm - 1;
                        vv[b] = ldg_v<VPL>(reinterpret_cast<const unsigned char*>(Vs + (size_t)(k0 + rw) * DP) +
                                           lane * VPL * 2);
                    }
                pmask = amask;
                pk0 = k0;
            }
            __syncwarp();  // the stage and the C tile are reused
        }
        if (pmask) consume();
        __syncthreads();  // clist is rewritten by the next segment
    }
    if (trace && lane == 0) atomicMax(reinterpret_cast<unsigned long long*>(trace + 5), (unsigned long long)lvk2::gtimer());

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
#pragma unroll
    for (int of = 16; of >= G; of >>= 1) lpart += __shfl_xor_sync(0xffffffffu, lpart, of);

    // ---- warp partials -> CTA partial
    __syncthreads();
    float* wred = reinterpret_cast<float*>(smem + Ge::OFF_WS);  // [kW][G][DP+2]
#pragma unroll
    for (int g = 0; g < G; ++g) {
        float* w = wred + (warp * G + g) * (DP + 2);
        if (lane == g) {
            w[0] = mrun;
            w[1] = lpart;
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
#pragma unroll
        for (int w = 0; w < kW; ++w) s = fmaf(shw[w * G + g], wred[(w * G + g) * (DP + 2) + 2 + c], s);
        part[g * (DP + 2) + 2 + c] = s;
    }

    LV8_TRACE(6)
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
    LV8_TRACE(8)
    merge5<DP, G>(p.partial_ws + ((size_t)slot * vp.nb + grp * kMG) * Wd, members,
                  vp.gpart + ((size_t)slot * vp.ngroups + grp) * Wd, nullptr, nullptr, nullptr, shw);
    LV8_TRACE(9)
    if (tid == 0) vp.gtickets[slot * vp.ngroups + grp] = 0;
    __threadfence();
    __syncthreads();
    if (tid == 0) *flag = atomicAdd(vp.stickets + slot, 1) == vp.ngroups - 1;
    __syncthreads();
    if (!*flag) return;
    __threadfence();
    LV8_TRACE(10)
    merge5<DP, G>(vp.gpart + (size_t)slot * vp.ngroups * Wd, vp.ngroups, nullptr,
                  p.out ? p.out + (size_t)slot * G * DP : nullptr,
                  p.partial_out ? p.partial_out + (size_t)slot * Wd : nullptr,
                  p.counts ? p.counts + (size_t)slot * G * 4 : nullptr, shw);
    if (tid == 0) vp.stickets[slot] = 0;
    LV8_TRACE(7)
#undef LV8_TRACE
}

cudaError_t launch_query_v8(int DP, int G, const V5Params& vp, int slots, cudaStream_t st);

}  // namespace lvk8
