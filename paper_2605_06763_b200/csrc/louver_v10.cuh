// Louver bf16 query path, v10: one warp-specialised persistent kernel per layer (sm_100a).
//
// Per slot (sequence b, kv head h) a team of nb CTAs (one per SM) shares a
// work queue in global memory. Inside every CTA:
//
//   producer warps (probe, LouverCache::query's filter stage, cache.cpp:30-47)
//       stream 16-cell summary tiles [hi | lo] with TMA (128-byte swizzle,
//       mbarrier completion) into a 3-deep ring, score the cell boxes against
//       [q+ | q-] on the tensor cores (q split in two bf16 parts), and append
//       every surviving cell's 16-key blocks to the slot's queue. A cell
//       survives for head g iff its box bound reaches tau_g - 2^-12 S_g (sound:
//       the split error is far inside the margin), or it holds buffer keys.
//   consumer warps (exact_check query.cpp:22-31 + sparse_attention
//       query.cpp:338-371) claim queue entries with one atomic each, load the
//       16-key block by TMA into a 4-deep ring, score it against [q0|q1|q2]
//       on the tensor cores, settle the pairs within 2^-13 S_g of tau with the
//       normative sequential fp32 dot (core.hpp:17-21), and fold the V rows of
//       the attended keys (selected ∪ buffer unless strict, cache.cpp:48-68)
//       into an online softmax with P.V on the tensor cores. Pipeline per warp:
//       K(j+2) in flight | K(j) scored, V(j) issued | V(j-2) folded.
//   merge: consumer (m, l, o) -> CTA partial -> the last CTA of the team
//       combines the nb partials (log-sum-exp) and resets the team's queue.
//
// Producers never wait on consumers, so the probe of later tiles overlaps the
// exact/attend work of earlier survivors, and every consumer of the team draws
// from the same queue, so the team finishes together whatever the survivors'
// spread over the sequence.
#pragma once

#include <cuda.h>

#include "louver_v2.cuh"

namespace lvk10 {

using lvk::Counters;
using lvk::QueryParams;
using lvk2::bf_bits;
using lvk2::bf_val;
using lvk2::mma16816;
using lvk2::smem_u32;

struct V10Params {
    CUtensorMap kmap;  // K arena [slots * cap][DP] bf16, box (64, 16), 128-byte swizzle
    CUtensorMap smap;  // summaries [slots * cap_cells][2 DP] bf16, box (64, 16), 128-byte swizzle
    QueryParams p;
    unsigned* qent;  // [slots][qcap] queue entries: 16-key block index + 1 (0 = empty)
    int* qctl;       // [slots][4]: reserved, claimed, producer warps done, merge ticket
    int qcap;        // entries per slot (cap / 16)
    int nb;          // team CTAs per slot
    int slots;
    int dbg;  // debug experiments: 1 = consumers skip the queue (probe timing only)
};

// ------------------------------------------------------------------ PTX helpers

__device__ __forceinline__ void tma2d(unsigned dst, const CUtensorMap* map, int x, int y, unsigned bar) {
    asm volatile(
        "cp.async.bulk.tensor.2d.shared::cluster.global.tile.mbarrier::complete_tx::bytes [%0], [%1, {%2, %3}], "
        "[%4];\n" ::"r"(dst),
        "l"(reinterpret_cast<unsigned long long>(map)), "r"(x), "r"(y), "r"(bar)
        : "memory");
}
__device__ __forceinline__ void mbar_init(unsigned bar, unsigned count) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;\n" ::"r"(bar), "r"(count) : "memory");
}
__device__ __forceinline__ void mbar_expect_tx(unsigned bar, unsigned bytes) {
    asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;\n" ::"r"(bar), "r"(bytes) : "memory");
}
__device__ __forceinline__ void mbar_wait(unsigned bar, unsigned parity) {
    asm volatile(
        "{\n"
        ".reg .pred p;\n"
        "WAIT_%=:\n"
        "mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n"
        "@!p bra WAIT_%=;\n"
        "}\n" ::"r"(bar),
        "r"(parity)
        : "memory");
}
__device__ __forceinline__ void cpa_arrive(unsigned bar) {  // arrives once this thread's cp.asyncs land
    asm volatile("cp.async.mbarrier.arrive.noinc.shared::cta.b64 [%0];\n" ::"r"(bar) : "memory");
}
__device__ __forceinline__ void cpa16(unsigned dst, const void* src) {
    asm volatile("cp.async.cg.shared.global [%0], [%1], 16;\n" ::"r"(dst), "l"(src) : "memory");
}
__device__ __forceinline__ void fence_async() { asm volatile("fence.proxy.async.shared::cta;\n" ::: "memory"); }
__device__ __forceinline__ void ldsm4(unsigned (&r)[4], unsigned a) {
    asm volatile("ldmatrix.sync.aligned.m8n8.x4.shared.b16 {%0,%1,%2,%3}, [%4];\n"
                 : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3])
                 : "r"(a)
                 : "memory");
}
__device__ __forceinline__ void ldsm4t(unsigned (&r)[4], unsigned a) {
    asm volatile("ldmatrix.sync.aligned.m8n8.x4.trans.shared.b16 {%0,%1,%2,%3}, [%4];\n"
                 : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3])
                 : "r"(a)
                 : "memory");
}
__device__ __forceinline__ uint4 lds16(unsigned a) {
    uint4 r;
    asm volatile("ld.shared.v4.u32 {%0,%1,%2,%3}, [%4];\n"
                 : "=r"(r.x), "=r"(r.y), "=r"(r.z), "=r"(r.w)
                 : "r"(a)
                 : "memory");
    return r;
}
__device__ __forceinline__ int ld_acquire(const int* p) {
    int v;
    asm volatile("ld.acquire.gpu.global.b32 %0, [%1];\n" : "=r"(v) : "l"(p) : "memory");
    return v;
}
__device__ __forceinline__ unsigned ld_relaxed(const unsigned* p) {
    unsigned v;
    asm volatile("ld.relaxed.gpu.global.b32 %0, [%1];\n" : "=r"(v) : "l"(p) : "memory");
    return v;
}
__device__ __forceinline__ int ld_relaxed_i(const int* p) {
    int v;
    asm volatile("ld.relaxed.gpu.global.b32 %0, [%1];\n" : "=r"(v) : "l"(p) : "memory");
    return v;
}
__device__ __forceinline__ void st_relaxed(unsigned* p, unsigned v) {
    asm volatile("st.relaxed.gpu.global.b32 [%0], %1;\n" ::"l"(p), "r"(v) : "memory");
}
__device__ __forceinline__ int atom_add_acq_rel(int* p, int v) {
    int old;
    asm volatile("atom.acq_rel.gpu.global.add.s32 %0, [%1], %2;\n" : "=r"(old) : "l"(p), "r"(v) : "memory");
    return old;
}
__device__ __forceinline__ void red_release(int* p, int v) {
    asm volatile("red.release.gpu.global.add.s32 [%0], %1;\n" ::"l"(p), "r"(v) : "memory");
}
__device__ __forceinline__ unsigned bf2(float lo, float hi) {
    return (unsigned)bf_bits(lo) | ((unsigned)bf_bits(hi) << 16);
}
// 16-byte chunk c of row `row` in a 16-row block stored as 64-element panels with the
// TMA 128-byte swizzle (panel = 16 rows x 128 B, chunk' = chunk ^ row % 8)
__device__ __forceinline__ unsigned swz(int row, int c) {
    return (unsigned)((c >> 3) * 2048 + row * 128 + (((c & 7) ^ (row & 7)) << 4));
}

// Ballot over pair lanes (lane = k G + g for row k of a 32/G-row block) ->
// bit k set iff any head of row k is set.
template <int G>
__device__ __forceinline__ unsigned row_bits(unsigned b) {
    if constexpr (G == 1) {
        return b & 0xffffu;
    } else if constexpr (G == 2) {
        unsigned x = (b | (b >> 1)) & 0x55555555u;
        x = (x | (x >> 1)) & 0x33333333u;
        x = (x | (x >> 2)) & 0x0f0f0f0fu;
        x = (x | (x >> 4)) & 0x00ff00ffu;
        return (x | (x >> 8)) & 0x0000ffffu;
    } else if constexpr (G == 4) {
        unsigned x = b | (b >> 1);
        x = (x | (x >> 2)) & 0x11111111u;
        x = (x | (x >> 3)) & 0x03030303u;
        x = (x | (x >> 6)) & 0x000f000fu;
        return (x | (x >> 12)) & 0xffu;
    } else {
        unsigned x = b | (b >> 1);
        x |= x >> 2;
        x = (x | (x >> 4)) & 0x01010101u;
        x = (x | (x >> 7)) & 0x00030003u;
        return (x | (x >> 14)) & 0xfu;
    }
}

template <int DP, int G>
struct C10 {
    static constexpr int NPAN = DP / 64;          // 64-element panels per row
    static constexpr int RB = DP * 2;             // bytes per bf16 row
    static constexpr int STAGE = 16 * RB;         // one 16-key block, or one half [hi] / [lo] of a 16-cell tile
    static constexpr int NT = (3 * G + 7) / 8;    // exact: n-tiles of [q0|q1|q2]
    static constexpr int NTP = (2 * G + 7) / 8;   // probe: n-tiles of [p0|p1]
    static constexpr int KS = DP / 16;
    static constexpr int CPR = DP / 8;            // 16-byte chunks per row
    static constexpr int PPL = G >= 2 ? G / 2 : 1;
    static constexpr int MT = DP / 16;            // P.V m-tiles (16 dims each)
    static constexpr int CT = 8 * (NT > NTP ? NT : NTP);  // C tile row pitch (floats)
    static constexpr int CST = 4;                 // ring depth per warp (stages)
    static constexpr int SZ_FRE = KS * NT * 32 * 8;
    static constexpr int SZ_FRP = 2 * KS * NTP * 32 * 8;
    static constexpr int SZ_Q = G * (DP + 4) * 4;
    static constexpr int MISC = 8 * G + 16 * G + 64;  // floats
    static constexpr int SZ_BAR = 16 * CST * 2 * 8;   // mbarriers: kbar, vbar per stage per warp
    static constexpr int SZ_KT = 16 * CST * 8;        // per warp: k0 of the blocks in its ring
    static constexpr int SZ_CT = 16 * CT * 4 + 16 * G * 4;  // per warp: C tile + P
    static constexpr int FIX = SZ_FRE + SZ_FRP + SZ_Q + MISC * 4 + SZ_BAR + SZ_KT + 1024;  // + alignment
    static constexpr int PERW = CST * STAGE + SZ_CT;
    static constexpr int BUDGET = 227 * 1024;
    static constexpr int NW0 = (BUDGET - FIX) / PERW;
    static constexpr int NW = NW0 > 16 ? 16 : NW0;
    static constexpr int NTHR = NW * 32;
    // byte offsets from the 1024-aligned base
    static constexpr int OFF_R = 0;  // rings [NW][CST][STAGE]
    static constexpr int OFF_CT = OFF_R + NW * CST * STAGE;
    static constexpr int OFF_FRE = OFF_CT + NW * SZ_CT;
    static constexpr int OFF_FRP = OFF_FRE + SZ_FRE;
    static constexpr int OFF_Q = OFF_FRP + SZ_FRP;
    static constexpr int OFF_M = OFF_Q + SZ_Q;
    static constexpr int OFF_BAR = (OFF_M + MISC * 4 + 7) / 8 * 8;
    static constexpr int OFF_KT = OFF_BAR + SZ_BAR;
    static constexpr int SMEM = OFF_KT + SZ_KT + 1024;
    static_assert(NW >= 2, "Louver v10: shared memory budget too small");
    static_assert(SMEM <= BUDGET, "Louver v10: shared memory over budget");
};

template <int DP, int G>
__global__ void __launch_bounds__(C10<DP, G>::NTHR, 1) louver_layer_v10(const __grid_constant__ V10Params vp) {
    using Ge = C10<DP, G>;
    constexpr int NW = Ge::NW, NTHR = Ge::NTHR, NT = Ge::NT, NTP = Ge::NTP, KS = Ge::KS, CPR = Ge::CPR,
                  RB = Ge::RB, PPL = Ge::PPL, MT = Ge::MT, CT = Ge::CT, NPAN = Ge::NPAN, CST = Ge::CST,
                  STAGE = Ge::STAGE;
    const QueryParams& p = vp.p;
    extern __shared__ unsigned char smem_raw[];
    const unsigned raw_u = smem_u32(smem_raw);
    const unsigned base_u = (raw_u + 1023u) & ~1023u;
    unsigned char* smem = smem_raw + (base_u - raw_u);
    uint2* fre = reinterpret_cast<uint2*>(smem + Ge::OFF_FRE);
    uint2* frp = reinterpret_cast<uint2*>(smem + Ge::OFF_FRP);
    float* qf = reinterpret_cast<float*>(smem + Ge::OFF_Q);
    float* misc = reinterpret_cast<float*>(smem + Ge::OFF_M);
    float* tau_s = misc;           // [G]
    float* taup_s = misc + G;      // [G] probe threshold tau - 2^-12 S
    float* marg_s = misc + 2 * G;  // [G] 2^-13 S
    float* red = misc + 8 * G;     // [16 G]
    int* iscr = reinterpret_cast<int*>(misc + 24 * G);  // [64]
    const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
    const int blk = blockIdx.x, nb = vp.nb;
    const int q4 = lane & 3;
    const int a_row = (lane & 7) + 8 * ((lane >> 3) & 1), a_hi = lane >> 4;
    const int v_row = (lane & 7) + 8 * (lane >> 4), v_hi = (lane >> 3) & 1;
    // per warp: CST stages, each with a TMA barrier (kbar) and a V cp.async barrier (vbar)
    const unsigned kbar = base_u + Ge::OFF_BAR + (unsigned)(warp * CST) * 8u;
    const unsigned vbar = base_u + Ge::OFF_BAR + (unsigned)((NW + warp) * CST) * 8u;
    const unsigned ring = base_u + Ge::OFF_R + (unsigned)(warp * CST * STAGE);
    float* ct = reinterpret_cast<float*>(smem + Ge::OFF_CT + warp * Ge::SZ_CT);
    float* pbuf = ct + 16 * CT;
    long long* kt = reinterpret_cast<long long*>(smem + Ge::OFF_KT) + warp * CST;

    if (lane == 0) {
        for (int s = 0; s < CST; ++s) {
            mbar_init(kbar + 8u * s, 1);
            mbar_init(vbar + 8u * s, 32);
        }
        asm volatile("fence.mbarrier_init.release.cluster;\n" ::: "memory");
    }
    // programmatic dependent launch: dispatched early, nothing is read before the
    // preceding kernel in the stream has completed and flushed
    asm volatile("griddepcontrol.wait;\n" ::: "memory");
    asm volatile("griddepcontrol.launch_dependents;\n" ::: "memory");
    __syncthreads();

    long long* trace = nullptr;
    unsigned sq = 0;    // running stage counter of this warp (stage = sq % CST)
    unsigned kpar = 0;  // per-stage phase parity of kbar / vbar
    unsigned vpar = 0;
    auto kwait = [&](unsigned st) {
        mbar_wait(kbar + 8u * st, (kpar >> st) & 1u);
        kpar ^= 1u << st;
    };
    auto vwait = [&](unsigned st) {
        mbar_wait(vbar + 8u * st, (vpar >> st) & 1u);
        vpar ^= 1u << st;
    };
    for (int slot = blockIdx.y; slot < vp.slots; slot += gridDim.y) {
        trace = p.tot_trace ? p.tot_trace + ((size_t)slot * nb + blk) * 64 : nullptr;
        if (trace && tid == 0) trace[0] = lvk2::gtimer();
        int* ctl = vp.qctl + (size_t)slot * 4;
        unsigned* qe = vp.qent + (size_t)slot * vp.qcap;
        const long long cap_cells = p.cap_cells;
        const int wg = blk * NW + warp;  // this warp's index in the team
        const int tw = nb * NW;          // warps per team
        const long long tiles_cap = cap_cells >> 4;
        // probe sub-block v of this warp = half (v & 1) ([hi] or [lo]) of tile wg + (v >> 1) tw
        auto p_issue = [&](unsigned seq, long long tile, int h) {  // lane 0
            const unsigned st = seq % CST, bar = kbar + 8u * st, dst = ring + st * STAGE;
            fence_async();
            mbar_expect_tx(bar, STAGE);
            const int y = (int)((long long)slot * cap_cells + tile * 16);
#pragma unroll
            for (int pan = 0; pan < NPAN; ++pan) tma2d(dst + pan * 2048, &vp.smap, (h * NPAN + pan) * 64, y, bar);
        };
        const unsigned sq0 = sq;
        int piss = 0;  // sub-blocks issued for this slot
        int cl[8];  // lane 0: queue claims of tasks 0..5 (ring slots, see the consumer loop)
        // ---- setup: q, S_g, thresholds, B fragments
        const long long n = __ldcg(&p.ctr->n);
        const long long indexed = __ldcg(&p.ctr->indexed);
        {
            const float* qsrc = p.q + (size_t)slot * G * DP;
            const float* colmax = p.colmax + (size_t)slot * DP;
            constexpr int QPT = (G * DP + NTHR - 1) / NTHR;
            float xq[QPT], xc[QPT];
#pragma unroll
            for (int k = 0; k < QPT; ++k) {
                const int i = tid + k * NTHR;
                xq[k] = i < G * DP ? __ldcg(qsrc + i) : 0.0f;
                xc[k] = i < G * DP ? __ldcg(colmax + i % DP) : 0.0f;
            }
            const float tau_r = tid < G ? __ldcg(p.tau + (size_t)slot * G + tid) : 0.0f;
            for (int i = tid; i < (Ge::SZ_FRE + Ge::SZ_FRP) / 16; i += NTHR)
                reinterpret_cast<uint4*>(smem + Ge::OFF_FRE)[i] = make_uint4(0u, 0u, 0u, 0u);
            float s[G];
#pragma unroll
            for (int g = 0; g < G; ++g) s[g] = 0.0f;
#pragma unroll
            for (int k = 0; k < QPT; ++k) {
                const int i = tid + k * NTHR;
                if (i < G * DP) {
                    const int g = i / DP, c = i % DP;
                    qf[g * (DP + 4) + c] = xq[k];
                    const float t = __fmul_ru(fabsf(xq[k]), xc[k]);
#pragma unroll
                    for (int h = 0; h < G; ++h)
                        if (h == g) s[h] = __fadd_ru(s[h], t);
                }
            }
            if (trace && tid == 0) trace[9] = lvk2::gtimer();
#pragma unroll
            for (int g = 0; g < G; ++g) {
                float v = s[g];
#pragma unroll
                for (int o = 16; o > 0; o >>= 1) v = __fadd_ru(v, __shfl_xor_sync(0xffffffffu, v, o));
                if (lane == 0) red[warp * G + g] = v;
            }
            __syncthreads();  // also: the fragment arrays are zero
            if (trace && tid == 0) trace[10] = lvk2::gtimer();
            if (tid < G) {
                float v = 0.0f;
                for (int w = 0; w < Ge::NW; ++w) v = __fadd_ru(v, red[w * G + tid]);
                tau_s[tid] = tau_r;
                taup_s[tid] = __fsub_rd(tau_r, __fmul_ru(v, 2.44140625e-4f));  // 2^-12 S
                marg_s[tid] = __fmul_ru(v, 1.220703125e-4f);                   // 2^-13 S
            }
            // each q element scatters its bf16 split parts straight into the B fragments:
            // element k of head g, part P sits in column P G + g; within a k-step of 16,
            // r = k % 16 -> lane quad (r & 7) / 2, half e = (r & 1) | (r >> 3) << 1
            unsigned short* fe = reinterpret_cast<unsigned short*>(fre);
            unsigned short* fp = reinterpret_cast<unsigned short*>(frp);
#pragma unroll
            for (int k = 0; k < QPT; ++k) {
                const int i = tid + k * NTHR;
                if (i < G * DP) {
                    const int g = i / DP, c = i % DP;
                    const int ks = c >> 4, rr = c & 15, e = (rr & 1) | ((rr >> 3) << 1), qq = (rr & 7) >> 1;
                    float y = xq[k];
#pragma unroll
                    for (int P = 0; P < 3; ++P) {
                        const unsigned short b = bf_bits(y);
                        y -= bf_val(b);
                        const int col = P * G + g;
                        fe[((ks * NT + (col >> 3)) * 32 + (col & 7) * 4 + qq) * 4 + e] = b;
                    }
#pragma unroll
                    for (int h = 0; h < 2; ++h) {
                        float z = h == 0 ? fmaxf(xq[k], 0.0f) : fminf(xq[k], 0.0f);  // [hi | lo] . [q+ | q-]
#pragma unroll
                        for (int P = 0; P < 2; ++P) {
                            const unsigned short b = bf_bits(z);
                            z -= bf_val(b);
                            const int col = P * G + g;
                            fp[(((h * KS + ks) * NTP + (col >> 3)) * 32 + (col & 7) * 4 + qq) * 4 + e] = b;
                        }
                    }
                }
            }
            if (tid == 0) iscr[0] = 0;  // tasks processed by this CTA (trace)
            __syncthreads();
        }
        if (trace && tid == 0) trace[1] = lvk2::gtimer();
        // setup is done: now flood the memory system with the first summary sub-blocks
        // (TMA issue stalls the issuing warp while the memory system is saturated, so it
        // must not sit in front of the setup's critical path)
        if (lane == 0) {
            for (int v = 0; v < CST; ++v) {
                const long long tile = wg + (long long)(v >> 1) * tw;
                if (tile >= tiles_cap) break;
                p_issue(sq0 + v, tile, v & 1);
                ++piss;
            }
#pragma unroll
            for (int k = 0; k < 6; ++k) cl[k] = atomicAdd(ctl + 1, 1);
        }
        piss = __shfl_sync(0xffffffffu, piss, 0);
        if (trace && tid == 0) trace[12] = lvk2::gtimer();
        const int rl = p.r_log2;
        const int tpc_l2 = rl - 4;  // log2(16-key blocks per cell)
        const long long ncells = (n + (1 << rl) - 1) >> rl;
        const int total_prod = nb * NW;  // every warp of the team probes, then consumes

        // per-consumer softmax state (also read by the CTA partial below)
        float o[MT][4];
#pragma unroll
        for (int mt = 0; mt < MT; ++mt) o[mt][0] = o[mt][1] = o[mt][2] = o[mt][3] = 0.0f;
        float mrun = -INFINITY, lpart = 0.0f;
        int my_sel = 0, my_att = 0;
        unsigned long long t_keys = 0, t_vals = 0;

        {
            // ================================================================ probe
            float taup[G];
#pragma unroll
            for (int g = 0; g < G; ++g) taup[g] = taup_s[g];
            const long long ntiles = (ncells + 15) >> 4;
            // survivors of the last PD tiles wait for their queue reservation (an atomic
            // whose result is consumed PD tiles later, so its round trip never stalls the probe)
            constexpr int PD = 1;
            unsigned pend_m[PD];
            int pend_t[PD], pend_base[PD];
#pragma unroll
            for (int k = 0; k < PD; ++k) pend_m[k] = 0u, pend_t[k] = 0, pend_base[k] = 0;
            auto write_entries = [&](unsigned pm, int pt, int pbase_l0) {
                if (!pm) return;
                const int base = __shfl_sync(0xffffffffu, pbase_l0, 0);
                if ((pm >> lane) & 1u) {
                    const int idx = __popc(pm & ((1u << lane) - 1u)) << tpc_l2;
                    const unsigned b0 = (unsigned)((((long long)pt * 16 + lane) << tpc_l2) + 1);
                    for (int sb = 0; sb < (1 << tpc_l2); ++sb) st_relaxed(qe + base + idx + sb, b0 + sb);
                }
            };
            float acc2[2][NTP][4];  // two independent chains (k-step parity), over both halves
            int v = 0;
            for (;; ++v) {
                const long long tile = wg + (long long)(v >> 1) * tw;
                const int h = v & 1;
                if (tile >= ntiles) break;
                const unsigned st = (sq0 + v) % CST;
                kwait(st);
                
                const unsigned tb = ring + st * STAGE;
                if (h == 0) {
#pragma unroll
                    for (int c = 0; c < 2; ++c)
#pragma unroll
                        for (int nt = 0; nt < NTP; ++nt) acc2[c][nt][0] = acc2[c][nt][1] = acc2[c][nt][2] = acc2[c][nt][3] = 0.0f;
                }
                // read the sub-block, free the stage for sub-block v + CST, then the mma chain
                unsigned af[KS][4];
#pragma unroll
                for (int ks = 0; ks < KS; ++ks) ldsm4(af[ks], tb + swz(a_row, 2 * ks + a_hi));
                unsigned dep = 0;  // lane 0 waits for its fragments, i.e. the warp's reads of the stage
#pragma unroll
                for (int ks = 0; ks < KS; ++ks) dep ^= af[ks][0] ^ af[ks][3];
                if (lane == 0) asm volatile("" ::"r"(dep));
                __syncwarp();
                {
                    const int v2 = v + CST;
                    const long long t2 = wg + (long long)(v2 >> 1) * tw;
                    if (t2 < ntiles) {
                        if (lane == 0) p_issue(sq0 + v2, t2, v2 & 1);
                        ++piss;
                    }
                }
                const uint2* fh = frp + h * KS * NTP * 32;
#pragma unroll
                for (int ks = 0; ks < KS; ++ks)
#pragma unroll
                    for (int nt = 0; nt < NTP; ++nt) {
                        const uint2 b = fh[(ks * NTP + nt) * 32 + lane];
                        mma16816(acc2[ks & 1][nt], af[ks], b.x, b.y);
                    }
                if (h == 0) continue;
#pragma unroll
                for (int nt = 0; nt < NTP; ++nt) {
                    const int rw = lane >> 2, col = nt * 8 + 2 * q4;
                    *reinterpret_cast<float2*>(ct + rw * CT + col) =
                        make_float2(acc2[0][nt][0] + acc2[1][nt][0], acc2[0][nt][1] + acc2[1][nt][1]);
                    *reinterpret_cast<float2*>(ct + (rw + 8) * CT + col) =
                        make_float2(acc2[0][nt][2] + acc2[1][nt][2], acc2[0][nt][3] + acc2[1][nt][3]);
                }
                __syncwarp();
                unsigned gm = 0;
                int scan = 0;
                const long long cell = tile * 16 + lane;
                if (lane < 16 && cell < ncells) {
                    const long long cs = cell << rl, ce = cs + (1 << rl);
                    if (ce > indexed) {
                        gm = (1u << G) - 1u;  // holds buffer keys: scanned densely
                    } else {
#pragma unroll
                        for (int g = 0; g < G; ++g)
                            if (ct[lane * CT + g] + ct[lane * CT + G + g] >= taup[g]) gm |= 1u << g;
                    }
                    scan = (int)((ce < n ? ce : n) - cs);
                }
                __syncwarp();
                const unsigned m = __ballot_sync(0xffffffffu, gm != 0) & 0xffffu;
                write_entries(pend_m[0], pend_t[0], pend_base[0]);
#pragma unroll
                for (int k = 0; k + 1 < PD; ++k) {
                    pend_m[k] = pend_m[k + 1];
                    pend_t[k] = pend_t[k + 1];
                    pend_base[k] = pend_base[k + 1];
                }
                pend_m[PD - 1] = m;
                pend_t[PD - 1] = (int)tile;
                if (m && lane == 0) pend_base[PD - 1] = atomicAdd(ctl + 0, __popc(m) << tpc_l2);
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
                        const int vv = lvk::warp_sum_int((gm >> g) & 1 ? scan : 0);
                        if (lane == 0 && vv) atomicAdd(p.counts + ((size_t)slot * G + g) * 4 + 2, vv);
                    }
                }
            }
#pragma unroll
            for (int k = 0; k < PD; ++k) write_entries(pend_m[k], pend_t[k], pend_base[k]);
            __syncwarp();
            if (lane == 0) {
                __threadfence();
                red_release(ctl + 2, 1);  // this warp's reservations are all made
            }
            // sub-blocks issued past the end of the sequence (prologue): retire their phases
            for (int k = v; k < piss; ++k) kwait((sq0 + k) % CST);
            sq = sq0 + piss;
            if (trace && tid == 0) trace[2] = lvk2::gtimer();
        }
        {
            // ================================================================ exact + attend
            const int g_me = lane % G;
            const float tau_me = tau_s[g_me], marg_me = marg_s[g_me];
            const float* q_me = qf + g_me * (DP + 4);
            const float scale = p.scale;
            const __nv_bfloat16* Vs = reinterpret_cast<const __nv_bfloat16*>(p.V) + (size_t)slot * p.cap * DP;
            const int qcap = vp.qcap;
            constexpr unsigned EXH = 0xffffffffu;
            // lane 0: block the warp until entry c is published or the queue is exhausted
            auto spin_resolve = [&](int c) -> unsigned {
                for (;;) {
                    if (c >= qcap) return EXH;
                    const unsigned e = ld_relaxed(qe + c);
                    const int pd = ld_acquire(ctl + 2);
                    if (e) return e;
                    if (pd >= total_prod) {
                        const int qr = ld_relaxed_i(ctl + 0);
                        if (c >= qr) return EXH;
                    }
                    __nanosleep(64);
                }
            };
            int nis = 0;  // blocks whose K load was issued (tasks [0, nis))
            bool exh = (vp.dbg & 1) != 0;
            // pending folds: A = task m-2, B = task m-1
            unsigned pbA[4] = {0u, 0u, 0u, 0u}, pbB[4] = {0u, 0u, 0u, 0u};
            bool pendA = false, pendB = false;
            float alphaB = 1.0f;  // alpha of task m-1 (frame m-2 -> m-1)
            int m = 0;
            // task j uses stage j % CST: start the consumer on a ring boundary (skipped stages
            // carry no pending phase, their parity bits are untouched)
            const unsigned sqc = (sq + CST - 1) / CST * CST;
            auto fold = [&](unsigned j, const unsigned (&pb)[4], bool any) {
                const unsigned st = (sqc + j) % CST;
                vwait(st);
                if (!any) return;
                const unsigned vb = ring + st * STAGE;
#pragma unroll
                for (int mt = 0; mt < MT; ++mt) {
                    unsigned a[4];
                    ldsm4t(a, vb + swz(v_row, 2 * mt + v_hi));
                    mma16816(o[mt], a, pb[0], pb[1]);
                    mma16816(o[mt], a, pb[2], pb[3]);
                }
            };
            auto rescale = [&](float alpha) {
                if (__any_sync(0xffffffffu, alpha != 1.0f)) {
                    const float a0 = __shfl_sync(0xffffffffu, alpha, (2 * q4) % G);
                    const float a1 = __shfl_sync(0xffffffffu, alpha, (2 * q4 + 1) % G);
#pragma unroll
                    for (int mt = 0; mt < MT; ++mt) {
                        o[mt][0] *= a0;
                        o[mt][1] *= a1;
                        o[mt][2] *= a0;
                        o[mt][3] *= a1;
                    }
                }
            };
            // Claims run 6 tasks ahead and their entries are read 4 tasks ahead, in rings of 8
            // indexed by compile-time slots (the loop body is unrolled 8 times): a register
            // whose atomic or load is still in flight is never copied, which would stall.
            // lane 0: cl[] holds claimed queue indices, en[] their entries (0 = not published yet)
            unsigned en[8];
            auto ld_entry = [&](int c) { return c < qcap ? ld_relaxed(qe + c) : EXH; };
            if (lane == 0) {
#pragma unroll
                for (int k = 0; k < 4; ++k) en[k] = ld_entry(cl[k]);
            }
            auto issue_k = [&](unsigned e) {  // lane 0: K block of task nis
                const unsigned st = (sqc + nis) % CST;
                const long long k0 = (long long)(e - 1) << 4;
                kt[st] = k0;
                fence_async();  // the stage was last touched by the generic proxy
                mbar_expect_tx(kbar + 8u * st, STAGE);
                const int y = (int)((long long)slot * p.cap + k0);
#pragma unroll
                for (int pan = 0; pan < NPAN; ++pan) tma2d(ring + st * STAGE + pan * 2048, &vp.kmap, pan * 64, y, kbar + 8u * st);
            };
            // task m + OFF (ring slot JS) if it is the next one to issue; blocking when OFF == 0
#define LV10_ISSUE(JS, OFF)                                                                   \
    if (!exh && nis == m + (OFF)) {                                                             \
        unsigned e = 0;                                                                         \
        if (lane == 0) {                                                                        \
            e = cl[JS] >= qcap ? EXH : en[JS];                                                  \
            if (e == 0) {                                                                       \
                if ((OFF) == 0) e = spin_resolve(cl[JS]);                                       \
                else en[JS] = ld_relaxed(qe + cl[JS]); /* not published yet: look again later */ \
            }                                                                                   \
            if (e != 0 && e != EXH) {                                                           \
                issue_k(e);                                                                     \
                st_relaxed(qe + cl[JS], 0u); /* consumed: the queue stays empty between launches */ \
                cl[((JS) + 6) % 8] = atomicAdd(ctl + 1, 1);                                     \
                en[((JS) + 4) % 8] = ld_entry(cl[((JS) + 4) % 8]);                              \
            }                                                                                   \
        }                                                                                       \
        e = __shfl_sync(0xffffffffu, e, 0);                                                     \
        if (e == EXH) exh = true;                                                               \
        else if (e != 0) ++nis;                                                                 \
    }
#define LV10_BODY(J)                                                  \
    {                                                                   \
        if (trace && warp == 0 && lane == 0 && m < 16) trace[16 + m] = lvk2::gtimer(); \
        if (m >= 2) { /* fold V(m-2) (frame m-2), then move o to frame m-1 */ \
            fold(m - 2, pbA, pendA);                                    \
            rescale(alphaB);                                            \
        }                                                               \
        __syncwarp();                                                   \
        LV10_ISSUE((J), 0)                                              \
        LV10_ISSUE(((J) + 1) % 8, 1)                                    \
        LV10_ISSUE(((J) + 2) % 8, 2)                                    \
        if (m >= nis) break; /* exhausted, every issued block processed */ \
        task();                                                         \
        ++m;                                                            \
    }
            auto task = [&]() {
                __syncwarp();
                // -- task m: scores of 16 keys x [q0|q1|q2] per head
                const unsigned st = (sqc + m) % CST;
                const long long k0 = kt[st];
                if (trace && m == 0 && warp == 0 && lane == 0) trace[3] = lvk2::gtimer();
                if (trace && warp == 0 && lane == 0 && m < 16) trace[32 + m] = lvk2::gtimer();
                kwait(st);
                if (trace && warp == 0 && lane == 0 && m < 16) trace[48 + m] = lvk2::gtimer();
                const unsigned sb = ring + st * STAGE;
                {
                    float acc2[2][NT][4];  // two independent chains (k-step parity)
#pragma unroll
                    for (int c = 0; c < 2; ++c)
#pragma unroll
                        for (int nt = 0; nt < NT; ++nt) acc2[c][nt][0] = acc2[c][nt][1] = acc2[c][nt][2] = acc2[c][nt][3] = 0.0f;
#pragma unroll
                    for (int ks = 0; ks < KS; ++ks) {
                        unsigned a[4];
                        ldsm4(a, sb + swz(a_row, 2 * ks + a_hi));
#pragma unroll
                        for (int nt = 0; nt < NT; ++nt) {
                            const uint2 b = fre[(ks * NT + nt) * 32 + lane];
                            mma16816(acc2[ks & 1][nt], a, b.x, b.y);
                        }
                    }
                    float acc[NT][4];
#pragma unroll
                    for (int nt = 0; nt < NT; ++nt)
#pragma unroll
                        for (int e = 0; e < 4; ++e) acc[nt][e] = acc2[0][nt][e] + acc2[1][nt][e];
#pragma unroll
                    for (int nt = 0; nt < NT; ++nt) {
                        const int rw = lane >> 2, col = nt * 8 + 2 * q4;
                        *reinterpret_cast<float2*>(ct + rw * CT + col) = make_float2(acc[nt][0], acc[nt][1]);
                        *reinterpret_cast<float2*>(ct + (rw + 8) * CT + col) = make_float2(acc[nt][2], acc[nt][3]);
                    }
                }
                __syncwarp();
                // -- classify this lane's pairs (row pi / G, head g_me)
                float s[PPL];
                unsigned und = 0, selb = 0;
#pragma unroll
                for (int jj = 0; jj < PPL; ++jj) {
                    const int pi = lane + 32 * jj, rw = pi / G;
                    const float* c = ct + (rw < 16 ? rw : 15) * CT;
                    const float sc = (c[g_me] + c[G + g_me]) + c[2 * G + g_me];
                    const bool valid = (G > 1 || lane < 16) && k0 + rw < n;
                    const bool sel = valid && sc >= tau_me + marg_me;
                    const bool u = valid && !sel && sc >= tau_me - marg_me;
                    s[jj] = sc;
                    und |= (unsigned)u << jj;
                    selb |= (unsigned)sel << jj;
                }
                if (__any_sync(0xffffffffu, und != 0)) {  // rare: the normative sequential dot
#pragma unroll
                    for (int jj = 0; jj < PPL; ++jj) {
                        if ((und >> jj) & 1) {
                            const int rw = (lane + 32 * jj) / G;
                            float a2 = 0.0f;
#pragma unroll 1
                            for (int cc = 0; cc < CPR; ++cc) {
                                const uint4 kv = lds16(sb + swz(rw, cc));
                                float kf[8];
                                lvk::unpack16<__nv_bfloat16>(kv, kf);
#pragma unroll
                                for (int e2 = 0; e2 < 8; ++e2) a2 = __fadd_rn(a2, __fmul_rn(q_me[cc * 8 + e2], kf[e2]));
                            }
                            s[jj] = a2;
                            if (a2 >= tau_me) selb |= 1u << jj;
                        }
                    }
                }
                unsigned amask = 0;  // rows with any attended head
                float mloc = -INFINITY;
#pragma unroll
                for (int jj = 0; jj < PPL; ++jj) {
                    const int pi = lane + 32 * jj, rw = pi / G;
                    const long long kk = k0 + rw;
                    const bool valid = (G > 1 || lane < 16) && kk < n;
                    const bool sel = (selb >> jj) & 1;
                    if (sel) {
                        ++my_sel;
                        if (p.bits)
                            atomicOr(p.bits + ((size_t)slot * G + g_me) * p.bits_words + (kk >> 5), 1u << (kk & 31));
                    }
                    const bool att = sel || (valid && !p.strict && kk >= indexed);
                    my_att += att;
                    s[jj] = att ? scale * s[jj] : -INFINITY;
                    mloc = fmaxf(mloc, s[jj]);
                    amask |= row_bits<G>(__ballot_sync(0xffffffffu, att)) << (jj * (32 / G));
                }
                if (lane == 0) t_keys += (k0 + 16 <= n) ? 16 : (n > k0 ? n - k0 : 0);
                float alpha = 1.0f;
                unsigned nbf[4] = {0u, 0u, 0u, 0u};
                if (amask) {
                    if (lane == 0) t_vals += __popc(amask);
#pragma unroll
                    for (int of = 16; of >= G; of >>= 1) mloc = fmaxf(mloc, __shfl_xor_sync(0xffffffffu, mloc, of));
                    // lazy rescale: the reference max moves only when a score exceeds it by
                    // more than 8 (weights stay <= e^8); o and l are rescaled only then
                    if (mloc > mrun + 8.0f) {
                        alpha = mrun == -INFINITY ? 0.0f : __expf(mrun - mloc);
                        mrun = mloc;
                    }
                    float lp = lpart * alpha;
#pragma unroll
                    for (int jj = 0; jj < PPL; ++jj) {
                        const float pv = s[jj] == -INFINITY ? 0.0f : __expf(s[jj] - mrun);
                        lp += pv;
                        if (G > 1 || lane < 16) pbuf[lane + 32 * jj] = pv;
                    }
                    lpart = lp;
                    __syncwarp();
                    // B fragment of P: k = rows (2q, 2q+1 | 2q+8, 2q+9), n = head lane/4
                    const int hn = lane >> 2;
                    float pv4[4] = {0.0f, 0.0f, 0.0f, 0.0f};
                    if (hn < G) {
                        pv4[0] = pbuf[(2 * q4) * G + hn];
                        pv4[1] = pbuf[(2 * q4 + 1) * G + hn];
                        pv4[2] = pbuf[(2 * q4 + 8) * G + hn];
                        pv4[3] = pbuf[(2 * q4 + 9) * G + hn];
                    }
                    float lo4[4];
#pragma unroll
                    for (int e = 0; e < 4; ++e) lo4[e] = pv4[e] - bf_val(bf_bits(pv4[e]));
                    nbf[0] = bf2(pv4[0], pv4[1]);
                    nbf[1] = bf2(pv4[2], pv4[3]);
                    nbf[2] = bf2(lo4[0], lo4[1]);
                    nbf[3] = bf2(lo4[2], lo4[3]);
                }
                __syncwarp();  // K(m) and pbuf reads done
                // -- V(m): attended rows into K(m)'s stage (same row positions)
                if (amask) {
                    constexpr int RPI = 32 / CPR;  // rows per warp instruction
                    unsigned mm = amask;
                    const int cc = lane % CPR, sub = lane / CPR;
                    const unsigned char* vsrc = reinterpret_cast<const unsigned char*>(Vs + (size_t)k0 * DP) + cc * 16;
                    while (mm) {
                        int rsel = -1;
#pragma unroll
                        for (int k = 0; k < RPI; ++k) {
                            const int rr = mm ? __ffs(mm) - 1 : -1;
                            mm &= mm - 1;
                            if (k == sub) rsel = rr;
                        }
                        if (rsel >= 0) cpa16(sb + swz(rsel, cc), vsrc + rsel * RB);
                    }
                }
                cpa_arrive(vbar + 8u * st);
                // shift the fold pipeline
#pragma unroll
                for (int e = 0; e < 4; ++e) {
                    pbA[e] = pbB[e];
                    pbB[e] = nbf[e];
                }
                pendA = pendB;
                pendB = amask != 0;
                // alpha of task m (frame m-1 -> m) applies once V(m-1) is folded
                alphaB = alpha;
            };
            for (;;) {
                LV10_BODY(0)
                LV10_BODY(1)
                LV10_BODY(2)
                LV10_BODY(3)
                LV10_BODY(4)
                LV10_BODY(5)
                LV10_BODY(6)
                LV10_BODY(7)
            }
#undef LV10_BODY
#undef LV10_ISSUE
            // drain: the exit round already folded V(m-2); V(m-1) remains (m = tasks processed)
            if (m >= 1) fold(m - 1, pbB, pendB);
            sq = sqc + nis;
            if (trace && warp == 0 && lane == 0) trace[4] = lvk2::gtimer();
            if (lane == 0 && trace) atomicAdd(iscr + 0, nis);
        }

        // ---- statistics: lanes with the same g = lane % G hold that head's counts
        {
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
        }

        // ---- consumer partials -> CTA partial [G][DP+2] (m, l, o)
        constexpr int Wd = G * (DP + 2);
        float* wred = reinterpret_cast<float*>(smem + Ge::OFF_R);  // [NW][Wd] over the rings
        float* shw = red;                                          // [NW][G] weights
        __syncthreads();
        if (trace && tid == 0) {
            trace[5] = lvk2::gtimer();
            trace[15] = iscr[0];
        }
        {
            float* w = wred + warp * Wd;
            if (lane < G) {
                w[lane * (DP + 2)] = mrun;
                w[lane * (DP + 2) + 1] = lpart;
            }
#pragma unroll
            for (int mt = 0; mt < MT; ++mt) {
#pragma unroll
                for (int e = 0; e < 4; ++e) {
                    const int h = 2 * q4 + (e & 1), c = 16 * mt + (lane >> 2) + 8 * (e >> 1);
                    if (h < G) w[h * (DP + 2) + 2 + c] = o[mt][e];
                }
            }
        }
        __syncthreads();
        float* part = p.partial_ws + ((size_t)slot * nb + blk) * Wd;
        if (tid < G) {
            float mm = -INFINITY;
            for (int w = 0; w < NW; ++w) mm = fmaxf(mm, wred[w * Wd + tid * (DP + 2)]);
            float l = 0.0f;
            for (int w = 0; w < NW; ++w) {
                const float mw = wred[w * Wd + tid * (DP + 2)];
                const float a = mw == -INFINITY ? 0.0f : __expf(mw - mm);
                shw[w * G + tid] = a;
                l += a * wred[w * Wd + tid * (DP + 2) + 1];
            }
            part[tid * (DP + 2)] = l > 0.0f ? mm : -INFINITY;
            part[tid * (DP + 2) + 1] = l;
        }
        __syncthreads();
        for (int i = tid; i < G * DP; i += NTHR) {
            const int g = i / DP, c = i % DP;
            float s = 0.0f;
#pragma unroll
            for (int w = 0; w < NW; ++w) s = fmaf(shw[w * G + g], wred[w * Wd + g * (DP + 2) + 2 + c], s);
            part[g * (DP + 2) + 2 + c] = s;
        }
        if (trace && tid == 0) trace[6] = lvk2::gtimer();

        // ---- the last CTA of the team merges the nb partials
        int* ticket = ctl + 3;
        __syncthreads();
        if (tid == 0) iscr[1] = atom_add_acq_rel(ticket, 1) == nb - 1;
        __syncthreads();
        if (iscr[1]) {
            if (trace && tid == 0) trace[8] = lvk2::gtimer();
            const float* src = p.partial_ws + (size_t)slot * nb * Wd;
            // scratch over the consumer rings: M[G], L[G], m/weights [nb][G], l [nb][G], then o chunks
            float* M = reinterpret_cast<float*>(smem + Ge::OFF_R);
            float* L = M + G;
            float* wgt = M + 2 * G;
            float* lsv = wgt + nb * G;
            const int hdr = (2 * G + 2 * nb * G + 3) / 4 * 4;
            constexpr int EPT = (G * DP + NTHR - 1) / NTHR;
            float accr[EPT];
#pragma unroll
            for (int k = 0; k < EPT; ++k) accr[k] = 0.0f;
            const int per_chunk = (NW * CST * STAGE - hdr * 4) / (Wd * 4);
            float* stage = M + hdr;
            const unsigned stage_u = smem_u32(stage);
            auto chunk_issue = [&](int s0) {
                const int cnt = nb - s0 < per_chunk ? nb - s0 : per_chunk;
                const float* cs = src + (size_t)s0 * Wd;
                for (int i = tid; i < cnt * Wd / 2; i += NTHR) {
                    const unsigned d = stage_u + i * 8;
                    asm volatile("cp.async.ca.shared.global [%0], [%1], 8;\n" ::"r"(d), "l"(cs + 2 * i) : "memory");
                }
                asm volatile("cp.async.commit_group;\n" ::: "memory");
            };
            chunk_issue(0);  // the first chunk of o rows travels with the headers
            for (int i = tid; i < nb * G; i += NTHR) {
                const float* h = src + (size_t)(i / G) * Wd + (i % G) * (DP + 2);
                wgt[i] = __ldcg(h);
                lsv[i] = __ldcg(h + 1);
            }
            __syncthreads();
            if (trace && tid == 0) trace[11] = lvk2::gtimer();
            for (int g = warp; g < G; g += Ge::NW) {  // one warp per head: max, weights, l
                float mm = -INFINITY;
                for (int s2 = lane; s2 < nb; s2 += 32) mm = fmaxf(mm, wgt[s2 * G + g]);
#pragma unroll
                for (int o2 = 16; o2 > 0; o2 >>= 1) mm = fmaxf(mm, __shfl_xor_sync(0xffffffffu, mm, o2));
                float l = 0.0f;
                for (int s2 = lane; s2 < nb; s2 += 32) {
                    const float ms = wgt[s2 * G + g];
                    const float w = ms == -INFINITY ? 0.0f : __expf(ms - mm);
                    wgt[s2 * G + g] = w;
                    l += w * lsv[s2 * G + g];
                }
#pragma unroll
                for (int o2 = 16; o2 > 0; o2 >>= 1) l += __shfl_xor_sync(0xffffffffu, l, o2);
                if (lane == 0) {
                    M[g] = mm;
                    L[g] = l;
                }
            }
            __syncthreads();
            for (int s0 = 0; s0 < nb; s0 += per_chunk) {
                const int cnt = nb - s0 < per_chunk ? nb - s0 : per_chunk;
                if (s0 > 0) chunk_issue(s0);
                asm volatile("cp.async.wait_group 0;\n" ::: "memory");
                __syncthreads();
#pragma unroll
                for (int k = 0; k < EPT; ++k) {
                    const int i = tid + k * NTHR;
                    if (i < G * DP) {
                        const int g = i / DP, c = i % DP;
                        float a = accr[k];
#pragma unroll 8
                        for (int s2 = 0; s2 < cnt; ++s2) a = fmaf(wgt[(s0 + s2) * G + g], stage[s2 * Wd + g * (DP + 2) + 2 + c], a);
                        accr[k] = a;
                    }
                }
                __syncthreads();
            }
#pragma unroll
            for (int k = 0; k < EPT; ++k) {
                const int i = tid + k * NTHR;
                if (i < G * DP) {
                    const int g = i / DP, c = i % DP;
                    const float l = L[g];
                    if (p.out) p.out[((size_t)slot * G + g) * DP + c] = l > 0.0f ? accr[k] / l : 0.0f;
                    if (p.partial_out) p.partial_out[(size_t)slot * Wd + g * (DP + 2) + 2 + c] = accr[k];
                }
            }
            if (tid < G) {
                if (p.partial_out) {
                    p.partial_out[(size_t)slot * Wd + tid * (DP + 2)] = L[tid] > 0.0f ? M[tid] : -INFINITY;
                    p.partial_out[(size_t)slot * Wd + tid * (DP + 2) + 1] = L[tid];
                }
                if (p.counts) p.counts[((size_t)slot * G + tid) * 4 + 3] = L[tid] > 0.0f ? 1 : 0;
            }
            if (tid < 4) ctl[tid] = 0;  // reserved, claimed, producers done, ticket: ready for the next launch
            if (trace && tid == 0) trace[7] = lvk2::gtimer();
        }
        __syncthreads();
    }
}

cudaError_t launch_layer_v10(int DP, int G, const V10Params& vp, int sms, cudaStream_t st, int* geo);
int v10_smem(int DP, int G);

}  // namespace lvk10
