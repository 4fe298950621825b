// Louver bf16 query path as ONE persistent kernel per layer (sm_100a).
//
// Grid = (team, slots): a slot (one sequence x kv head) is served by a team of nb CTAs,
// one CTA per SM, and CTA b of the team owns the slot's cells b, b + nb, b + 2 nb, ...
// (a fine interleave, so every CTA sees the same mix of the sequence and no team-wide
// exchange is needed before the merge). Phases per CTA:
//
//   A  probe      cell summaries [hi | lo] (16 cells = one tile) are scored against
//                 [q+ | q-] on the tensor cores; a cell survives for head g iff its box
//                 bound reaches tau_g - 2^-12 S_g (sound: the bf16 split error is far
//                 inside the margin) or it holds buffer keys. Survivors are appended to
//                 the CTA's list in shared memory (warp ballot compaction).
//                 (reference: gate_bounds + query_ta / query_full_subspace, query.cpp:47-303)
//   B  exact      16-key tasks of the listed cells, claimed by the CTA's warps through a
//      + attend   shared counter, are scored on the tensor cores (q in three bf16 parts);
//                 pairs within 2^-13 S_g of tau are settled with the normative sequential
//                 fp32 dot (core.hpp:17-21, exact_check query.cpp:22-31); the V rows of the
//                 attended keys (selected ∪ buffer unless strict, cache.cpp:48-68) are folded
//                 in with P.V on the tensor cores (P split in two bf16 parts, V bf16 exact);
//                 online softmax with a lazy reference max (sparse_attention, query.cpp:338-371).
//   C  merge      warp partials -> CTA partial (m, l, o) in global scratch; an acq_rel
//                 ticket elects the team's last CTA, which combines the nb partials.
//
// DENSE = true is the full-scan decode (the speed-up denominator): no probe, every key of
// the CTA's cells is attended; same pipeline, same score precision.
//
// Every block of keys, summaries or values moves global -> shared with cp.async into a
// per-warp 3-stage ring, laid out as the TMA 128-byte swizzle (see lay()), read with ldmatrix, so no
// register holds an in-flight block and the fragments need no register shuffling. Per
// warp the exact phase is a software pipeline:
// K(t+1) in flight | K(t) scored | V(t-1) in flight, folded after K(t) is scored.
// The launch uses programmatic dependent launch: the first summary sub-blocks of sealed
// cells are requested before griddepcontrol.wait.
#pragma once

#include <cuda.h>  // CUtensorMap

#include "louver_common.cuh"
#include "louver_kernels.cuh"

namespace lvk9 {

using lvk::QueryParams;
using namespace lvc;

struct LayerParams {
    QueryParams p;
    const __nv_bfloat16* sum;  // [slot][cap_cells][2*DP] cell rows [hi | lo]
    int* stickets;             // [slots] merge tickets (self-resetting)
    int nb;                    // team CTAs per slot (slots >= nfull: nb - 1)
    int nfull;                 // slots with teams of nb CTAs (148 SMs over 8 slots: 4 of 19, 4 of 18)
    int slots;                 // slots of the layer (the grid may loop over them)
    unsigned short* glist;     // survivor lists in global scratch when they outgrow smem (else null)
    int list_cap;              // entries per CTA list
    long long sealed;          // cells complete when the query was enqueued (immutable summaries)
    int npre;                  // summary sub-blocks requested before griddepcontrol.wait (0..3)
    int ktma;                  // key blocks by TMA (kmap) instead of cp.async
    int kpf;                   // the CTA's first kpf listed cells: key blocks L2-prefetched by the probe
    int vtail;                 // the CTA's last vtail tasks: value blocks L2-prefetched when claimed
    int spread;                // grid (slots, team): the CTAs dispatched last are one member of each slot
    alignas(64) CUtensorMap kmap;  // K arena as [slots * cap][DP] bf16, box 64 x 16, 128-byte swizzle
};

// one 2D TMA tile (box of the tensor map) into shared memory, completing on an mbarrier
__device__ __forceinline__ void tma_load_2d(unsigned dst, const CUtensorMap* map, int x, int y, unsigned bar) {
    asm volatile(
        "cp.async.bulk.tensor.2d.shared::cluster.global.tile.mbarrier::complete_tx::bytes [%0], [%1, {%2, %3}], [%4];\n" ::"r"(dst),
        "l"(reinterpret_cast<unsigned long long>(map)), "r"(x), "r"(y), "r"(bar)
        : "memory");
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

// Stage layout (the TMA SWIZZLE_128B image of a 16-row block): 128-byte column halves of
// 16 rows each, half h at h * 2048; 16-byte chunk c of row r at
//   (c >> 3) * 2048 + r * 128 + ((c & 7) ^ ((r + b7) & 7)) * 16,
// b7 = bits 7..9 of the stage's shared address (the hardware swizzle XORs with the
// absolute address bits), so ldmatrix reads of 8 rows at one chunk are conflict-free.
__device__ __forceinline__ unsigned lay(int r, int c, int b7) {
    return ((unsigned)(c >> 3) << 11) + ((unsigned)r << 7) + ((unsigned)((c & 7) ^ ((r + b7) & 7)) << 4);
}
// k-step ks's chunk (2 ks + hi) of a row whose swizzle key is rx = (row + b7) & 7,
// relative to the row start
__device__ __forceinline__ unsigned swz_off(int ks, int a_hi, int rx) {
    return ((unsigned)(ks >> 2) << 11) + ((unsigned)(((2 * (ks & 3) + a_hi) ^ rx)) << 4);
}

template <int DP, int G>
struct C9 {
    static constexpr int NT = (3 * G + 7) / 8;   // exact: n-tiles of [q0|q1|q2]
    static constexpr int NTP = (2 * G + 7) / 8;  // probe: n-tiles of [p0|p1]
    static constexpr int KS = DP / 16;
    static constexpr int CPR = DP / 8;           // 16-byte chunks per row
    static constexpr int RB = DP * 2;            // bytes per bf16 row
    static constexpr int STAGE = 16 * RB;
    static constexpr int PPL = G >= 2 ? G / 2 : 1;
    static constexpr int MT = DP / 16;           // P.V m-tiles (16 dims each)
    static constexpr int CT = 8 * (NT > NTP ? NT : NTP);  // C tile row pitch (floats)
    static constexpr int MINB = 1;               // one CTA per SM: its warps share every task of the SM
    static constexpr int SZ_FRE = KS * NT * 32 * 8;
    static constexpr int SZ_FRP = 2 * KS * NTP * 32 * 8;
    static constexpr int OFF_FRE = 0;
    static constexpr int OFF_FRP = OFF_FRE + SZ_FRE;
    static constexpr int OFF_Q = OFF_FRP + SZ_FRP;                    // [G][DP+4] f32
    static constexpr int OFF_M = OFF_Q + G * (DP + 4) * 4;            // misc
    static constexpr int MISC = 5 * G + 16 * G + 32 + 4 * G;  // ..., iscr, per-head counts
    static constexpr int OFF_BAR = (OFF_M + MISC * 4 + 7) / 8 * 8;   // [16 warps][3 stages] mbarriers
    static constexpr int FIX = (OFF_BAR + 16 * 3 * 8 + 127) / 128 * 128;
    static constexpr int PERW = 3 * STAGE + 16 * CT * 4 + 16 * G * 4;  // ring, C tile, P
    static constexpr int BUDGET = 223 * 1024;    // + the survivor list, within 227 KB
    static constexpr int NW0 = (BUDGET - FIX) / PERW;
    static constexpr int NW = NW0 > 16 ? 16 : NW0;
    static constexpr int NTHR = NW * 32;
    static constexpr int OFF_W = FIX;                                 // per-warp areas
    static constexpr int DYN = OFF_W + NW * PERW;                     // then the survivor list
    static int smem(int list_cap) { return DYN + list_cap * 2; }     // survivor list (u16 interleave index)
    static_assert(NW >= 2, "Louver v9: shared memory budget too small");
};

// CNT: the launch writes p.counts (an instantiation of its own, so that the launches
// without statistics — the bench, the production decode step — keep their code).
// SOLO: the launch has teams of one CTA (many slots, e.g. C3): the CTA's partial is the
// slot's result and is written out directly, with no ticket (also its own instantiation,
// so that the team path keeps its code).
template <int DP, int G, bool DENSE, bool CNT, bool SOLO = false>
__global__ void __launch_bounds__(C9<DP, G>::NTHR, C9<DP, G>::MINB) louver_layer_v9(const __grid_constant__ LayerParams vp) {
    using Ge = C9<DP, G>;
    constexpr bool PACK = G <= 4;  // P.V: hi and lo parts of P share one n-tile
    constexpr int NW = Ge::NW, NTHR = Ge::NTHR, NT = Ge::NT, NTP = Ge::NTP, KS = Ge::KS, CPR = Ge::CPR,
                  RB = Ge::RB, PPL = Ge::PPL, MT = Ge::MT, CT = Ge::CT;
    const QueryParams& p = vp.p;
    extern __shared__ __align__(128) unsigned char smem[];
    uint2* fre = reinterpret_cast<uint2*>(smem + Ge::OFF_FRE);
    uint2* frp = reinterpret_cast<uint2*>(smem + Ge::OFF_FRP);
    float* qf = reinterpret_cast<float*>(smem + Ge::OFF_Q);
    float* misc = reinterpret_cast<float*>(smem + Ge::OFF_M);
    float* tau_s = misc;               // [G]
    float* taup_s = misc + G;          // [G] probe threshold tau - 2^-12 S
    float* marg_s = misc + 2 * G;      // [G] 2^-13 S
    float* S_s = misc + 3 * G;         // [G]
    float* red = misc + 5 * G;         // [16 G]
    int* iscr = reinterpret_cast<int*>(misc + 21 * G);  // [32]
    // iscr[32 .. 32 + 4 G): this CTA's per-head counts (selected, attended, keys scanned); they
    // travel in its partial record and the merge writes the totals, so p.counts needs no
    // zeroing before the launch
    // this CTA's surviving cells as interleave indices k (cell = blk + k nb): in smem, or in
    // global scratch when the list outgrows shared memory
    unsigned short* slist_s = reinterpret_cast<unsigned short*>(smem + Ge::DYN);
    const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
    const int blk = vp.spread ? blockIdx.y : blockIdx.x, nbs = vp.nb;  // records / lists / traces: nbs per slot
    unsigned char* wbase = smem + Ge::OFF_W + warp * Ge::PERW;
    const unsigned ring = smem_u32(wbase);
    const int b7 = (int)((ring >> 7) & 7u);  // the same for every stage of the warp (4 KiB apart)
    const bool ktma = vp.ktma != 0;
    const unsigned kbar = smem_u32(smem + Ge::OFF_BAR) + warp * 24;  // this warp's 3 stage barriers
    unsigned kph = 0;                                                // their phase bits
    if (ktma) {
        if (lane == 0) {
            for (int i = 0; i < 3; ++i) mbar_init(kbar + 8 * i, 1);
            asm volatile("fence.mbarrier_init.release.cluster;\n" ::: "memory");
        }
        __syncwarp();
    }
    float* ct = reinterpret_cast<float*>(wbase + 3 * Ge::STAGE);
    float* pbuf = ct + 16 * CT;
    // C tile element (r, c) at r CT + c, its 16-byte chunk XORed with the bit-reversed
    // (r >> 1) & 3 when rows are 16 floats (mod 32 banks): the accumulator stores (rows r,
    // r + 2 of a half-warp get disjoint chunk pairs) and the per-row reads (rows of equal
    // parity get distinct chunks) are then bank-conflict free. Other pitches need no swizzle.
    constexpr bool CSW = CT % 32 == 16;
    auto cto = [](int r, int c) {
        if constexpr (!CSW) return r * CT + c;
        const int x = (r >> 1) & 3, f = ((x & 1) << 1) | (x >> 1);
        return r * CT + ((((c >> 2) ^ f) << 2) | (c & 3));
    };
    const int q4 = lane & 3;
    // per-lane ldmatrix offsets: A (rows = keys / cells) and V^T (trans)
    const int a_row = (lane & 7) + 8 * ((lane >> 3) & 1), a_hi = lane >> 4;
    const unsigned a_off = a_row * 128;
    const int a_rx = (a_row + b7) & 7;
    const int v_row = (lane & 7) + 8 * (lane >> 4), v_hi = (lane >> 3) & 1;
    const unsigned v_off = v_row * 128;
    const int v_rx = (v_row + b7) & 7;

    // programmatic dependent launch: dispatched early, while the preceding kernel in the
    // stream drains; only immutable data (sealed cell summaries) is read before
    // griddepcontrol.wait below
    asm volatile("griddepcontrol.launch_dependents;\n" ::: "memory");
    bool waited = false;
    long long* trace = nullptr;
#define LV9_TRACE(i) \
    if (trace && tid == 0) trace[i] = gtimer();

    // (no ring zeroing: a V stage is always the stage of its task's K block, loaded whole,
    // with rows past n zero-filled, so rows that are not attended hold finite values)

    const int slot0 = vp.spread ? blockIdx.x : blockIdx.y, sstep = vp.spread ? gridDim.x : gridDim.y;
    for (int slot = slot0; slot < vp.slots; slot += sstep) {
        const int nb = slot < vp.nfull ? nbs : nbs - 1;  // this slot's team
        if (blk >= nb) continue;                         // (uniform per CTA)
        trace = p.tot_trace ? p.tot_trace + ((size_t)slot * nbs + blk) * 64 : nullptr;
        LV9_TRACE(0)
        const __nv_bfloat16* Ks = reinterpret_cast<const __nv_bfloat16*>(p.K) + (size_t)slot * p.cap * DP;
        const __nv_bfloat16* Vs = reinterpret_cast<const __nv_bfloat16*>(p.V) + (size_t)slot * p.cap * DP;
        const unsigned char* sumb =
            reinterpret_cast<const unsigned char*>(vp.sum + (size_t)slot * p.cap_cells * (2 * DP));

        // ---- phase A prologue: the first summary blocks depend on nothing.
        // CTA blk of the team probes the slot's cells blk, blk + nb, blk + 2 nb, ... (a
        // fine interleave: every CTA sees the same mix of the sequence, so the survivors
        // split evenly with no team-wide exchange). CTA-local tile j = cells
        // blk + (16 j + i) nb, i < 16; warp w takes tiles w, w + NW, ...
        // Sub-task u of a warp: tile warp + (u >> 1) NW, half u & 1 ([hi] or [lo] rows).
        unsigned short* slist = vp.glist ? vp.glist + ((size_t)slot * nbs + blk) * vp.list_cap : slist_s;
        if (tid == 0) {
            iscr[2] = 0;  // survivors listed
            iscr[3] = 0;  // tasks claimed
        }
        if (CNT && tid < 4 * G) iscr[32 + tid] = 0;
        const long long cap_cells = p.cap_cells;
        // chunk k*32 + lane of a 16-row sub-block: row k*RPI0 + lane/CPR, chunk lane%CPR; the
        // swizzled destination repeats with period P0 in k (precomputed per lane)
        constexpr int RPI0 = 32 / CPR, P0 = 8 / RPI0;
        unsigned pdoff[P0];
#pragma unroll
        for (int kk = 0; kk < P0; ++kk) {
            const int row = kk * RPI0 + lane / CPR, c = lane % CPR;
            pdoff[kk] = lay(row, c, b7);
        }
        const size_t plane = ((size_t)(lane / CPR) * nb * (4 * DP)) + (size_t)(lane % CPR) * 16;
        const size_t pkstride = (size_t)RPI0 * nb * (4 * DP);
        auto p_issue = [&](int u, long long bound) {
            const long long c0 = blk + (long long)16 * (warp + (u >> 1) * NW) * nb;
            if (c0 < bound) {
                const unsigned dst = ring + (u % 3) * Ge::STAGE;
                const size_t hoff = (size_t)(u & 1) * DP * 2;
                if (c0 + 15LL * nb < cap_cells) {  // every row inside the arena
                    const unsigned char* src = sumb + (size_t)c0 * (4 * DP) + hoff + plane;
#pragma unroll
                    for (int k = 0; k < CPR / 2; ++k) cpa16(dst + (k / P0) * 8 * 128 + pdoff[k % P0], src + k * pkstride);
                } else {
#pragma unroll
                    for (int k = 0; k < CPR / 2; ++k) {
                        const int ch = k * 32 + lane, row = ch / CPR, c = ch % CPR;
                        long long cell = c0 + (long long)row * nb;
                        cell = cell < cap_cells ? cell : cap_cells - 1;  // past the arena: any row, ignored
                        cpa16(dst + lay(row, c, b7), sumb + (size_t)cell * (4 * DP) + hoff + c * 16);
                    }
                }
            }
            cpa_commit();
        };
        // The first summary tile of this warp is prefetched before the dependency wait when
        // its cells were complete when the query was enqueued (vp.sealed): a complete
        // cell's box never changes, so it cannot depend on the preceding kernel (an insert
        // only writes the open cell). Its stream then overlaps the preceding kernel's tail.
        bool pre = false;
        if (!waited) {
            // sub-blocks 0, 1 (tile warp) and 2 (tile warp + NW) fill the 3-stage ring
            const long long c0 = blk + (long long)16 * warp * nb, c1 = c0 + (long long)16 * NW * nb;
            pre = !DENSE && (c0 >= cap_cells || c0 + 15LL * nb < vp.sealed) &&
                  (c1 >= cap_cells || c1 + 15LL * nb < vp.sealed);
            if (pre)
                for (int u = 0; u < vp.npre; ++u) p_issue(u, cap_cells);
            asm volatile("griddepcontrol.wait;\n" ::: "memory");
            waited = true;
            LV9_TRACE(13)
        }
        // ---- setup: q, S_g, thresholds, B fragments (all inputs requested in one round trip,
        // ahead of the summary prefetch so they do not queue behind it in the memory system)
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
            const float tau_r = (!DENSE && tid < G) ? __ldcg(p.tau + (size_t)slot * G + tid) : 0.0f;
            // zero the fragment arrays (columns past PARTS * G stay zero)
            for (int i = tid; i < (Ge::SZ_FRE + Ge::SZ_FRP) / 16; i += NTHR)
                reinterpret_cast<uint4*>(smem + Ge::OFF_FRE)[i] = make_uint4(0u, 0u, 0u, 0u);
            float s[G];
#pragma unroll
            for (int g = 0; g < G; ++g) s[g] = 0.0f;
            if (trace && tid == 0) {
                asm volatile("" ::"f"(xq[0]));
                trace[9] = gtimer();
                asm volatile("" ::"f"(xc[0]));
                trace[12] = gtimer();
            }
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
                for (int w = 0; w < NW; ++w) v = __fadd_ru(v, red[w * G + tid]);
                const float tau = tau_r;
                S_s[tid] = v;
                tau_s[tid] = tau;
                taup_s[tid] = __fsub_rd(tau, __fmul_ru(v, 2.44140625e-4f));  // 2^-12 S
                marg_s[tid] = __fmul_ru(v, 1.220703125e-4f);                 // 2^-13 S
            }
            LV9_TRACE(10)
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
                        fe[((((ks >> 1) * NT + (col >> 3)) * 32 + (col & 7) * 4 + qq) * 2 + (ks & 1)) * 4 + e] = b;
                    }
#pragma unroll
                    for (int h = 0; h < 2; ++h) {
                        float z = h == 0 ? fmaxf(xq[k], 0.0f) : fminf(xq[k], 0.0f);  // [hi | lo] . [q+ | q-]
#pragma unroll
                        for (int P = 0; P < 2; ++P) {
                            const unsigned short b = bf_bits(z);
                            z -= bf_val(b);
                            const int col = P * G + g;
                            fp[((((h * (KS / 2) + (ks >> 1)) * NTP + (col >> 3)) * 32 + (col & 7) * 4 + qq) * 2 + (ks & 1)) * 4 + e] = b;
                        }
                    }
                }
            }
            __syncthreads();
        }
        LV9_TRACE(1)
        // the summary prefetch starts only now: cp.async issue stalls the issuing warp once
        // the memory system is saturated, so it must not sit in front of the setup
        if (!DENSE)
            for (int u = pre ? vp.npre : 0; u < 3; ++u) p_issue(u, cap_cells);
        const int rl = p.r_log2, r = 1 << rl;
        const long long ncells = (n + r - 1) >> rl;

        // ---- phase A: probe
        if (!DENSE) {
            float taup[G];
#pragma unroll
            for (int g = 0; g < G; ++g) taup[g] = taup_s[g];
            float acc[NTP][4];
            for (int u = 0;; ++u) {
                const long long c0 = blk + (long long)16 * (warp + (u >> 1) * NW) * nb;
                if (c0 >= ncells) break;
                cpa_wait<2>();  // sub-block u landed (u + 1, u + 2 may pend)
                __syncwarp();
                if (trace && lane == 0 && NW <= 16 && u == 0) trace[48 + warp] = gtimer();
                const int half = u & 1;
                if (half == 0) {
#pragma unroll
                    for (int nt = 0; nt < NTP; ++nt) acc[nt][0] = acc[nt][1] = acc[nt][2] = acc[nt][3] = 0.0f;
                }
                const unsigned sb = ring + (u % 3) * Ge::STAGE + a_off;
                const uint4* fh = reinterpret_cast<const uint4*>(frp) + half * (KS / 2) * NTP * 32;
#pragma unroll
                for (int k2 = 0; k2 < KS / 2; ++k2) {
                    unsigned a0[4], a1[4];
                    ldsm4(a0, sb + swz_off(2 * k2, a_hi, a_rx));
                    ldsm4(a1, sb + swz_off(2 * k2 + 1, a_hi, a_rx));
#pragma unroll
                    for (int nt = 0; nt < NTP; ++nt) {
                        const uint4 b = fh[(k2 * NTP + nt) * 32 + lane];
                        mma16816(acc[nt], a0, b.x, b.y);
                        mma16816(acc[nt], a1, b.z, b.w);
                    }
                }
                if (half == 1) {
#pragma unroll
                    for (int nt = 0; nt < NTP; ++nt) {
                        const int rw = lane >> 2, col = nt * 8 + 2 * q4;
                        *reinterpret_cast<float2*>(ct + cto(rw, col)) = make_float2(acc[nt][0], acc[nt][1]);
                        *reinterpret_cast<float2*>(ct + cto(rw + 8, col)) = make_float2(acc[nt][2], acc[nt][3]);
                    }
                    __syncwarp();
                    unsigned gm = 0;
                    int scan = 0;
                    const long long cell = c0 + (long long)lane * nb;
                    if (lane < 16 && cell < ncells) {
                        const long long cs = cell << rl, ce = cs + r;
                        if (ce > indexed) {
                            gm = (1u << G) - 1u;  // holds buffer keys: scanned densely
                        } else {
#pragma unroll
                            for (int g = 0; g < G; ++g)
                                if (ct[cto(lane, g)] + ct[cto(lane, G + g)] >= taup[g]) gm |= 1u << g;
                        }
                        scan = (int)((ce < n ? ce : n) - cs);
                    }
                    const unsigned m = __ballot_sync(0xffffffffu, gm != 0) & 0xffffu;
                    if (m) {  // append the survivors to the CTA's list
                        int base = 0;
                        if (lane == 0) base = atomicAdd(iscr + 2, __popc(m));
                        base = __shfl_sync(0xffffffffu, base, 0);
                        if (gm) {
                            const int at = base + __popc(m & ((1u << lane) - 1u));
                            slist[at] = (unsigned short)(16 * (warp + (u >> 1) * NW) + lane);
                            // the survivor's key blocks are requested into L2 now: the HBM is
                            // mostly idle while the probe finishes, and the exact phase that
                            // follows is HBM-bound (its first tasks then hit in L2)
                            if (at < vp.kpf) bulk_prefetch_l2(Ks + ((size_t)cell << rl) * DP, (unsigned)(RB << rl));
                        }
                    }
                    if (p.totals) {
                        const int tested = __popc(__ballot_sync(0xffffffffu, lane < 16 && cell < ncells));
                        if (lane == 0) {
                            atomicAdd(p.totals + 0, (unsigned long long)tested);
                            atomicAdd(p.totals + 1, (unsigned long long)__popc(m));
                        }
                    }
                    if constexpr (CNT) {
#pragma unroll
                        for (int g = 0; g < G; ++g) {
                            const int v = lvk::warp_sum_int((gm >> g) & 1 ? scan : 0);
                            if (lane == 0 && v) atomicAdd(iscr + 32 + g * 4 + 2, v);
                        }
                    }
                }
                __syncwarp();
                p_issue(u + 3, ncells);  // into the stage just consumed
            }
            cpa_wait<0>();
            __syncwarp();
            if (trace && lane == 0 && NW <= 16) trace[32 + warp] = gtimer();
        }
        LV9_TRACE(2)

        __syncthreads();  // the CTA's survivor list is complete
        LV9_TRACE(3)
        // DENSE: every cell the CTA owns (blk, blk + nb, ... < ncells), in order
        const int nsurv = DENSE ? (int)(ncells > blk ? (ncells - blk + nb - 1) / nb : 0) : iscr[2];
        LV9_TRACE(4)
        if (trace && tid == 0) trace[15] = nsurv;

        // ---- phase B: exact + attend
        const int g_me = lane % G;
        const float tau_me = tau_s[g_me], marg_me = marg_s[g_me];
        const float* q_me = qf + g_me * (DP + 4);
        // scores in log2 units: exp(scale s - m) = 2^(scale log2(e) s - m / ln 2)
        const float scale = p.scale * 1.4426950408889634f;
        const int tpc_l2 = rl - 4;  // log2(16-row tasks per cell)
        float o[MT][4];
#pragma unroll
        for (int mt = 0; mt < MT; ++mt) o[mt][0] = o[mt][1] = o[mt][2] = o[mt][3] = 0.0f;
        float mrun = -INFINITY, lpart = 0.0f;
        int my_sel = 0, my_att = 0;
        unsigned long long t_keys = 0, t_vals = 0;

        {
            // tasks = 16-key blocks of the listed cells, claimed through a shared counter
            // one task ahead (balances warps whatever each task costs)
            const int ntask = nsurv << tpc_l2;
            // 32-bit key indices: the launcher guarantees cap < 2^31 rows per slot
            const int n32 = (int)n, idx32 = (int)indexed;
            auto key0 = [&](int t) -> int {
                const int cell = blk + (DENSE ? (t >> tpc_l2) : (int)slist[t >> tpc_l2]) * nb;
                return (cell << rl) + ((t & ((1 << tpc_l2) - 1)) << 4);
            };
            // chunk k*32 + lane of a 16-row block: row k*RPI + lane/CPR, column chunk lane%CPR,
            // so the source is base + 512 k + 16 lane and the swizzled destination repeats
            // with period P in k: precompute the P per-lane destination offsets
            constexpr int RPI = 32 / CPR, P = 8 / RPI;
            unsigned doff[P];
#pragma unroll
            for (int kk = 0; kk < P; ++kk) {
                const int row = kk * RPI + lane / CPR, c = lane % CPR;
                doff[kk] = lay(row, c, b7);
            }
            auto k_issue = [&](int t, int kb, int stage) {  // rows past n land as zeros
                if (ktma) {  // one TMA tile per 128-byte column half; rows past n are the arena's zeros
                    if (t < ntask) {
                        __syncwarp();
                        if (lane == 0) {
                            fence_proxy_async();  // the stage's last generic reads / cp.async writes
                            const unsigned bar = kbar + 8 * stage, dst = ring + stage * Ge::STAGE;
                            mbar_expect_tx(bar, Ge::STAGE);
                            const int row = (int)(slot * p.cap) + kb;
#pragma unroll
                            for (int h = 0; h < DP / 64; ++h) tma_load_2d(dst + h * 2048, &vp.kmap, h * 64, row, bar);
                        }
                    }
                    return;
                }
                if (t < ntask) {
                    const unsigned char* src = reinterpret_cast<const unsigned char*>(Ks) + (size_t)kb * RB + lane * 16;
                    const unsigned dst = ring + stage * Ge::STAGE;
                    if (kb + 16 <= n32) {  // the common case: the whole block is stored keys
#pragma unroll
                        for (int k = 0; k < CPR / 2; ++k) cpa16(dst + (k / P) * 8 * 128 + doff[k % P], src + k * 512);
                    } else {
                        const int lim = n32 - kb - lane / CPR;
#pragma unroll
                        for (int k = 0; k < CPR / 2; ++k)
                            cpa16z(dst + (k / P) * 8 * 128 + doff[k % P], src + k * 512, k * RPI < lim);
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
            bool pend = false;
            unsigned pb[4] = {0u, 0u, 0u, 0u};  // B fragments of the pending task's P (hi b0 b1, lo b0 b1)
            int k0 = t < ntask ? key0(t) : 0;  // first key of task t
            k_issue(t, k0, 0);
            cpa_commit();  // stands for V(t-1)
            while (t < ntask) {
                const int s1 = st == 2 ? 0 : st + 1;
                const int s2 = st == 0 ? 2 : st - 1;  // stage of V(t-1)
                const int tn = __shfl_sync(0xffffffffu, cb, 0);
                if (lane == 0 && tn < ntask) cb = atomicAdd(iscr + 3, 1);
                const int kn = tn < ntask ? key0(tn) : 0;
                k_issue(tn, kn, s1);
                // the CTA's last tasks end on the chain K round trip -> scores -> V round trip:
                // their value blocks are requested into L2 with the keys
                if (lane == 0 && tn < ntask && tn >= ntask - vp.vtail)
                    bulk_prefetch_l2(Vs + (size_t)kn * DP, 16 * RB);
                if (ktma) {  // K(t) landed
                    mbar_wait(kbar + 8 * st, (kph >> st) & 1u);
                    kph ^= 1u << st;
                } else {
                    cpa_wait<2>();  // K(t) landed (V(t-1), K(t+1) may pend)
                }
                __syncwarp();
                // -- scores: 16 keys x [q0|q1|q2] per head
                const unsigned sb = ring + st * Ge::STAGE;
                {
                    float acc[NT][4];
#pragma unroll
                    for (int nt = 0; nt < NT; ++nt) acc[nt][0] = acc[nt][1] = acc[nt][2] = acc[nt][3] = 0.0f;
                    const uint4* fq = reinterpret_cast<const uint4*>(fre);
#pragma unroll
                    for (int k2 = 0; k2 < KS / 2; ++k2) {
                        unsigned a0[4], a1[4];
                        ldsm4(a0, sb + a_off + swz_off(2 * k2, a_hi, a_rx));
                        ldsm4(a1, sb + a_off + swz_off(2 * k2 + 1, a_hi, a_rx));
#pragma unroll
                        for (int nt = 0; nt < NT; ++nt) {
                            const uint4 b = fq[(k2 * NT + nt) * 32 + lane];
                            mma16816(acc[nt], a0, b.x, b.y);
                            mma16816(acc[nt], a1, b.z, b.w);
                        }
                    }
#pragma unroll
                    for (int nt = 0; nt < NT; ++nt) {
                        const int rw = lane >> 2, col = nt * 8 + 2 * q4;
                        *reinterpret_cast<float2*>(ct + cto(rw, col)) = make_float2(acc[nt][0], acc[nt][1]);
                        *reinterpret_cast<float2*>(ct + cto(rw + 8, col)) = make_float2(acc[nt][2], acc[nt][3]);
                    }
                }
                __syncwarp();
                // -- classify this lane's pairs (row pi / G, head g_me)
                float s[PPL];
                unsigned und = 0, selb = 0;
#pragma unroll
                for (int j = 0; j < PPL; ++j) {
                    const int pi = lane + 32 * j, rw = pi / G;
                    const int rc = rw < 16 ? rw : 15;
                    const float sc = (ct[cto(rc, g_me)] + ct[cto(rc, G + g_me)]) + ct[cto(rc, 2 * G + g_me)];
                    const bool valid = (G > 1 || lane < 16) && k0 + rw < n32;
                    const bool sel = valid && (DENSE || sc >= tau_me + marg_me);
                    const bool u = !DENSE && valid && !sel && sc >= tau_me - marg_me;
                    s[j] = sc;
                    und |= (unsigned)u << j;
                    selb |= (unsigned)sel << j;
                }
                if (!DENSE && __any_sync(0xffffffffu, und != 0)) {  // rare: the normative sequential dot
#pragma unroll
                    for (int j = 0; j < PPL; ++j) {
                        if ((und >> j) & 1) {
                            const int rw = (lane + 32 * j) / G;
                            const unsigned rb = sb;
                            float a2 = 0.0f;
#pragma unroll 1
                            for (int cc = 0; cc < CPR; ++cc) {
                                const uint4 kv = lds16(rb + lay(rw, cc, b7));
                                float kf[8];
                                lvk::unpack16<__nv_bfloat16>(kv, kf);
#pragma unroll
                                for (int e2 = 0; e2 < 8; ++e2) a2 = __fadd_rn(a2, __fmul_rn(q_me[cc * 8 + e2], kf[e2]));
                            }
                            s[j] = a2;
                            if (a2 >= tau_me) selb |= 1u << j;
                        }
                    }
                }
                unsigned amask = 0;  // rows with any attended head
                float mloc = -INFINITY;
#pragma unroll
                for (int j = 0; j < PPL; ++j) {
                    const int pi = lane + 32 * j, rw = pi / G;
                    const int kk = k0 + rw;
                    const bool valid = (G > 1 || lane < 16) && kk < n32;
                    const bool sel = (selb >> j) & 1;
                    if (sel) {
                        ++my_sel;
                        if (!DENSE && p.bits)
                            atomicOr(p.bits + ((size_t)slot * G + g_me) * p.bits_words + (kk >> 5), 1u << (kk & 31));
                    }
                    const bool att = sel || (valid && !p.strict && kk >= idx32);
                    my_att += att;
                    s[j] = att ? scale * s[j] : -INFINITY;
                    mloc = fmaxf(mloc, s[j]);
                    amask |= row_bits<G>(__ballot_sync(0xffffffffu, att)) << (j * (32 / G));
                }
                if (p.totals && lane == 0) t_keys += (k0 + 16 <= n32) ? 16 : (n32 > k0 ? n32 - k0 : 0);
                float alpha = 1.0f;
                unsigned nbf[4] = {0u, 0u, 0u, 0u};
                if (amask) {
                    if (p.totals && lane == 0) t_vals += __popc(amask);
#pragma unroll
                    for (int of = 16; of >= G; of >>= 1) mloc = fmaxf(mloc, __shfl_xor_sync(0xffffffffu, mloc, of));
                    // lazy rescale: the reference max moves only when a score exceeds it by
                    // more than 8 nats (weights stay <= e^8); o and l are rescaled only then.
                    // The first move (from -inf) needs no rescale: o and l are still zero.
                    if (mloc > mrun + 11.541560327111707f) {
                        if (mrun != -INFINITY) alpha = ex2f(mrun - mloc);
                        mrun = mloc;
                    }
                    float lp = lpart * alpha;
#pragma unroll
                    for (int j = 0; j < PPL; ++j) {
                        const float pv = s[j] == -INFINITY ? 0.0f : ex2f(s[j] - mrun);
                        lp += pv;
                        if (G > 1 || lane < 16) pbuf[lane + 32 * j] = pv;
                    }
                    lpart = lp;
                    __syncwarp();
                    // B fragment of P: k = rows (2q, 2q+1 | 2q+8, 2q+9), n = head lane/4
                    const int hn = lane >> 2;
                    float pv4[4] = {0.0f, 0.0f, 0.0f, 0.0f};
                    // G <= 4: one n-tile carries both parts, column h = hi part of head h,
                    // column G + h = lo part (summed after the loop); G = 8: two n-tiles
                    const int hh = PACK ? hn % G : hn;
                    if (PACK ? hn < 2 * G : hn < G) {
                        pv4[0] = pbuf[(2 * q4) * G + hh];
                        pv4[1] = pbuf[(2 * q4 + 1) * G + hh];
                        pv4[2] = pbuf[(2 * q4 + 8) * G + hh];
                        pv4[3] = pbuf[(2 * q4 + 9) * G + hh];
                    }
                    float lo4[4];
#pragma unroll
                    for (int e = 0; e < 4; ++e) lo4[e] = pv4[e] - bf_val(bf_bits(pv4[e]));
                    if (PACK) {
                        const bool lo = hn >= G;
                        nbf[0] = lo ? bf2(lo4[0], lo4[1]) : bf2(pv4[0], pv4[1]);
                        nbf[1] = lo ? bf2(lo4[2], lo4[3]) : bf2(pv4[2], pv4[3]);
                    } else {
                        nbf[0] = bf2(pv4[0], pv4[1]);
                        nbf[1] = bf2(pv4[2], pv4[3]);
                        nbf[2] = bf2(lo4[0], lo4[1]);
                        nbf[3] = bf2(lo4[2], lo4[3]);
                    }
                }
                __syncwarp();  // K(t) and pbuf reads done
                // -- V(t): attended rows into K(t)'s stage (same row positions)
                if (amask) {  // RPI rows per warp instruction, from a rank list of the attended rows
                    unsigned char* rows8 = reinterpret_cast<unsigned char*>(ct);  // the C tile is dead here
                    if (lane < 16 && ((amask >> lane) & 1u)) rows8[__popc(amask & ((1u << lane) - 1u))] = (unsigned char)lane;
                    __syncwarp();
                    const int nr = __popc(amask), cc = lane % CPR;
                    const unsigned dst = ring + st * Ge::STAGE;
                    const unsigned char* vsrc = reinterpret_cast<const unsigned char*>(Vs + (size_t)k0 * DP) + cc * 16;
                    for (int k = lane / CPR; k < nr; k += RPI) {
                        const int rsel = rows8[k];
                        cpa16(dst + lay(rsel, cc, b7), vsrc + rsel * RB);
                    }
                }
                cpa_commit();
                // -- fold V(t-1) (frame m_{t-1}), then move o to frame m_t
                if (ktma)
                    cpa_wait<1>();  // V(t-1) landed (V(t) may pend)
                else
                    cpa_wait<2>();  // V(t-1) landed (K(t+1), V(t) may pend)
                __syncwarp();
                if (pend) {
                    const unsigned vb = ring + s2 * Ge::STAGE + v_off;
#pragma unroll
                    for (int mt = 0; mt < MT; ++mt) {
                        unsigned a[4];
                        ldsm4t(a, vb + swz_off(mt, v_hi, v_rx));
                        mma16816(o[mt], a, pb[0], pb[1]);
                        if (!PACK) mma16816(o[mt], a, pb[2], pb[3]);
                    }
                }
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
                pend = amask != 0;
#pragma unroll
                for (int e = 0; e < 4; ++e) pb[e] = nbf[e];
                st = s1;
                t = tn;
                k0 = kn;
            }
            cpa_wait<0>();
            __syncwarp();
            if (pend) {  // the last task's V
                const int s2 = st == 0 ? 2 : st - 1;
                const unsigned vb = ring + s2 * Ge::STAGE + v_off;
#pragma unroll
                for (int mt = 0; mt < MT; ++mt) {
                    unsigned a[4];
                    ldsm4t(a, vb + swz_off(mt, v_hi, v_rx));
                    mma16816(o[mt], a, pb[0], pb[1]);
                    if (!PACK) mma16816(o[mt], a, pb[2], pb[3]);
                }
            }
            __syncwarp();
        }
        if (PACK) {  // fold the lo-part columns (G + h) into the hi-part columns (h)
#pragma unroll
            for (int mt = 0; mt < MT; ++mt) {
                if (G == 1) {
                    o[mt][0] += o[mt][1];
                    o[mt][2] += o[mt][3];
                } else {
#pragma unroll
                    for (int e = 0; e < 4; ++e) o[mt][e] += __shfl_xor_sync(0xffffffffu, o[mt][e], G / 2);
                }
            }
        }
        LV9_TRACE(5)
        if (trace && lane == 0 && NW <= 16) trace[16 + warp] = gtimer();

        // ---- statistics: lanes with the same g = lane % G hold that head's counts
        if constexpr (CNT) {
            int s0 = my_sel, s1 = my_att;
#pragma unroll
            for (int of = 16; of >= G; of >>= 1) {
                s0 += __shfl_xor_sync(0xffffffffu, s0, of);
                s1 += __shfl_xor_sync(0xffffffffu, s1, of);
            }
            if (lane < G) {
                if (s0) atomicAdd(iscr + 32 + lane * 4 + 0, s0);
                if (s1) atomicAdd(iscr + 32 + lane * 4 + 1, s1);
            }
        }
        if (p.totals && lane == 0) {
            if (t_keys) atomicAdd(p.totals + 2, t_keys);
            if (t_vals) atomicAdd(p.totals + 3, t_vals);
        }
#pragma unroll
        for (int of = 16; of >= G; of >>= 1) lpart += __shfl_xor_sync(0xffffffffu, lpart, of);

        // ---- warp partials -> CTA partial [G][DP+2] (m, l, o)
        constexpr int Wd = G * (DP + 2);
        constexpr int Wp = Wd + (CNT ? 4 * G : 0);  // the CTA's partial record: [G][DP+2] (then the counts [G][4])
        // in shared memory a head's row is DP + 4 floats (== 4 mod 32 banks): the o stores of
        // the lanes' (head, column) pairs below then hit distinct banks
        constexpr int WP = DP + 4;
        static_assert(G * (DP + 4) * 4 <= Ge::PERW, "a warp partial fits its ring area");
        // warp w's partial sits at the start of its own ring area (free once its tasks are
        // done), so a warp writes it as soon as it finishes, with no CTA barrier in front
        // warp stride in floats: the ring area plus 2, so the header reads of lanes w < NW at
        // w WS (one per warp) fall in distinct banks; the partial stays inside the warp's area
        constexpr int WS = Ge::PERW / 4 + 2;
        static_assert(G * (DP + 4) * 4 + 8 * 16 <= Ge::PERW, "the shifted warp partial fits its ring area");
        float* wred = reinterpret_cast<float*>(smem + Ge::OFF_W);  // [NW][WS]
        float* shw = red;                                           // [NW][G] weights
        {
            float* w = wred + warp * WS;
            if (lane < G) {
                w[lane * WP] = mrun * 0.6931471805599453f;  // back to nats
                w[lane * WP + 1] = lpart;
            }
#pragma unroll
            for (int mt = 0; mt < MT; ++mt) {
#pragma unroll
                for (int e = 0; e < 4; ++e) {
                    const int h = 2 * q4 + (e & 1), c = 16 * mt + (lane >> 2) + 8 * (e >> 1);
                    if (h < G) w[h * WP + 2 + c] = o[mt][e];
                }
            }
        }
        __syncthreads();
        float* part = p.partial_ws + ((size_t)slot * nbs + blk) * Wp;
        if (CNT && tid < 4 * G) reinterpret_cast<int*>(part + Wd)[tid] = iscr[32 + tid];
        for (int g = warp; g < G; g += NW) {  // warp g combines head g's NW warp headers, one warp per lane
            const float mw = lane < NW ? wred[lane * WS + g * WP] : -INFINITY;
            const float lw = lane < NW ? wred[lane * WS + g * WP + 1] : 0.0f;
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
            float s = 0.0f;
#pragma unroll
            for (int w = 0; w < NW; ++w) s = fmaf(shw[w * G + g], wred[w * WS + g * WP + 2 + c], s);
            part[g * (DP + 2) + 2 + c] = s;
        }
        LV9_TRACE(6)

        // ---- phase C: the last CTA of the team merges the nb partials
        int* ticket = vp.stickets + slot;
        __syncthreads();
        if constexpr (SOLO) {  // a team of one (nb == 1): its partial is the result, no ticket
            for (int i = tid; i < G * DP; i += NTHR) {
                const int g = i / DP, c = i % DP;
                const float l = __ldcg(part + g * (DP + 2) + 1), o = __ldcg(part + g * (DP + 2) + 2 + c);
                if (p.out) p.out[((size_t)slot * G + g) * DP + c] = l > 0.0f ? o / l : 0.0f;
                if (p.partial_out) p.partial_out[(size_t)slot * Wd + g * (DP + 2) + 2 + c] = o;
            }
            if (tid < G) {
                const float m = __ldcg(part + tid * (DP + 2)), l = __ldcg(part + tid * (DP + 2) + 1);
                if (p.partial_out) {
                    p.partial_out[(size_t)slot * Wd + tid * (DP + 2)] = m;
                    p.partial_out[(size_t)slot * Wd + tid * (DP + 2) + 1] = l;
                }
                if (CNT) p.counts[((size_t)slot * G + tid) * 4 + 3] = l > 0.0f ? 1 : 0;
            }
            if (CNT && tid < 3 * G) p.counts[((size_t)slot * G + tid / 3) * 4 + tid % 3] = iscr[32 + (tid / 3) * 4 + tid % 3];
            __syncthreads();
            __syncthreads();  // (as at the end of the merge: the rings are reused by the next slot)
            continue;
        }
        if (tid == 0) iscr[1] = atom_add_acq_rel(ticket, 1) == nb - 1;
        __syncthreads();
        if (iscr[1]) {
            LV9_TRACE(8)
            // one round trip: every thread requests its o elements of CH partials into
            // registers, the header warps request the (m, l) pairs alongside, and the
            // weights are ready by the time the o values land
            const float* src = p.partial_ws + (size_t)slot * nbs * Wp;
            float* M = reinterpret_cast<float*>(smem + Ge::OFF_W);  // scratch over the rings
            float* L = M + G;
            float* wgt = M + 2 * G;  // [nb][G]
            constexpr int EPT = (G * DP + NTHR - 1) / NTHR;
            constexpr int CH = EPT == 1 ? 24 : 12;  // partials per register chunk
            int csum = 0;  // thread tid < 3 G: head tid / 3's count tid % 3 over the team
            if (CNT && tid < 3 * G) {
                const int* cs = reinterpret_cast<const int*>(src + Wd) + (tid / 3) * 4 + tid % 3;
#pragma unroll 8
                for (int s2 = 0; s2 < nb; ++s2) csum += __ldcg(cs + (size_t)s2 * Wp);
            }
            float accr[EPT];
#pragma unroll
            for (int k = 0; k < EPT; ++k) accr[k] = 0.0f;
            for (int s0 = 0; s0 < nb; s0 += CH) {
                const int cnt = nb - s0 < CH ? nb - s0 : CH;
                float ov[EPT][CH];
#pragma unroll
                for (int k = 0; k < EPT; ++k) {
                    const int i = tid + k * NTHR;
                    const float* os = src + (size_t)s0 * Wp + (i / DP) * (DP + 2) + 2 + i % DP;
#pragma unroll
                    for (int j = 0; j < CH; ++j) ov[k][j] = (i < G * DP && j < cnt) ? __ldcg(os + (size_t)j * Wp) : 0.0f;
                }
                if (s0 == 0) {
                    LV9_TRACE(11)
                    for (int g = warp; g < G; g += NW) {  // one warp per head: max, weights, l
                        float mh[2], lh[2];
#pragma unroll
                        for (int t = 0; t < 2; ++t) {
                            const int s2 = lane + 32 * t;
                            mh[t] = s2 < nb ? __ldcg(src + (size_t)s2 * Wp + g * (DP + 2)) : -INFINITY;
                            lh[t] = s2 < nb ? __ldcg(src + (size_t)s2 * Wp + g * (DP + 2) + 1) : 0.0f;
                        }
                        float mm = fmaxf(mh[0], mh[1]);
                        for (int s2 = lane + 64; s2 < nb; s2 += 32) mm = fmaxf(mm, __ldcg(src + (size_t)s2 * Wp + g * (DP + 2)));
#pragma unroll
                        for (int o2 = 16; o2 > 0; o2 >>= 1) mm = fmaxf(mm, __shfl_xor_sync(0xffffffffu, mm, o2));
                        float l = 0.0f;
#pragma unroll
                        for (int t = 0; t < 2; ++t) {
                            const int s2 = lane + 32 * t;
                            const float w = mh[t] == -INFINITY ? 0.0f : __expf(mh[t] - mm);
                            if (s2 < nb) wgt[s2 * G + g] = w;
                            l += w * lh[t];
                        }
                        for (int s2 = lane + 64; s2 < nb; s2 += 32) {
                            const float ms = __ldcg(src + (size_t)s2 * Wp + g * (DP + 2));
                            const float w = ms == -INFINITY ? 0.0f : __expf(ms - mm);
                            wgt[s2 * G + g] = w;
                            l += w * __ldcg(src + (size_t)s2 * Wp + g * (DP + 2) + 1);
                        }
#pragma unroll
                        for (int o2 = 16; o2 > 0; o2 >>= 1) l += __shfl_xor_sync(0xffffffffu, l, o2);
                        if (lane == 0) {
                            M[g] = mm;
                            L[g] = l;
                        }
                    }
                    __syncthreads();
                }
#pragma unroll
                for (int k = 0; k < EPT; ++k) {
                    const int i = tid + k * NTHR;
                    const int g = (i / DP) < G ? i / DP : 0;
                    float a = accr[k];
#pragma unroll
                    for (int j = 0; j < CH; ++j)
                        if (j < cnt) a = fmaf(wgt[(s0 + j) * G + g], ov[k][j], a);
                    accr[k] = a;
                }
            }
            LV9_TRACE(14)
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
                if (CNT) p.counts[((size_t)slot * G + tid) * 4 + 3] = L[tid] > 0.0f ? 1 : 0;
            }
            if (CNT && tid < 3 * G) {  // the team's selected / attended / scanned totals
                p.counts[((size_t)slot * G + tid / 3) * 4 + tid % 3] = csum;
            }
            if (tid == 0) *ticket = 0;
            LV9_TRACE(7)
        }
        __syncthreads();
        __syncthreads();  // the rings served as merge scratch
    }
#undef LV9_TRACE
}

cudaError_t launch_layer_v9(int DP, int G, bool dense, LayerParams vp, int slots, int sms, cudaStream_t st, int* geo);

}  // namespace lvk9
