// Louver bf16 query path, v11: loader-fed persistent kernel per layer (sm_100a).
//
// Per slot (sequence b, kv head h) a team of nb CTAs (one per SM) shares a work
// queue in global memory. Each CTA is one loader warp plus NC compute warps around
// a pool of SP stage pairs (2 x 16 rows each) with full/empty mbarriers:
//
//   loader   lane 0 only issues memory traffic, so no compute warp ever stalls on a
//            saturated memory system: first the CTA's 16-cell summary tiles
//            ([hi] and [lo] halves, TMA with the 128-byte swizzle), then pairs of
//            16-key blocks claimed from the slot's queue (one atomic per pair), then
//            one DONE group per compute warp. Group g goes to stage pair g % SP and
//            compute warp g % NC.
//   compute  a probe group scores the tile's cell boxes against [q+ | q-] on the
//            tensor cores (LouverCache::query's filter stage, cache.cpp:30-47) and
//            appends the surviving cells' 16-key blocks to the queue; a cell survives
//            for head g iff its bound reaches tau_g - 2^-12 S_g (sound: the bf16 split
//            error is far inside the margin), or it holds buffer keys. A key group
//            scores 2 x 16 keys against [q0|q1|q2] (exact_check, query.cpp:22-31),
//            settles the pairs within 2^-13 S_g of tau with the normative sequential
//            fp32 dot (core.hpp:17-21), gathers the V rows of the attended keys
//            (selected ∪ buffer unless strict, cache.cpp:48-68) into a private
//            double buffer and folds them into an online softmax with P.V on the
//            tensor cores (sparse_attention, query.cpp:338-371).
//   merge    compute (m, l, o) -> CTA partial -> the last CTA of the team combines
//            the nb partials (log-sum-exp) and resets the team's queue.
#pragma once

#include "louver_v10.cuh"

namespace lvk11 {

using lvk::QueryParams;
using lvk10::V10Params;
using namespace lvk10;

enum : int { kProbe = 1, kKeys = 2, kDone = 3 };

struct GroupMeta {
    int type;       // kProbe, kKeys, kDone
    int last;       // kProbe: the compute warp's last probe group of this slot
    long long a;    // kProbe: tile; kKeys: first block's key row
    long long b;    // kKeys: second block's key row, or -1
    long long pad;
};

template <int DP, int G>
struct C11 {
    static constexpr int NPAN = DP / 64;
    static constexpr int RB = DP * 2;
    static constexpr int STAGE = 16 * RB;  // 16 rows: one key block, or one half of a summary tile
    static constexpr int NT = (3 * G + 7) / 8;
    static constexpr int NTP = (2 * G + 7) / 8;
    static constexpr int KS = DP / 16;
    static constexpr int CPR = DP / 8;
    static constexpr int PPL = G >= 2 ? G / 2 : 1;
    static constexpr int MT = DP / 16;
    static constexpr int CT = 8 * (NT > NTP ? NT : NTP);
    static constexpr int NC = DP == 64 ? 12 : (DP == 128 ? 8 : 5);  // compute warps
    static constexpr int NW = NC + 1;                                  // + the loader warp
    static constexpr int NTHR = NW * 32;
    static constexpr int VB = 3;  // V buffers per compute warp (V of task t is folded at task t + 2)
    static constexpr int SZ_FRE = KS * NT * 32 * 8;
    static constexpr int SZ_FRP = 2 * KS * NTP * 32 * 8;
    static constexpr int SZ_Q = G * (DP + 4) * 4;
    static constexpr int MISC = 8 * G + 16 * G + 64;  // floats
    static constexpr int SZ_CT = 16 * CT * 4 + 16 * G * 4;
    static constexpr int PERW = VB * STAGE + SZ_CT;
    static constexpr int SPMAX = 32;
    static constexpr int FIX = SZ_FRE + SZ_FRP + SZ_Q + MISC * 4 + SPMAX * (16 + (int)sizeof(GroupMeta)) + 1024;
    static constexpr int BUDGET = 227 * 1024;
    static constexpr int SP0 = (BUDGET - FIX - NC * PERW) / (2 * STAGE);
    static constexpr int SP = SP0 > SPMAX ? SPMAX : SP0;  // stage pairs
    static constexpr int OFF_POOL = 0;
    static constexpr int OFF_V = OFF_POOL + SP * 2 * STAGE;
    static constexpr int OFF_CT = OFF_V + NC * VB * STAGE;
    static constexpr int OFF_FRE = OFF_CT + NC * SZ_CT;
    static constexpr int OFF_FRP = OFF_FRE + SZ_FRE;
    static constexpr int OFF_Q = OFF_FRP + SZ_FRP;
    static constexpr int OFF_M = OFF_Q + SZ_Q;
    static constexpr int OFF_BAR = (OFF_M + MISC * 4 + 15) / 16 * 16;  // full[SP], empty[SP]
    static constexpr int OFF_META = OFF_BAR + SPMAX * 16;
    static constexpr int SMEM = OFF_META + SPMAX * (int)sizeof(GroupMeta) + 1024;
    static_assert(SP >= 2, "Louver v11: too few stage pairs");
    static_assert(SMEM <= BUDGET, "Louver v11: shared memory over budget");
};

__device__ __forceinline__ void mbar_arrive(unsigned bar) {
    asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];\n" ::"r"(bar) : "memory");
}
__device__ __forceinline__ int ld_volatile_s(const int* p) { return *reinterpret_cast<const volatile int*>(p); }

template <int DP, int G>
__global__ void __launch_bounds__(C11<DP, G>::NTHR, 1) louver_layer_v11(const __grid_constant__ V10Params vp) {
    using Ge = C11<DP, G>;
    constexpr int NC = Ge::NC, NW = Ge::NW, NTHR = Ge::NTHR, NT = Ge::NT, NTP = Ge::NTP, KS = Ge::KS,
                  CPR = Ge::CPR, RB = Ge::RB, PPL = Ge::PPL, MT = Ge::MT, CT = Ge::CT, NPAN = Ge::NPAN,
                  SP = Ge::SP, STAGE = Ge::STAGE, VB = Ge::VB;
    const QueryParams& p = vp.p;
    extern __shared__ unsigned char smem_raw[];
    const unsigned raw_u = smem_u32(smem_raw);
    const unsigned base_u = (raw_u + 1023u) & ~1023u;
    unsigned char* smem = smem_raw + (base_u - raw_u);
    uint2* fre = reinterpret_cast<uint2*>(smem + Ge::OFF_FRE);
    uint2* frp = reinterpret_cast<uint2*>(smem + Ge::OFF_FRP);
    float* qf = reinterpret_cast<float*>(smem + Ge::OFF_Q);
    float* misc = reinterpret_cast<float*>(smem + Ge::OFF_M);
    float* tau_s = misc;
    float* taup_s = misc + G;
    float* marg_s = misc + 2 * G;
    float* red = misc + 8 * G;                          // [16 G]
    int* iscr = reinterpret_cast<int*>(misc + 24 * G);  // [64]: 0 tasks, 1 merge winner, 2 probe tiles published
    GroupMeta* meta = reinterpret_cast<GroupMeta*>(smem + Ge::OFF_META);
    const unsigned fullb = base_u + Ge::OFF_BAR, emptyb = fullb + SP * 8;
    const unsigned pool = base_u + Ge::OFF_POOL;
    const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
    const bool loader = warp == NC;
    const int blk = blockIdx.x, nb = vp.nb;
    const int q4 = lane & 3;
    const int a_row = (lane & 7) + 8 * ((lane >> 3) & 1), a_hi = lane >> 4;
    const int v_row = (lane & 7) + 8 * (lane >> 4), v_hi = (lane >> 3) & 1;
    const unsigned vbuf = base_u + Ge::OFF_V + (unsigned)(warp % NC * VB * STAGE);
    float* ct = reinterpret_cast<float*>(smem + Ge::OFF_CT + warp % NC * Ge::SZ_CT);
    float* pbuf = ct + 16 * CT;

    if (tid == 0) {
        for (int s = 0; s < SP; ++s) {
            mbar_init(fullb + 8u * s, 1);
            mbar_init(emptyb + 8u * s, 1);
        }
        asm volatile("fence.mbarrier_init.release.cluster;\n" ::: "memory");
    }
    // V buffers start as zeros: rows a task does not load meet P = 0 and must be finite
    for (int i = tid; i < NC * VB * STAGE / 16; i += NTHR)
        reinterpret_cast<uint4*>(smem + Ge::OFF_V)[i] = make_uint4(0u, 0u, 0u, 0u);
    // programmatic dependent launch: dispatched early, nothing is read before the
    // preceding kernel in the stream has completed and flushed
    asm volatile("griddepcontrol.wait;\n" ::: "memory");
    asm volatile("griddepcontrol.launch_dependents;\n" ::: "memory");
    __syncthreads();

    long long* trace = nullptr;
    long long gl = 0;     // loader: groups issued so far (all slots)
    long long mg = warp;  // compute warp: its next group (groups g with g % NC == warp)
    for (int slot = blockIdx.y; slot < vp.slots; slot += gridDim.y) {
        trace = p.tot_trace ? p.tot_trace + ((size_t)slot * nb + blk) * 64 : nullptr;
        if (trace && tid == 0) trace[0] = lvk2::gtimer();
        int* ctl = vp.qctl + (size_t)slot * 4;
        unsigned* qe = vp.qent + (size_t)slot * vp.qcap;
        const int rl = p.r_log2;
        const int tpc_l2 = rl - 4;  // log2(16-key blocks per cell)
        if (tid == 0) {
            iscr[0] = 0;
            iscr[2] = 0;
        }
        const long long n = __ldcg(&p.ctr->n);
        const long long indexed = __ldcg(&p.ctr->indexed);
        const long long ncells = (n + (1 << rl) - 1) >> rl;
        const long long ntiles = (ncells + 15) >> 4;
        // this CTA's probe tiles: blk, blk + nb, ...
        const int ptiles = ntiles > blk ? (int)((ntiles - blk + nb - 1) / nb) : 0;

        if (loader) {
            // ============================================================ loader
            if (lane == 0) {
                auto take = [&](long long g) {  // wait until stage pair g % SP is free
                    const unsigned sp = (unsigned)(g % SP);
                    const long long use = g / SP;
                    if (use > 0) mbar_wait(emptyb + 8u * sp, (unsigned)((use - 1) & 1));
                    return sp;
                };
                // -- probe groups
                const long long gp0 = gl;
                for (int u = 0; u < ptiles; ++u) {
                    const long long g = gl++;
                    const unsigned sp = take(g);
                    const long long tile = blk + (long long)u * nb;
                    GroupMeta& md = meta[sp];
                    md.type = kProbe;
                    md.a = tile;
                    md.last = (u + NC >= ptiles) ? 1 : 0;  // no later probe group for this warp
                    fence_async();
                    mbar_expect_tx(fullb + 8u * sp, 2 * STAGE);
                    const unsigned dst = pool + sp * 2 * STAGE;
                    const int y = (int)((long long)slot * p.cap_cells + tile * 16);
#pragma unroll
                    for (int h = 0; h < 2; ++h)
#pragma unroll
                        for (int pan = 0; pan < NPAN; ++pan)
                            tma2d(dst + h * STAGE + pan * 2048, &vp.smap, (h * NPAN + pan) * 64, y, fullb + 8u * sp);
                }
                (void)gp0;
                if (trace) trace[13] = lvk2::gtimer();
                // -- key groups: pairs of 16-key blocks from the slot's queue
                const int qcap = vp.qcap;
                bool pdone_sent = false;
                auto maybe_pdone = [&]() {
                    if (!pdone_sent && ld_volatile_s(iscr + 2) >= ptiles) {
                        __threadfence();
                        red_release(ctl + 2, 1);  // this CTA's survivors are all in the queue
                        pdone_sent = true;
                    }
                };
                // claims run CQ pairs ahead and their entries are read EQ pairs ahead, so the
                // atomic and load round trips overlap the issue of earlier groups. The rings are
                // indexed by compile-time step numbers (the loop body is unrolled CQ times): a
                // register that still awaits its load is never copied, which would stall.
                constexpr int CQ = 8, EQ = 4;
                int cq[CQ];
                unsigned eqa[CQ], eqb[CQ];
#pragma unroll
                for (int k = 0; k < CQ; ++k) cq[k] = atomicAdd(ctl + 1, 2);
                auto ld_entry = [&](int c) { return c < qcap ? ld_relaxed(qe + c) : 0xffffffffu; };
#pragma unroll
                for (int k = 0; k < EQ; ++k) {
                    eqa[k] = ld_entry(cq[k]);
                    eqb[k] = ld_entry(cq[k] + 1);
                }
                bool stop = false;
                const long long gk0 = gl;
                // one key group from claim slot J; returns true at the end of the queue
#define LV11_STEP(J)                                                                                         \
    {                                                                                                          \
        maybe_pdone();                                                                                         \
        const int c = cq[J];                                                                                   \
        unsigned e0 = eqa[J], e1 = eqb[J];                                                                     \
        bool end0 = c >= qcap, end1 = c + 1 >= qcap;                                                           \
        while ((e0 == 0 && !end0) || (e1 == 0 && !end1)) { /* not published yet, or past the end */          \
            maybe_pdone();                                                                                     \
            const int pd = ld_acquire(ctl + 2);                                                                \
            if (pd >= nb) { /* every survivor of the team is reserved: qres is final */                       \
                const int qr = ld_relaxed_i(ctl + 0);                                                          \
                if (c >= qr) end0 = true;                                                                      \
                if (c + 1 >= qr) end1 = true;                                                                  \
            }                                                                                                  \
            if (e0 == 0 && !end0) e0 = ld_relaxed(qe + c);                                                     \
            if (e1 == 0 && !end1) e1 = ld_relaxed(qe + c + 1);                                                 \
            if ((e0 == 0 && !end0) || (e1 == 0 && !end1)) __nanosleep(32);                                     \
        }                                                                                                      \
        if (end0) {                                                                                            \
            stop = true;                                                                                       \
        } else {                                                                                               \
            st_relaxed(qe + c, 0u); /* consumed: the queue is left empty for the next launch */                \
            if (!end1) st_relaxed(qe + c + 1, 0u);                                                             \
            const long long g = gl++;                                                                          \
            if (trace && g - gk0 < 16) trace[16 + g - gk0] = lvk2::gtimer();                                   \
            const unsigned sp = take(g);                                                                       \
            GroupMeta& md = meta[sp];                                                                          \
            md.type = kKeys;                                                                                   \
            md.a = (long long)(e0 - 1) << 4;                                                                   \
            md.b = end1 ? -1 : (long long)(e1 - 1) << 4;                                                       \
            fence_async();                                                                                     \
            mbar_expect_tx(fullb + 8u * sp, (end1 ? 1 : 2) * STAGE);                                           \
            const unsigned dst = pool + sp * 2 * STAGE;                                                        \
            _Pragma("unroll") for (int pan = 0; pan < NPAN; ++pan)                                             \
                tma2d(dst + pan * 2048, &vp.kmap, pan * 64, (int)((long long)slot * p.cap + md.a), fullb + 8u * sp); \
            if (!end1) {                                                                                       \
                _Pragma("unroll") for (int pan = 0; pan < NPAN; ++pan)                                         \
                    tma2d(dst + STAGE + pan * 2048, &vp.kmap, pan * 64, (int)((long long)slot * p.cap + md.b), \
                          fullb + 8u * sp);                                                                    \
            }                                                                                                  \
            if (end1) {                                                                                        \
                stop = true;                                                                                   \
            } else {                                                                                           \
                cq[J] = atomicAdd(ctl + 1, 2);                                                                 \
                eqa[(J + EQ) % CQ] = ld_entry(cq[(J + EQ) % CQ]);                                              \
                eqb[(J + EQ) % CQ] = ld_entry(cq[(J + EQ) % CQ] + 1);                                          \
            }                                                                                                  \
        }                                                                                                      \
    }                                                                                                          \
    if (stop) break;
                for (;;) {
                    LV11_STEP(0)
                    LV11_STEP(1)
                    LV11_STEP(2)
                    LV11_STEP(3)
                    LV11_STEP(4)
                    LV11_STEP(5)
                    LV11_STEP(6)
                    LV11_STEP(7)
                }
#undef LV11_STEP
                while (!pdone_sent) maybe_pdone();
                if (trace) trace[14] = lvk2::gtimer();
                // -- one DONE group per compute warp
                for (int k = 0; k < NC; ++k) {
                    const long long g = gl++;
                    const unsigned sp = take(g);
                    meta[sp].type = kDone;
                    mbar_arrive(fullb + 8u * sp);
                }
            }
            gl = __shfl_sync(0xffffffffu, gl, 0);
            __syncwarp();
        } else {
            // ============================================================ compute warps
            // ---- setup: q, S_g, thresholds, B fragments (compute warps only: named barrier 1)
            {
                const float* qsrc = p.q + (size_t)slot * G * DP;
                const float* colmax = p.colmax + (size_t)slot * DP;
                constexpr int CTH = NC * 32;
                constexpr int QPT = (G * DP + CTH - 1) / CTH;
                float xq[QPT], xc[QPT];
#pragma unroll
                for (int k = 0; k < QPT; ++k) {
                    const int i = tid + k * CTH;
                    xq[k] = i < G * DP ? __ldcg(qsrc + i) : 0.0f;
                    xc[k] = i < G * DP ? __ldcg(colmax + i % DP) : 0.0f;
                }
                const float tau_r = tid < G ? __ldcg(p.tau + (size_t)slot * G + tid) : 0.0f;
                for (int i = tid; i < (Ge::SZ_FRE + Ge::SZ_FRP) / 16; i += CTH)
                    reinterpret_cast<uint4*>(smem + Ge::OFF_FRE)[i] = make_uint4(0u, 0u, 0u, 0u);
                float s[G];
#pragma unroll
                for (int g = 0; g < G; ++g) s[g] = 0.0f;
#pragma unroll
                for (int k = 0; k < QPT; ++k) {
                    const int i = tid + k * CTH;
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
                asm volatile("bar.sync 1, %0;\n" ::"n"(CTH) : "memory");
                if (tid < G) {
                    float v = 0.0f;
                    for (int w = 0; w < NC; ++w) v = __fadd_ru(v, red[w * G + tid]);
                    tau_s[tid] = tau_r;
                    taup_s[tid] = __fsub_rd(tau_r, __fmul_ru(v, 2.44140625e-4f));  // 2^-12 S
                    marg_s[tid] = __fmul_ru(v, 1.220703125e-4f);                   // 2^-13 S
                }
                unsigned short* fe = reinterpret_cast<unsigned short*>(fre);
                unsigned short* fp = reinterpret_cast<unsigned short*>(frp);
#pragma unroll
                for (int k = 0; k < QPT; ++k) {
                    const int i = tid + k * CTH;
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
                asm volatile("bar.sync 1, %0;\n" ::"n"(CTH) : "memory");
            }
            if (trace && tid == 0) trace[1] = lvk2::gtimer();

            const int g_me = lane % G;
            const float tau_me = tau_s[g_me], marg_me = marg_s[g_me];
            const float* q_me = qf + g_me * (DP + 4);
            const float scale = p.scale;
            float taup[G];
#pragma unroll
            for (int g = 0; g < G; ++g) taup[g] = taup_s[g];
            const __nv_bfloat16* Vs = reinterpret_cast<const __nv_bfloat16*>(p.V) + (size_t)slot * p.cap * DP;

            float o[MT][4];
#pragma unroll
            for (int mt = 0; mt < MT; ++mt) o[mt][0] = o[mt][1] = o[mt][2] = o[mt][3] = 0.0f;
            float mrun = -INFINITY, lpart = 0.0f;
            int my_sel = 0, my_att = 0, ntask = 0;
            unsigned long long t_keys = 0, t_vals = 0;
            // tasks t-2 (A) and t-1 (B) await their V fold: P fragments, any rows, alpha (the
            // factor from the previous task's frame to their own)
            unsigned pbA[4] = {0u, 0u, 0u, 0u}, pbB[4] = {0u, 0u, 0u, 0u};
            bool pendA = false, pendB = false;
            float alphaA = 1.0f, alphaB = 1.0f;
            // probe survivors wait one group for their queue reservation (atomic result)
            unsigned pend_m = 0;
            long long pend_t = 0;
            int pend_base = 0;
            auto write_entries = [&]() {
                if (!pend_m) return;
                const int base = __shfl_sync(0xffffffffu, pend_base, 0);
                if ((pend_m >> lane) & 1u) {
                    const int idx = __popc(pend_m & ((1u << lane) - 1u)) << tpc_l2;
                    const unsigned b0 = (unsigned)(((pend_t * 16 + lane) << tpc_l2) + 1);
                    for (int sb = 0; sb < (1 << tpc_l2); ++sb) st_relaxed(qe + base + idx + sb, b0 + sb);
                }
                pend_m = 0;
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
            // fold task u's V: move o to u's frame (alpha_u), then o += V(u) P(u)
            auto fold = [&](int u, const unsigned (&pb)[4], bool any, float alpha) {
                rescale(alpha);
                __syncwarp();
                if (any) {
                    const unsigned vb = vbuf + (u % VB) * STAGE;
#pragma unroll
                    for (int mt = 0; mt < MT; ++mt) {
                        unsigned a[4];
                        ldsm4t(a, vb + swz(v_row, 2 * mt + v_hi));
                        mma16816(o[mt], a, pb[0], pb[1]);
                        mma16816(o[mt], a, pb[2], pb[3]);
                    }
                }
            };
            // one 16-key task from a staged block: scores, classify, softmax, V gather, fold
            auto task = [&](unsigned sb, long long k0) {
                float acc2[2][NT][4];
#pragma unroll
                for (int cc = 0; cc < 2; ++cc)
#pragma unroll
                    for (int nt = 0; nt < NT; ++nt) acc2[cc][nt][0] = acc2[cc][nt][1] = acc2[cc][nt][2] = acc2[cc][nt][3] = 0.0f;
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
#pragma unroll
                for (int nt = 0; nt < NT; ++nt) {
                    const int rw = lane >> 2, col = nt * 8 + 2 * q4;
                    *reinterpret_cast<float2*>(ct + rw * CT + col) =
                        make_float2(acc2[0][nt][0] + acc2[1][nt][0], acc2[0][nt][1] + acc2[1][nt][1]);
                    *reinterpret_cast<float2*>(ct + (rw + 8) * CT + col) =
                        make_float2(acc2[0][nt][2] + acc2[1][nt][2], acc2[0][nt][3] + acc2[1][nt][3]);
                }
                __syncwarp();
                float s[PPL];
                unsigned und = 0, selb = 0;
#pragma unroll
                for (int jj = 0; jj < PPL; ++jj) {
                    const int pi = lane + 32 * jj, rw = pi / G;
                    const float* cr = ct + (rw < 16 ? rw : 15) * CT;
                    const float sc = (cr[g_me] + cr[G + g_me]) + cr[2 * G + g_me];
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
                unsigned amask = 0;
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
                    if (mloc > mrun + 8.0f) {  // lazy rescale: weights stay <= e^8
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
                __syncwarp();
                // V rows of the attended keys into this task's V buffer (same row positions)
                if (amask) {
                    constexpr int RPI = 32 / CPR;
                    const unsigned vb = vbuf + (ntask % VB) * STAGE;
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
                        if (rsel >= 0) cpa16(vb + swz(rsel, cc), vsrc + rsel * RB);
                    }
                }
                asm volatile("cp.async.commit_group;\n" ::: "memory");
                if (ntask >= 2) {  // V(t-2) has landed (V(t-1), V(t) may pend)
                    asm volatile("cp.async.wait_group 2;\n" ::: "memory");
                    fold(ntask - 2, pbA, pendA, alphaA);
                }
#pragma unroll
                for (int e = 0; e < 4; ++e) {
                    pbA[e] = pbB[e];
                    pbB[e] = nbf[e];
                }
                pendA = pendB;
                pendB = amask != 0;
                alphaA = alphaB;
                alphaB = alpha;
                ++ntask;
            };

            int ngrp = 0;
            for (;; mg += NC) {
                const unsigned sp = (unsigned)(mg % SP);
                if (trace && warp == 0 && lane == 0 && ngrp < 16) trace[32 + ngrp] = lvk2::gtimer();
                mbar_wait(fullb + 8u * sp, (unsigned)((mg / SP) & 1));
                if (trace && warp == 0 && lane == 0 && ngrp < 16) trace[48 + ngrp] = lvk2::gtimer();
                ++ngrp;
                const GroupMeta md = meta[sp];
                const unsigned sbase = pool + sp * 2 * STAGE;
                if (md.type == kDone) {
                    __syncwarp();
                    if (lane == 0) mbar_arrive(emptyb + 8u * sp);
                    mg += NC;
                    break;
                }
                if (md.type == kProbe) {
                    const long long tile = md.a;
                    float acc2[2][NTP][4];
#pragma unroll
                    for (int cc = 0; cc < 2; ++cc)
#pragma unroll
                        for (int nt = 0; nt < NTP; ++nt) acc2[cc][nt][0] = acc2[cc][nt][1] = acc2[cc][nt][2] = acc2[cc][nt][3] = 0.0f;
#pragma unroll
                    for (int h = 0; h < 2; ++h) {
                        const uint2* fh = frp + h * KS * NTP * 32;
#pragma unroll
                        for (int ks = 0; ks < KS; ++ks) {
                            unsigned a[4];
                            ldsm4(a, sbase + h * STAGE + swz(a_row, 2 * ks + a_hi));
#pragma unroll
                            for (int nt = 0; nt < NTP; ++nt) {
                                const uint2 b = fh[(ks * NTP + nt) * 32 + lane];
                                mma16816(acc2[ks & 1][nt], a, b.x, b.y);
                            }
                        }
                    }
                    __syncwarp();
                    if (lane == 0) mbar_arrive(emptyb + 8u * sp);  // the tile is in registers
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
                    write_entries();  // the previous probe group's reservation has returned
                    if (m) {
                        if (lane == 0) pend_base = atomicAdd(ctl + 0, __popc(m) << tpc_l2);
                        pend_m = m;
                        pend_t = tile;
                    }
                    if (md.last) write_entries();  // nothing later would publish them
                    __syncwarp();
                    if (lane == 0) atomicAdd(iscr + 2, 1);  // tile published (read by the loader)
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
                    continue;
                }
                // kKeys: one or two 16-key tasks
                task(sbase, md.a);
                if (md.b >= 0) task(sbase + STAGE, md.b);
                __syncwarp();
                if (lane == 0) mbar_arrive(emptyb + 8u * sp);
            }
            // the last two tasks' V
            if (ntask >= 2) {
                asm volatile("cp.async.wait_group 1;\n" ::: "memory");
                fold(ntask - 2, pbA, pendA, alphaA);
            }
            if (ntask >= 1) {
                asm volatile("cp.async.wait_group 0;\n" ::: "memory");
                fold(ntask - 1, pbB, pendB, alphaB);
            }
            if (trace && warp == 0 && lane == 0) trace[4] = lvk2::gtimer();
            if (lane == 0) atomicAdd(iscr + 0, ntask);

            // ---- statistics: lanes with the same g = lane % G hold that head's counts
            if (p.counts) {
                int s0 = my_sel, s1 = my_att;
#pragma unroll
                for (int of = 16; of >= G; of >>= 1) {
                    s0 += __shfl_xor_sync(0xffffffffu, s0, of);
                    s1 += __shfl_xor_sync(0xffffffffu, s1, of);
                }
                if (lane < G) {
                    int* cnt = p.counts + ((size_t)slot * G + lane) * 4;
                    if (s0) atomicAdd(cnt + 0, s0);
                    if (s1) atomicAdd(cnt + 1, s1);
                }
            }
            if (p.totals && lane == 0) {
                if (t_keys) atomicAdd(p.totals + 2, t_keys);
                if (t_vals) atomicAdd(p.totals + 3, t_vals);
            }
#pragma unroll
            for (int of = 16; of >= G; of >>= 1) lpart += __shfl_xor_sync(0xffffffffu, lpart, of);
            // warp partial (m, l, o) into the V buffers area (this warp's own)
            constexpr int Wd = G * (DP + 2);
            static_assert(Wd * 4 <= VB * STAGE, "warp partial must fit the V buffers");
            float* w = reinterpret_cast<float*>(smem + Ge::OFF_V + warp * VB * STAGE);
            if (lane < G) {
                w[lane * (DP + 2)] = mrun;
                w[lane * (DP + 2) + 1] = lpart;
            }
#pragma unroll
            for (int mt = 0; mt < MT; ++mt) {
#pragma unroll
                for (int e = 0; e < 4; ++e) {
                    const int h = 2 * q4 + (e & 1), cc = 16 * mt + (lane >> 2) + 8 * (e >> 1);
                    if (h < G) w[h * (DP + 2) + 2 + cc] = o[mt][e];
                }
            }
        }

        // ---- warp partials -> CTA partial [G][DP+2] (m, l, o)
        constexpr int Wd = G * (DP + 2);
        float* shw = red;  // [NC][G] weights
        __syncthreads();
        if (trace && tid == 0) {
            trace[5] = lvk2::gtimer();
            trace[15] = iscr[0];
        }
        auto wpart = [&](int w) { return reinterpret_cast<const float*>(smem + Ge::OFF_V + w * VB * STAGE); };
        float* part = p.partial_ws + ((size_t)slot * nb + blk) * Wd;
        if (tid < G) {
            float mm = -INFINITY;
            for (int w = 0; w < NC; ++w) mm = fmaxf(mm, wpart(w)[tid * (DP + 2)]);
            float l = 0.0f;
            for (int w = 0; w < NC; ++w) {
                const float mw = wpart(w)[tid * (DP + 2)];
                const float a = mw == -INFINITY ? 0.0f : __expf(mw - mm);
                shw[w * G + tid] = a;
                l += a * wpart(w)[tid * (DP + 2) + 1];
            }
            part[tid * (DP + 2)] = l > 0.0f ? mm : -INFINITY;
            part[tid * (DP + 2) + 1] = l;
        }
        __syncthreads();
        for (int i = tid; i < G * DP; i += NTHR) {
            const int g = i / DP, c = i % DP;
            float s = 0.0f;
#pragma unroll
            for (int w = 0; w < NC; ++w) s = fmaf(shw[w * G + g], wpart(w)[g * (DP + 2) + 2 + c], s);
            part[g * (DP + 2) + 2 + c] = s;
        }
        if (trace && tid == 0) trace[6] = lvk2::gtimer();

        // ---- the last CTA of the team merges the nb partials (one round trip for all of them)
        int* ticket = ctl + 3;
        __syncthreads();
        if (tid == 0) iscr[1] = atom_add_acq_rel(ticket, 1) == nb - 1;
        __syncthreads();
        if (iscr[1]) {
            if (trace && tid == 0) trace[8] = lvk2::gtimer();
            const float* src = p.partial_ws + (size_t)slot * nb * Wd;
            // scratch over the stage pool (idle now): M[G], L[G], weights [nb][G], then the partials
            float* M = reinterpret_cast<float*>(smem + Ge::OFF_POOL);
            float* L = M + G;
            float* wgt = M + 2 * G;
            float* stg = wgt + ((nb * G + 3) / 4) * 4;  // 16-byte aligned
            constexpr int EPT = (G * DP + NTHR - 1) / NTHR;
            const int per_chunk = (SP * 2 * STAGE - (2 * G + nb * G + 4) * 4) / (Wd * 4);
            float accr[EPT];
#pragma unroll
            for (int k = 0; k < EPT; ++k) accr[k] = 0.0f;
            for (int s0 = 0; s0 < nb; s0 += per_chunk) {
                const int cnt = nb - s0 < per_chunk ? nb - s0 : per_chunk;
                const float2* cs = reinterpret_cast<const float2*>(src + (size_t)s0 * Wd);
                for (int i = tid; i < cnt * Wd / 2; i += NTHR) reinterpret_cast<float2*>(stg)[i] = __ldcg(cs + i);
                __syncthreads();
                if (s0 == 0) {
                    if (trace && tid == 0) trace[11] = lvk2::gtimer();
                    // per-head max and weights over all nb partials (headers from the staged copy
                    // when every partial fits one chunk, else from global)
                    const bool one = cnt == nb;
                    auto hdr = [&](int s2, int g, int k) {
                        return one ? stg[s2 * Wd + g * (DP + 2) + k] : __ldcg(src + (size_t)s2 * Wd + g * (DP + 2) + k);
                    };
                    for (int g = warp; g < G; g += NW) {
                        float mm = -INFINITY;
                        for (int s2 = lane; s2 < nb; s2 += 32) mm = fmaxf(mm, hdr(s2, g, 0));
#pragma unroll
                        for (int o2 = 16; o2 > 0; o2 >>= 1) mm = fmaxf(mm, __shfl_xor_sync(0xffffffffu, mm, o2));
                        float l = 0.0f;
                        for (int s2 = lane; s2 < nb; s2 += 32) {
                            const float ms = hdr(s2, g, 0);
                            const float wv = ms == -INFINITY ? 0.0f : __expf(ms - mm);
                            wgt[s2 * G + g] = wv;
                            l += wv * hdr(s2, g, 1);
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
                    if (i < G * DP) {
                        const int g = i / DP, c = i % DP;
                        float a = accr[k];
#pragma unroll 4
                        for (int s2 = 0; s2 < cnt; ++s2) a = fmaf(wgt[(s0 + s2) * G + g], stg[s2 * Wd + g * (DP + 2) + 2 + c], a);
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
            if (tid < 4) ctl[tid] = 0;  // reserved, claimed, CTAs probed, ticket: ready for the next launch
            if (trace && tid == 0) trace[7] = lvk2::gtimer();
        }
        __syncthreads();
        // the V buffers held partials: zero them again for the next slot
        for (int i = tid; i < NC * VB * STAGE / 16; i += NTHR)
            reinterpret_cast<uint4*>(smem + Ge::OFF_V)[i] = make_uint4(0u, 0u, 0u, 0u);
        __syncthreads();
    }
}

cudaError_t launch_layer_v11(int DP, int G, const V10Params& vp, int sms, cudaStream_t st, int* geo);

}  // namespace lvk11
