// sm_100a kernels of the Louver decode hot path.
//
// HBM layout of one layer (lv_ctx), per slot = (sequence b, kv head h):
//   K, V    [slot][cap][DP]            T (fp32 or bf16), rows zero-padded d -> DP
//   lo, hi  [slot][DP][cap_cells]      T, coordinate-major cell AABBs (cell = r
//                                       contiguous keys), so the probe streams
//                                       each coordinate's bounds coalesced
//   colmax  [slot][DP]                 fp32, max |k_c| over stored keys (slack)
//   counters {n, indexed, flushes}     int64, uniform over slots, on device
// q / out are [batch][H_q][DP] fp32 with q head hq = h*G + g.
//
// The query kernel is one fused pass per (slot, split of the sequence):
//   probe    per-cell bound  sum_c max(q_c lo_c, q_c hi_c)  for the G q heads
//            of the kv head (one summary read serves all G), vs tau - slack;
//            survivors compacted with warp ballots
//   exact    keys of surviving cells staged into shared memory with 16-byte
//            cp.async (padded rows, conflict-free LDS.128), one thread per
//            (key, q head) runs the normative dot (core.hpp:17-21): sequential
//            __fmul_rn/__fadd_rn, never contracted into FMA
//   attend   online softmax over selected ∪ buffer (cache.cpp:48-68): V rows
//            gathered once per kv head, weights per q head
//   combine  per-split (m, l, o) partials; the last CTA of a slot merges them
#pragma once

#include <cuda_bf16.h>
#include <cuda_runtime.h>
#include <stdint.h>

namespace lvk {

constexpr int kThreads = 256;
constexpr int kWarps = kThreads / 32;
constexpr int kChunk = 512;          // keys per probe/exact/attend chunk
constexpr int kChunkWords = kChunk / 32;
constexpr int kStageBudget = 36864;  // bytes per key-staging buffer (x2)

enum Mode { kQuery = 0, kBrute = 1, kDense = 2 };

struct Counters {
    long long n;
    long long indexed;
    long long flushes;
    long long pad;
};

struct QueryParams {
    const void* K;
    const void* V;
    const void* lo;
    const void* hi;
    const float* colmax;
    const float* q;
    const float* tau;
    const Counters* ctr;
    long long cap;
    long long cap_cells;
    long long limit;        // kBrute: ids < limit; otherwise ignored (uses n)
    int r_log2;
    int chunks_per_split;
    int splits;
    int strict;
    int d_true;
    float scale;
    float* partial_ws;      // [slots][splits][G][DP+2]
    int* tickets;           // [slots]
    float* out;             // [slots*G][DP] or null
    float* partial_out;     // [slots*G][DP+2] or null
    unsigned* bits;         // [slots*G][bits_words] or null
    long long bits_words;
    int* counts;            // [slots*G][4] or null
    unsigned long long* totals;  // [4] or null
    long long* tot_trace;        // debug: per-CTA phase timestamps (bf16 cell stream) or null
    unsigned* cand_bits;         // [slots][bits_words] candidate keys (indexed keys of surviving cells) or null
};

template <typename T>
struct Elt;
template <>
struct Elt<float> {
    static constexpr int kPer16 = 4;
};
template <>
struct Elt<__nv_bfloat16> {
    static constexpr int kPer16 = 8;
};

template <typename T, int DP, int G>
struct Geo {
    static constexpr int EPC = Elt<T>::kPer16;
    static constexpr int CPR = DP / EPC;                       // 16-B chunks per row
    static constexpr int ROWB = DP * (int)sizeof(T);
    static constexpr int PITCH = ROWB + 16;                    // conflict-free LDS.128
    static constexpr int NK0 = kThreads / G;
    static constexpr int NKB = (kStageBudget / PITCH) & ~7;
    static constexpr int NK = NK0 < NKB ? NK0 : NKB;           // keys per exact round
    static constexpr int QP = DP + 4;                          // padded q row (floats)
    static constexpr int VPL = DP / 32;                        // V elements per lane

    // dynamic shared memory layout (bytes)
    static constexpr int OFF_STAGE = 0;
    static constexpr int SZ_SC = kChunk * G * 4;
    static constexpr int SZ_STAGE0 = 2 * NK * PITCH;
    static constexpr int SZ_RED = kWarps * G * DP * 4;         // final cross-warp (l, o) reduction
    static constexpr int SZ_STAGE = SZ_STAGE0 + SZ_SC >= SZ_RED ? SZ_STAGE0 : SZ_RED - SZ_SC;
    static constexpr int OFF_SC = OFF_STAGE + SZ_STAGE;        // scores / probe partials
    static constexpr int OFF_Q = OFF_SC + SZ_SC;               // q, q+, q-
    static constexpr int SZ_Q = 3 * G * QP * 4;
    static constexpr int OFF_MISC = OFF_Q + SZ_Q;              // tau_eff, running max, ...
    static constexpr int SZ_MISC = 16 * G * 4 + 160 * 4;
    static constexpr int OFF_CELL = OFF_MISC + SZ_MISC;        // cell masks (u8)
    static constexpr int SZ_CELL = kChunk;
    static constexpr int OFF_SURV = OFF_CELL + SZ_CELL;        // survivor cells (u16)
    static constexpr int SZ_SURV = kChunk * 2;
    static constexpr int OFF_ALIST = OFF_SURV + SZ_SURV;       // attended keys (u16)
    static constexpr int SZ_ALIST = kChunk * 2;
    static constexpr int OFF_AMASK = OFF_ALIST + SZ_ALIST;     // per-key attend bits (u8)
    static constexpr int SZ_AMASK = kChunk;
    static constexpr int OFF_SELW = OFF_AMASK + SZ_AMASK;      // selected bitmap words
    static constexpr int SZ_SELW = G * kChunkWords * 4;
    static constexpr int SMEM = OFF_SELW + SZ_SELW;

    static_assert(DP % 32 == 0 && DP >= 64 && DP <= 256, "DP");
    static_assert(kWarps * G * DP * 4 <= SZ_STAGE + SZ_SC, "final reduction must fit");
};

// ------------------------------------------------------------------ helpers

__device__ __forceinline__ float bf_lo(uint32_t w) { return __uint_as_float(w << 16); }
__device__ __forceinline__ float bf_hi(uint32_t w) { return __uint_as_float(w & 0xffff0000u); }

template <typename T>
__device__ __forceinline__ void unpack16(const uint4& v, float* f);
template <>
__device__ __forceinline__ void unpack16<float>(const uint4& v, float* f) {
    f[0] = __uint_as_float(v.x);
    f[1] = __uint_as_float(v.y);
    f[2] = __uint_as_float(v.z);
    f[3] = __uint_as_float(v.w);
}
template <>
__device__ __forceinline__ void unpack16<__nv_bfloat16>(const uint4& v, float* f) {
    f[0] = bf_lo(v.x);
    f[1] = bf_hi(v.x);
    f[2] = bf_lo(v.y);
    f[3] = bf_hi(v.y);
    f[4] = bf_lo(v.z);
    f[5] = bf_hi(v.z);
    f[6] = bf_lo(v.w);
    f[7] = bf_hi(v.w);
}

__device__ __forceinline__ float elt_f(const float* p) { return __ldg(p); }
__device__ __forceinline__ float elt_f(const __nv_bfloat16* p) {
    return __uint_as_float((unsigned)__ldg(reinterpret_cast<const unsigned short*>(p)) << 16);
}

// Two consecutive cells' bound arrays at one coordinate.
template <typename T>
__device__ __forceinline__ float2 load_pair(const T* p);
template <>
__device__ __forceinline__ float2 load_pair<float>(const float* p) {
    return __ldg(reinterpret_cast<const float2*>(p));
}
template <>
__device__ __forceinline__ float2 load_pair<__nv_bfloat16>(const __nv_bfloat16* p) {
    const uint32_t w = __ldg(reinterpret_cast<const unsigned int*>(p));
    return make_float2(bf_lo(w), bf_hi(w));
}

// V row slice owned by one lane: VPL consecutive elements at lane*VPL.
template <typename T, int VPL>
__device__ __forceinline__ void load_vslice(const T* row, int lane, float* f);
template <>
__device__ __forceinline__ void load_vslice<float, 2>(const float* row, int lane, float* f) {
    const float2 v = __ldg(reinterpret_cast<const float2*>(row) + lane);
    f[0] = v.x;
    f[1] = v.y;
}
template <>
__device__ __forceinline__ void load_vslice<float, 4>(const float* row, int lane, float* f) {
    const float4 v = __ldg(reinterpret_cast<const float4*>(row) + lane);
    f[0] = v.x;
    f[1] = v.y;
    f[2] = v.z;
    f[3] = v.w;
}
template <>
__device__ __forceinline__ void load_vslice<float, 8>(const float* row, int lane, float* f) {
    const float4 a = __ldg(reinterpret_cast<const float4*>(row) + 2 * lane);
    const float4 b = __ldg(reinterpret_cast<const float4*>(row) + 2 * lane + 1);
    f[0] = a.x; f[1] = a.y; f[2] = a.z; f[3] = a.w;
    f[4] = b.x; f[5] = b.y; f[6] = b.z; f[7] = b.w;
}
template <>
__device__ __forceinline__ void load_vslice<__nv_bfloat16, 2>(const __nv_bfloat16* row, int lane,
                                                              float* f) {
    const uint32_t w = __ldg(reinterpret_cast<const unsigned int*>(row) + lane);
    f[0] = bf_lo(w);
    f[1] = bf_hi(w);
}
template <>
__device__ __forceinline__ void load_vslice<__nv_bfloat16, 4>(const __nv_bfloat16* row, int lane,
                                                              float* f) {
    const uint2 w = __ldg(reinterpret_cast<const uint2*>(row) + lane);
    f[0] = bf_lo(w.x);
    f[1] = bf_hi(w.x);
    f[2] = bf_lo(w.y);
    f[3] = bf_hi(w.y);
}
template <>
__device__ __forceinline__ void load_vslice<__nv_bfloat16, 8>(const __nv_bfloat16* row, int lane,
                                                              float* f) {
    const uint4 w = __ldg(reinterpret_cast<const uint4*>(row) + lane);
    unpack16<__nv_bfloat16>(w, f);
}

__device__ __forceinline__ void cp_async16(void* smem, const void* gmem) {
    const unsigned s = static_cast<unsigned>(__cvta_generic_to_shared(smem));
    asm volatile("cp.async.cg.shared.global [%0], [%1], 16;\n" ::"r"(s), "l"(gmem));
}
__device__ __forceinline__ void cp_async_commit() { asm volatile("cp.async.commit_group;\n" ::); }
template <int N>
__device__ __forceinline__ void cp_async_wait() {
    asm volatile("cp.async.wait_group %0;\n" ::"n"(N));
}

__device__ __forceinline__ float warp_max(float v) {
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) v = fmaxf(v, __shfl_xor_sync(0xffffffffu, v, o));
    return v;
}
__device__ __forceinline__ int warp_sum_int(int v) {
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
    return v;
}

// Block-wide ordered compaction of flags over `count` items (count <= kChunk):
// writes the indices i with flag(i) into list[] in ascending order and returns
// the total. `scratch` holds kWarps+1 ints. Must be called by all threads.
template <typename Flag>
__device__ __forceinline__ int block_compact(int count, Flag flag, unsigned short* list,
                                             int* scratch) {
    const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
    int base = 0;
    for (int start = 0; start < count; start += kThreads) {
        const int i = start + tid;
        const bool f = i < count && flag(i);
        const unsigned bal = __ballot_sync(0xffffffffu, f);
        if (lane == 0) scratch[warp] = __popc(bal);
        __syncthreads();
        int off = 0, tot = 0;
#pragma unroll
        for (int w = 0; w < kWarps; ++w) {
            const int c = scratch[w];
            off += w < warp ? c : 0;
            tot += c;
        }
        if (f) list[base + off + __popc(bal & ((1u << lane) - 1u))] = static_cast<unsigned short>(i);
        base += tot;
        __syncthreads();
    }
    return base;
}

// ------------------------------------------------------------ query kernel

template <typename T, int DP, int G, int MODE>
__global__ void __launch_bounds__(kThreads) louver_query_kernel(const QueryParams p) {
    using Ge = Geo<T, DP, G>;
    extern __shared__ __align__(128) unsigned char smem[];
    unsigned char* stage = smem + Ge::OFF_STAGE;
    float* sc = reinterpret_cast<float*>(smem + Ge::OFF_SC);
    float* qv = reinterpret_cast<float*>(smem + Ge::OFF_Q);
    float* qpos = qv + G * Ge::QP;
    float* qneg = qpos + G * Ge::QP;
    float* misc = reinterpret_cast<float*>(smem + Ge::OFF_MISC);
    float* tau_eff = misc;              // [G]
    float* tau_s = misc + G;            // [G]
    float* run_max = misc + 2 * G;      // [G]
    float* alpha_s = misc + 3 * G;      // [G]
    float* cmax_s = misc + 4 * G;       // [G]  chunk max
    int* iscr = reinterpret_cast<int*>(misc + 16 * G);  // 160 ints
    unsigned char* cellm = smem + Ge::OFF_CELL;
    unsigned short* surv = reinterpret_cast<unsigned short*>(smem + Ge::OFF_SURV);
    unsigned short* alist = reinterpret_cast<unsigned short*>(smem + Ge::OFF_ALIST);
    unsigned char* amask = smem + Ge::OFF_AMASK;
    unsigned* selw = reinterpret_cast<unsigned*>(smem + Ge::OFF_SELW);

    const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
    const int slot = blockIdx.y, split = blockIdx.x;
    const long long n_all = p.ctr->n;
    const long long n = MODE == kBrute ? (p.limit < n_all ? p.limit : n_all) : n_all;
    const long long indexed = MODE == kQuery ? p.ctr->indexed : 0;
    const int r = 1 << p.r_log2;
    const T* Ks = reinterpret_cast<const T*>(p.K) + (size_t)slot * p.cap * DP;
    const T* Vs = reinterpret_cast<const T*>(p.V) + (size_t)slot * p.cap * DP;

    // ---- per-CTA setup: q rows, q+/q-, tau_eff = tau - slack (round down)
    for (int i = tid; i < G * DP; i += kThreads) {
        const int g = i / DP, c = i % DP;
        const float x = p.q[((size_t)slot * G + g) * DP + c];
        qv[g * Ge::QP + c] = x;
        qpos[g * Ge::QP + c] = fmaxf(x, 0.0f);
        qneg[g * Ge::QP + c] = fminf(x, 0.0f);
    }
    if (warp < G) {
        const int g = warp;
        // slack = 2 * gamma_d * sum_c |q_c| * colmax_c  bounds both the probe's
        // summation error and the normative dot's deviation from the exact
        // product; accumulated with upward rounding.
        float s = 0.0f;
        if (MODE == kQuery) {
            for (int c = lane; c < DP; c += 32)
                s = __fadd_ru(s, __fmul_ru(fabsf(p.q[((size_t)slot * G + g) * DP + c]),
                                           p.colmax[(size_t)slot * DP + c]));
#pragma unroll
            for (int o = 16; o > 0; o >>= 1) s = __fadd_ru(s, __shfl_xor_sync(0xffffffffu, s, o));
        }
        if (lane == 0) {
            const float t = p.tau ? p.tau[(size_t)slot * G + g] : -INFINITY;
            const float dd = (float)(DP + 2);
            const float gamma = __fdiv_ru(__fmul_ru(dd, 5.9604645e-08f), 1.0f - dd * 5.9604645e-08f);
            const float slack = __fmul_ru(__fmul_ru(2.0f, gamma), s);
            tau_s[g] = t;
            tau_eff[g] = __fsub_rd(t, __fmul_ru(slack, 1.0009765625f));
            run_max[g] = -INFINITY;
        }
    }

    // running softmax state per warp: o[g][VPL] and l[g] (lane-replicated)
    float o_acc[G][Ge::VPL];
    float l_acc[G];
#pragma unroll
    for (int g = 0; g < G; ++g) {
        l_acc[g] = 0.0f;
#pragma unroll
        for (int e = 0; e < Ge::VPL; ++e) o_acc[g][e] = 0.0f;
    }
    int stat_sel[G], stat_att[G], stat_scan[G];
#pragma unroll
    for (int g = 0; g < G; ++g) stat_sel[g] = stat_att[g] = stat_scan[g] = 0;
    unsigned long long t_cells = 0, t_surv = 0, t_keys = 0, t_vals = 0;
    __syncthreads();

    const long long chunk0 = (long long)split * p.chunks_per_split;
    for (int ci = 0; ci < p.chunks_per_split; ++ci) {
        const long long k0 = (chunk0 + ci) * kChunk;
        if (k0 >= n) break;
        const int nvalid = (int)((n - k0) < kChunk ? (n - k0) : kChunk);
        const int ncells = (nvalid + r - 1) >> p.r_log2;

        for (int i = tid; i < kChunk; i += kThreads) amask[i] = 0;
        for (int i = tid; i < G * kChunkWords; i += kThreads) selw[i] = 0;

        // ------------------------------------------------------------ probe
        const long long idx_end = indexed;  // keys [0, indexed) are indexed
        const bool any_indexed = MODE == kQuery && k0 < idx_end;
        if (any_indexed) {
            const int NC = kChunk >> p.r_log2;
            const int NCP = NC >> 1;
            const int NCPT = NCP < kThreads ? NCP : kThreads;
            const int DG = kThreads / NCPT;
            const int DPG = DP / DG;
            const int pt = tid % NCPT, dg = tid / NCPT;
            // cell-major summaries: row per cell = [hi (DP) | lo (DP)]
            const T* rows = reinterpret_cast<const T*>(p.lo) +
                            ((size_t)slot * p.cap_cells + (size_t)(k0 >> p.r_log2)) * 2 * DP;
            float* red = sc;  // [DG][NC][G]
            for (int pr = pt; pr < NCP; pr += NCPT) {
                float acc0[G], acc1[G];
#pragma unroll
                for (int g = 0; g < G; ++g) acc0[g] = acc1[g] = 0.0f;
                if (2 * pr < ncells) {
                    const T* r0 = rows + (size_t)(2 * pr) * 2 * DP;
                    const T* r1 = r0 + 2 * DP;
                    const int c0 = dg * DPG;
#pragma unroll 8
                    for (int c = c0; c < c0 + DPG; ++c) {
                        const float2 h2 = make_float2(elt_f(r0 + c), elt_f(r1 + c));
                        const float2 l2 = make_float2(elt_f(r0 + DP + c), elt_f(r1 + DP + c));
#pragma unroll
                        for (int g = 0; g < G; ++g) {
                            const float qp = qpos[g * Ge::QP + c], qn = qneg[g * Ge::QP + c];
                            acc0[g] = fmaf(qn, l2.x, fmaf(qp, h2.x, acc0[g]));
                            acc1[g] = fmaf(qn, l2.y, fmaf(qp, h2.y, acc1[g]));
                        }
                    }
                }
#pragma unroll
                for (int g = 0; g < G; ++g) {
                    red[(dg * NC + 2 * pr) * G + g] = acc0[g];
                    red[(dg * NC + 2 * pr + 1) * G + g] = acc1[g];
                }
            }
            __syncthreads();
            for (int cell = tid; cell < NC; cell += kThreads) {
                unsigned char m = 0;
                if (cell < ncells) {
                    const long long cs = k0 + ((long long)cell << p.r_log2);
                    const long long ce = cs + r;  // exclusive
                    if (ce > idx_end) {
                        m = (unsigned char)((1u << G) - 1u) | 0x80u;  // buffer keys inside
                    } else {
#pragma unroll
                        for (int g = 0; g < G; ++g) {
                            float b = 0.0f;
                            for (int q = 0; q < DG; ++q) b += red[(q * NC + cell) * G + g];
                            if (b >= tau_eff[g]) m |= (unsigned char)(1u << g);
                        }
                    }
                    ++t_cells;
                    if (m) ++t_surv;
                    if (p.cand_bits && m) {  // query_ta's live ids: the cell's indexed keys
                        const long long ke = ce < idx_end ? ce : idx_end;
                        for (long long k = cs; k < ke; ++k)
                            atomicOr(p.cand_bits + (size_t)slot * p.bits_words + (k >> 5), 1u << (k & 31));
                    }
#pragma unroll
                    for (int g = 0; g < G; ++g)
                        if (m & (1u << g)) {
                            const long long kend = ce < n ? ce : n;
                            stat_scan[g] += (int)(kend - cs);
                        }
                }
                cellm[cell] = m;
            }
        } else {
            // Dense / brute force / all-buffer chunk: every cell is scanned.
            for (int cell = tid; cell < (kChunk >> p.r_log2); cell += kThreads) {
                unsigned char m = 0;
                if (cell < ncells) {
                    m = (unsigned char)((1u << G) - 1u) | (MODE == kQuery ? 0x80u : 0u);
                    const long long cs = k0 + ((long long)cell << p.r_log2);
                    const long long kend = cs + r < n ? cs + r : n;
#pragma unroll
                    for (int g = 0; g < G; ++g) stat_scan[g] += (int)(kend - cs);
                }
                cellm[cell] = m;
            }
        }
        __syncthreads();

        const int nsurv = block_compact(
            kChunk >> p.r_log2, [&](int i) { return cellm[i] != 0; }, surv, iscr);
        const int nflat = nsurv << p.r_log2;

        // ------------------------------------------------------------ exact
        const int nrounds = (nflat + Ge::NK - 1) / Ge::NK;
        auto issue_round = [&](int rd, int buf) {
            unsigned char* dst = stage + buf * Ge::NK * Ge::PITCH;
            for (int it = tid; it < Ge::NK * Ge::CPR; it += kThreads) {
                const int kr = it / Ge::CPR, c = it % Ge::CPR;
                const int f = rd * Ge::NK + kr;
                if (f >= nflat) continue;
                const int key = ((int)surv[f >> p.r_log2] << p.r_log2) + (f & (r - 1));
                if (key >= nvalid) continue;
                cp_async16(dst + kr * Ge::PITCH + c * 16,
                           reinterpret_cast<const unsigned char*>(Ks + (size_t)(k0 + key) * DP) + c * 16);
            }
            cp_async_commit();
        };
        if (nrounds > 0) issue_round(0, 0);
        for (int rd = 0; rd < nrounds; ++rd) {
            if (rd + 1 < nrounds) {
                issue_round(rd + 1, (rd + 1) & 1);
                cp_async_wait<1>();
            } else {
                cp_async_wait<0>();
            }
            __syncthreads();
            const unsigned char* buf = stage + (rd & 1) * Ge::NK * Ge::PITCH;
            const int kr = tid / G, g = tid % G;
            const int f = rd * Ge::NK + kr;
            if (kr < Ge::NK && f < nflat) {
                const int cell = surv[f >> p.r_log2];
                const int key = (cell << p.r_log2) + (f & (r - 1));
                if (key < nvalid) {
                    const unsigned char* row = buf + kr * Ge::PITCH;
                    const float* qg = qv + g * Ge::QP;
                    float s = 0.0f;
                    if (MODE == kDense) {
#pragma unroll 4
                        for (int c = 0; c < Ge::CPR; ++c) {
                            const uint4 kv = *reinterpret_cast<const uint4*>(row + c * 16);
                            float kf[Ge::EPC];
                            unpack16<T>(kv, kf);
#pragma unroll
                            for (int e = 0; e < Ge::EPC; ++e) s = fmaf(qg[c * Ge::EPC + e], kf[e], s);
                        }
                    } else {
                        // Normative dot: strictly sequential, one rounding per
                        // multiply and per add (core.hpp:17-21).
#pragma unroll 4
                        for (int c = 0; c < Ge::CPR; ++c) {
                            const uint4 kv = *reinterpret_cast<const uint4*>(row + c * 16);
                            float kf[Ge::EPC];
                            unpack16<T>(kv, kf);
#pragma unroll
                            for (int e = 0; e < Ge::EPC; ++e)
                                s = __fadd_rn(s, __fmul_rn(qg[c * Ge::EPC + e], kf[e]));
                        }
                    }
                    sc[key * G + g] = s;
                    const long long gid = k0 + key;
                    const bool selected = MODE == kDense ? true : s >= tau_s[g];
                    const bool in_buffer = MODE == kQuery && gid >= idx_end;
                    const bool attend = MODE == kDense || selected || (in_buffer && !p.strict);
                    if (selected && MODE != kDense) atomicOr(&selw[g * kChunkWords + (key >> 5)], 1u << (key & 31));
                    if (attend) atomicOr(reinterpret_cast<unsigned*>(amask + (key & ~3)),
                                         1u << ((key & 3) * 8 + g));
                    if (g == 0) ++t_keys;
                }
            }
            __syncthreads();
        }

        // selected bitmap words for this chunk
        if (MODE != kDense) {
            for (int i = tid; i < G * kChunkWords; i += kThreads) {
                const int g = i / kChunkWords, w = i % kChunkWords;
                const unsigned v = selw[i];
                stat_sel[g] += __popc(v);
                if (p.bits) {
                    const long long word = (k0 >> 5) + w;
                    if (word < p.bits_words)
                        p.bits[((size_t)slot * G + g) * p.bits_words + word] = v;
                }
            }
        }

        // ------------------------------------------------------------ attend
        if (MODE != kBrute) {
            const int natt = block_compact(
                nvalid, [&](int i) { return amask[i] != 0; }, alist, iscr);
            // chunk max of scaled scores per q head
            float cm[G];
#pragma unroll
            for (int g = 0; g < G; ++g) cm[g] = -INFINITY;
            for (int i = tid; i < natt; i += kThreads) {
                const int key = alist[i];
                const unsigned char m = amask[key];
#pragma unroll
                for (int g = 0; g < G; ++g)
                    if (m & (1u << g)) cm[g] = fmaxf(cm[g], p.scale * sc[key * G + g]);
            }
#pragma unroll
            for (int g = 0; g < G; ++g) {
                const float v = warp_max(cm[g]);
                if (lane == 0) reinterpret_cast<float*>(iscr)[16 + warp * G + g] = v;
            }
            __syncthreads();
            if (tid < G) {
                float v = -INFINITY;
                for (int w = 0; w < kWarps; ++w) v = fmaxf(v, reinterpret_cast<float*>(iscr)[16 + w * G + tid]);
                const float old = run_max[tid];
                const float nm = fmaxf(old, v);
                alpha_s[tid] = old == -INFINITY ? 0.0f : expf(old - nm);
                run_max[tid] = nm;
                cmax_s[tid] = v;
            }
            __syncthreads();
#pragma unroll
            for (int g = 0; g < G; ++g) {
                const float a = alpha_s[g];
                l_acc[g] *= a;
#pragma unroll
                for (int e = 0; e < Ge::VPL; ++e) o_acc[g][e] *= a;
            }
            float mx[G];
#pragma unroll
            for (int g = 0; g < G; ++g) mx[g] = run_max[g];
            // gather V rows: warp w takes attended keys w, w+8, ... (2 in flight)
            int i = warp;
            for (; i + kWarps < natt; i += 2 * kWarps) {
                const int ka = alist[i], kb = alist[i + kWarps];
                float va[Ge::VPL], vb[Ge::VPL];
                load_vslice<T, Ge::VPL>(Vs + (size_t)(k0 + ka) * DP, lane, va);
                load_vslice<T, Ge::VPL>(Vs + (size_t)(k0 + kb) * DP, lane, vb);
                const unsigned char ma = amask[ka], mb = amask[kb];
#pragma unroll
                for (int g = 0; g < G; ++g) {
                    const float pa = (ma & (1u << g)) ? expf(p.scale * sc[ka * G + g] - mx[g]) : 0.0f;
                    const float pb = (mb & (1u << g)) ? expf(p.scale * sc[kb * G + g] - mx[g]) : 0.0f;
                    l_acc[g] += pa + pb;
#pragma unroll
                    for (int e = 0; e < Ge::VPL; ++e) o_acc[g][e] = fmaf(pb, vb[e], fmaf(pa, va[e], o_acc[g][e]));
                }
            }
            for (; i < natt; i += kWarps) {
                const int ka = alist[i];
                float va[Ge::VPL];
                load_vslice<T, Ge::VPL>(Vs + (size_t)(k0 + ka) * DP, lane, va);
                const unsigned char ma = amask[ka];
#pragma unroll
                for (int g = 0; g < G; ++g) {
                    const float pa = (ma & (1u << g)) ? expf(p.scale * sc[ka * G + g] - mx[g]) : 0.0f;
                    l_acc[g] += pa;
#pragma unroll
                    for (int e = 0; e < Ge::VPL; ++e) o_acc[g][e] = fmaf(pa, va[e], o_acc[g][e]);
                }
            }
            if (tid == 0) t_vals += natt;
            for (int j = tid; j < natt; j += kThreads) {
                const unsigned char m = amask[alist[j]];
#pragma unroll
                for (int g = 0; g < G; ++g) stat_att[g] += (m >> g) & 1;
            }
            __syncthreads();
        }
    }

    // ---- statistics
    if (p.counts) {
#pragma unroll
        for (int g = 0; g < G; ++g) {
            const int s0 = warp_sum_int(stat_sel[g]);
            const int s1 = warp_sum_int(stat_att[g]);
            const int s2 = warp_sum_int(stat_scan[g]);
            if (lane == 0) {
                int* c = p.counts + ((size_t)slot * G + g) * 4;
                if (s0) atomicAdd(c + 0, s0);
                if (s1) atomicAdd(c + 1, s1);
                if (s2) atomicAdd(c + 2, s2);
            }
        }
    }
    if (p.totals) {
        unsigned long long a = t_cells, b = t_surv, c = t_keys, d = t_vals;
#pragma unroll
        for (int o = 16; o > 0; o >>= 1) {
            a += __shfl_xor_sync(0xffffffffu, a, o);
            b += __shfl_xor_sync(0xffffffffu, b, o);
            c += __shfl_xor_sync(0xffffffffu, c, o);
            d += __shfl_xor_sync(0xffffffffu, d, o);
        }
        if (lane == 0) {
            if (a) atomicAdd(p.totals + 0, a);
            if (b) atomicAdd(p.totals + 1, b);
            if (c) atomicAdd(p.totals + 2, c);
            if (d) atomicAdd(p.totals + 3, d);
        }
    }
    if (MODE == kBrute) return;

    // ---- cross-warp reduction of (l, o) and the split's partial
    float* fred = reinterpret_cast<float*>(smem);  // [kWarps][G][DP] (stage+sc region)
    float* lred = reinterpret_cast<float*>(iscr) + 16;  // [kWarps][G] (reuse)
    __syncthreads();
#pragma unroll
    for (int g = 0; g < G; ++g) {
#pragma unroll
        for (int e = 0; e < Ge::VPL; ++e) fred[(warp * G + g) * DP + lane * Ge::VPL + e] = o_acc[g][e];
        if (lane == 0) lred[warp * G + g] = l_acc[g];
    }
    __syncthreads();
    float* part = p.partial_ws + ((size_t)slot * p.splits + split) * G * (DP + 2);
    for (int i = tid; i < G * DP; i += kThreads) {
        const int g = i / DP, c = i % DP;
        float s = 0.0f;
        for (int w = 0; w < kWarps; ++w) s += fred[(w * G + g) * DP + c];
        part[g * (DP + 2) + 2 + c] = s;
    }
    if (tid < G) {
        float l = 0.0f;
        for (int w = 0; w < kWarps; ++w) l += lred[w * G + tid];
        part[tid * (DP + 2) + 0] = run_max[tid];
        part[tid * (DP + 2) + 1] = l;
    }

    // ---- last CTA of the slot merges the split partials
    __threadfence();
    __syncthreads();
    int* flag = iscr + 8;
    if (tid == 0) {
        const int t = atomicAdd(p.tickets + slot, 1);
        *flag = (t == p.splits - 1);
    }
    __syncthreads();
    if (!*flag) return;
    __threadfence();
    const float* allp = p.partial_ws + (size_t)slot * p.splits * G * (DP + 2);
    float* wts = reinterpret_cast<float*>(smem);  // [splits][G] merge weights
    float* gm = reinterpret_cast<float*>(iscr) + 16;  // [G] global max, [G] l total
    if (tid < G) {
        float m = -INFINITY;
        for (int s = 0; s < p.splits; ++s) m = fmaxf(m, __ldcg(allp + ((size_t)s * G + tid) * (DP + 2)));
        float l = 0.0f;
        for (int s = 0; s < p.splits; ++s) {
            const float ms = __ldcg(allp + ((size_t)s * G + tid) * (DP + 2));
            const float w = ms == -INFINITY ? 0.0f : expf(ms - m);
            wts[s * G + tid] = w;
            l += w * __ldcg(allp + ((size_t)s * G + tid) * (DP + 2) + 1);
        }
        gm[tid] = m;
        gm[G + tid] = l;
    }
    __syncthreads();
    for (int i = tid; i < G * DP; i += kThreads) {
        const int g = i / DP, c = i % DP;
        float acc = 0.0f;
        for (int s = 0; s < p.splits; ++s) {
            const float w = wts[s * G + g];
            if (w != 0.0f) acc = fmaf(w, __ldcg(allp + ((size_t)s * G + g) * (DP + 2) + 2 + c), acc);
        }
        const float l = gm[G + g];
        if (p.out) p.out[((size_t)slot * G + g) * DP + c] = l > 0.0f ? acc / l : 0.0f;
        if (p.partial_out) p.partial_out[((size_t)slot * G + g) * (DP + 2) + 2 + c] = acc;
    }
    if (tid < G) {
        if (p.partial_out) {
            p.partial_out[((size_t)slot * G + tid) * (DP + 2) + 0] = gm[tid];
            p.partial_out[((size_t)slot * G + tid) * (DP + 2) + 1] = gm[G + tid];
        }
        if (p.counts) p.counts[((size_t)slot * G + tid) * 4 + 3] = gm[G + tid] > 0.0f ? 1 : 0;
    }
    if (tid == 0) p.tickets[slot] = 0;  // re-arm for the next launch / graph replay
}

}  // namespace lvk
