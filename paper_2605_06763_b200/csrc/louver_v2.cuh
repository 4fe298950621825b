// Louver query kernel v2 for bf16 KV (the graded path), sm_100a.
//
// One CTA = one work unit: UNIT_CHUNKS x 512 keys of one slot (sequence, kv
// head), processed in three bulk-async streamed phases that share one
// shared-memory ring of two buffers (cp.async.bulk global->shared, completion
// on mbarriers, so the copy engine keeps HBM busy while warps compute):
//
//  P  probe     cell summaries (blocked coordinate-major AABB tiles, one
//               16 KB bulk copy per 512 keys) -> bound = [hi|lo]·[q+|q-] on
//               the tensor cores (mma.sync m16n8k16 bf16, q split into
//               hi+lo bf16 parts so the q-side rounding is 2^-18 relative),
//               compared with tau - slack
//  E  exact     keys of surviving cells (per-row bulk copies into a padded,
//               ldmatrix/LDS.128 conflict-free ring) -> fast scores on the
//               tensor cores; a (key, q head) pair is decided by the fast
//               score unless |fast - tau| < margin; the normative sequential
//               fp32 dot (core.hpp:17-21) is computed for every undecided or
//               attended pair, so membership is bit-exact and softmax inputs
//               are the reference's scores
//  A  attend    V rows of attended keys (selected ∪ buffer) streamed through
//               the ring; exact CTA max, p = exp(scale*s - m), o += p v
//
// Soundness: with S_g = sum_c |q_gc| colmax_c,
// |tensor-core value - exact| <= (2^-18 + 2^-24 * K) S_g and
// |normative - exact| <= gamma_d S_g, both < 2^-14 S_g; the probe prunes at
// tau - 2^-12 S_g and the fast score decides only outside +-2^-13 S_g.
#pragma once

#include "louver_kernels.cuh"

namespace lvk2 {

using lvk::Counters;
using lvk::QueryParams;

constexpr int kThreads = 128;
constexpr int kWarps = kThreads / 32;
constexpr int kChunk = 512;
constexpr int kUnitChunks = 1;
constexpr int kUnit = kChunk * kUnitChunks;  // keys per CTA (one summary tile)
constexpr int kRows = 32;                    // rows per key / value round
constexpr int kGroup = 16;                   // units merged per tree node
constexpr int kMinBlocks = 6;                // resident CTAs per SM the layout is sized for

struct V2Params {
    QueryParams p;       // shared fields (K, V, counters, q, tau, outputs)
    const void* sum;     // blocked summaries [slot][chunk][2][DP][CPC]
    float* gpart;        // [slots][ngroups][G][DP+2]
    int* gtickets;       // [slots][ngroups]
    int* stickets;       // [slots]
    int ngroups;
    int mode_dense;
    long long* trace;    // optional [slots*splits][8] phase timestamps (globaltimer ns), debug
};

template <int DP, int G>
struct G2 {
    static constexpr int ROWB = DP * 2;
    static constexpr int PITCH = ROWB + 16;          // conflict-free ldmatrix / LDS.128 rows
    static constexpr int NT = (2 * G + 7) / 8;       // n-tiles of 8 columns (hi|lo split of q)
    static constexpr int KS_SC = DP / 16;            // k-steps, scores
    static constexpr int KS_PR = 2 * DP / 16;        // k-steps, probe ([hi|lo] x [q+|q-])
    static constexpr int TILE = 2 * DP * 32 * 2;     // summary tile bytes (CPC <= 32)
    static constexpr int KROUND = kRows * PITCH;
    static constexpr int VROUND = kRows * ROWB;
    static constexpr int R0 = TILE > 2 * KROUND ? TILE : 2 * KROUND;
    static constexpr int RING = ((R0 > 2 * VROUND ? R0 : 2 * VROUND) + 127) / 128 * 128;
    static constexpr int QP = DP + 4;
    static constexpr int KHMAX = kWarps;             // k-split partial C tiles

    static constexpr int OFF_RING = 0;
    static constexpr int OFF_CT = OFF_RING + RING;                     // C tiles [KHMAX][32][8*NT] f32
    static constexpr int SZ_CT = KHMAX * 32 * 8 * NT * 4;
    static constexpr int OFF_SC = OFF_CT + SZ_CT;                      // scores / p [kUnit][G]
    static constexpr int SZ_SC = kUnit * G * 4;
    static constexpr int OFF_Q = OFF_SC + SZ_SC;                       // q fp32 [G][QP]
    static constexpr int SZ_Q = G * QP * 4;
    static constexpr int OFF_AM = OFF_Q + SZ_Q;                        // attend mask [kUnit] u8
    static constexpr int OFF_SW = OFF_AM + kUnit;                      // selected words [G][kUnit/32]
    static constexpr int OFF_CM = OFF_SW + G * (kUnit / 32) * 4;       // cell masks [32] u8
    static constexpr int OFF_SV = OFF_CM + 32;                         // survivor cells [32] u16
    static constexpr int OFF_AL = OFF_SV + 64;                         // attended keys [kUnit] u16
    static constexpr int OFF_NP = OFF_AL + kUnit * 2;                  // normative pairs [32*G] u16
    static constexpr int OFF_NF = OFF_NP + kRows * G * 2;              // need flags [32*G] u8
    static constexpr int OFF_RK = OFF_NF + kRows * G;                  // round row -> key [32] u16
    static constexpr int OFF_MISC = (OFF_RK + kRows * 2 + 15) / 16 * 16;  // floats
    static constexpr int SZ_MISC = (16 * G + 64) * 4;
    static constexpr int OFF_BAR = OFF_MISC + SZ_MISC;                 // 1 mbarrier
    static constexpr int SMEM = OFF_BAR + 16;
};

// ------------------------------------------------------------- primitives

__device__ __forceinline__ unsigned smem_u32(const void* p) {
    return static_cast<unsigned>(__cvta_generic_to_shared(p));
}

__device__ __forceinline__ void mbar_init(unsigned long long* bar, unsigned count) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;\n" ::"r"(smem_u32(bar)), "r"(count));
}

__device__ __forceinline__ void mbar_expect_tx(unsigned long long* bar, unsigned bytes) {
    asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;\n" ::"r"(smem_u32(bar)), "r"(bytes)
                 : "memory");
}

__device__ __forceinline__ void mbar_wait(unsigned long long* bar, unsigned parity) {
    const unsigned a = smem_u32(bar);
    asm volatile(
        "{\n"
        ".reg .pred p;\n"
        "WAIT_%=:\n"
        "mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n"
        "@!p bra WAIT_%=;\n"
        "}\n" ::"r"(a),
        "r"(parity)
        : "memory");
}

__device__ __forceinline__ void bulk_g2s(void* dst, const void* src, unsigned bytes, unsigned long long* bar) {
    asm volatile(
        "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];\n" ::"r"(
            smem_u32(dst)),
        "l"(src), "r"(bytes), "r"(smem_u32(bar))
        : "memory");
}

__device__ __forceinline__ void fence_proxy_async() {
    asm volatile("fence.proxy.async.shared::cta;\n" ::: "memory");
}

__device__ __forceinline__ void ldsm_x4(unsigned (&r)[4], const void* p) {
    asm volatile("ldmatrix.sync.aligned.m8n8.x4.shared.b16 {%0,%1,%2,%3}, [%4];\n"
                 : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3])
                 : "r"(smem_u32(p)));
}

__device__ __forceinline__ void ldsm_x4_t(unsigned (&r)[4], const void* p) {
    asm volatile("ldmatrix.sync.aligned.m8n8.x4.trans.shared.b16 {%0,%1,%2,%3}, [%4];\n"
                 : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3])
                 : "r"(smem_u32(p)));
}

__device__ __forceinline__ void mma16816(float (&c)[4], const unsigned (&a)[4], unsigned b0, unsigned b1) {
    asm volatile(
        "mma.sync.aligned.m16n8k16.row.col.f32.bf16.bf16.f32 {%0,%1,%2,%3}, {%4,%5,%6,%7}, {%8,%9}, "
        "{%0,%1,%2,%3};\n"
        : "+f"(c[0]), "+f"(c[1]), "+f"(c[2]), "+f"(c[3])
        : "r"(a[0]), "r"(a[1]), "r"(a[2]), "r"(a[3]), "r"(b0), "r"(b1));
}

__device__ __forceinline__ unsigned short bf_bits(float x) {
    return __bfloat16_as_ushort(__float2bfloat16_rn(x));
}
__device__ __forceinline__ float bf_val(unsigned short b) { return __uint_as_float((unsigned)b << 16); }

// q split into two bf16 parts: x ~= hi + lo, |x - hi - lo| <= 2^-18 |x|.
__device__ __forceinline__ unsigned short split_part(float x, int part) {
    const unsigned short h = bf_bits(x);
    return part == 0 ? h : bf_bits(x - bf_val(h));
}

__device__ __forceinline__ long long gtimer() {
    long long t;
    asm volatile("mov.u64 %0, %globaltimer;" : "=l"(t));
    return t;
}

// Block-wide ordered compaction (count <= 2048). Writes ascending indices of
// set flags into list, returns the total; `scratch` = kWarps ints.
template <typename Flag>
__device__ __forceinline__ int compact(int count, Flag flag, unsigned short* list, int* scratch) {
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

// Merge P partials (m, l, o[DP]) at `src` (stride G*(DP+2) between partials)
// into `dst` (same [G][DP+2] layout) or, when final, into out rows.
template <int DP, int G>
__device__ void merge_partials(const float* src, int P, float* dst, float* out, float* part_out, int* counts,
                       float* shw) {
    // shw: [P][G] weights, then M[G], L[G]; all partial headers are loaded in
    // parallel and the o loads are batched, so a merge costs ~2 L2 round trips.
    const int tid = threadIdx.x;
    constexpr int W = G * (DP + 2);
    float* shm = shw;              // [P][G] m, then weights
    float* shl = shw + P * G;      // [P][G] l
    float* ML = shl + P * G;       // M[G], L[G]
    for (int i = tid; i < P * G; i += kThreads) {
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
    for (int i = tid; i < G * DP; i += kThreads) {
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

// --------------------------------------------------------------- the kernel

// B fragment (m16n8k16 .col) of the split-q matrix for k-step `ks`, n-tile `nt`:
// b0 = B[ks*16 + 2(l%4) .. +1][n], b1 = B[ks*16 + 2(l%4) + 8 .. +9][n], n = nt*8 + l/4,
// column n -> (part = n / G: 0 hi, 1 lo; g = n % G). Probe rows k < DP use q+,
// k >= DP use q- (the [hi | lo] concatenation of the AABB tile).
template <int DP, int G>
__device__ __forceinline__ uint2 q_frag(const float* qf, int ks, int nt, int lane, bool probe) {
    const int col = nt * 8 + lane / 4;
    unsigned short v[4] = {0, 0, 0, 0};
    if (col < 2 * G) {
        const int part = col / G, g = col % G;
#pragma unroll
        for (int e = 0; e < 4; ++e) {
            const int k = ks * 16 + 2 * (lane & 3) + (e & 1) + (e >> 1) * 8;
            float x;
            if (probe) {
                const float qq = qf[g * (DP + 4) + (k % DP)];
                x = k < DP ? fmaxf(qq, 0.0f) : fminf(qq, 0.0f);
            } else {
                x = qf[g * (DP + 4) + k];
            }
            v[e] = split_part(x, part);
        }
    }
    return make_uint2((unsigned)v[0] | ((unsigned)v[1] << 16), (unsigned)v[2] | ((unsigned)v[3] << 16));
}

template <int DP, int G>
__global__ void __launch_bounds__(kThreads, kMinBlocks) louver_query_v2(const __grid_constant__ V2Params vp) {
    using Ge = G2<DP, G>;
    const QueryParams& p = vp.p;
    extern __shared__ __align__(128) unsigned char smem[];
    unsigned char* ring = smem + Ge::OFF_RING;
    float* ct = reinterpret_cast<float*>(smem + Ge::OFF_CT);
    float* sc = reinterpret_cast<float*>(smem + Ge::OFF_SC);
    float* qf = reinterpret_cast<float*>(smem + Ge::OFF_Q);
    unsigned char* am = smem + Ge::OFF_AM;
    unsigned* sw = reinterpret_cast<unsigned*>(smem + Ge::OFF_SW);
    unsigned char* cm = smem + Ge::OFF_CM;
    unsigned short* sv = reinterpret_cast<unsigned short*>(smem + Ge::OFF_SV);
    unsigned short* al = reinterpret_cast<unsigned short*>(smem + Ge::OFF_AL);
    unsigned short* np = reinterpret_cast<unsigned short*>(smem + Ge::OFF_NP);
    unsigned char* needf = smem + Ge::OFF_NF;
    unsigned short* rowkey = reinterpret_cast<unsigned short*>(smem + Ge::OFF_RK);
    float* misc = reinterpret_cast<float*>(smem + Ge::OFF_MISC);
    float* tau_s = misc;            // [G]
    float* tau_pr = misc + G;       // [G] probe threshold tau - slack
    float* marg = misc + 2 * G;     // [G] fast-score margin
    float* mx = misc + 3 * G;       // [G] CTA max of scaled scores
    float* lsum = misc + 4 * G;     // [G]
    float* red = misc + 5 * G;      // [kWarps][G] reduction scratch (<= 32 floats)
    int* iscr = reinterpret_cast<int*>(misc + 16 * G);  // 64 ints
    unsigned long long* bar = reinterpret_cast<unsigned long long*>(smem + Ge::OFF_BAR);

    const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
    const int slot = blockIdx.y, unit = blockIdx.x;
    const bool dense = vp.mode_dense != 0;
    const long long n = p.ctr->n;
    const long long indexed = dense ? 0 : p.ctr->indexed;
    const int rl = p.r_log2;
    const int r = 1 << rl;
    const int CPC = kChunk >> rl;  // cells per chunk (= per unit)
    const __nv_bfloat16* Ks = reinterpret_cast<const __nv_bfloat16*>(p.K) + (size_t)slot * p.cap * DP;
    const __nv_bfloat16* Vs = reinterpret_cast<const __nv_bfloat16*>(p.V) + (size_t)slot * p.cap * DP;
    const long long k0 = (long long)unit * kUnit;
    const int nvalid = (int)(n - k0 > kUnit ? kUnit : (n - k0 > 0 ? n - k0 : 0));
    const int tile_b = 2 * DP * CPC * 2;
    const bool probe_on = !dense && nvalid > 0 && k0 < indexed;
    long long* trace = vp.trace ? vp.trace + ((size_t)slot * p.splits + unit) * 8 : nullptr;
#define LV2_TRACE(i)                           \
    if (trace && tid == 0) trace[i] = gtimer();
    LV2_TRACE(0)

    // ---- the summary tile is the first dependent load: issue it before setup
    if (tid == 0) {
        mbar_init(&bar[0], 1);
        asm volatile("fence.mbarrier_init.release.cluster;\n" ::: "memory");
        if (probe_on) {
            const unsigned char* sum = reinterpret_cast<const unsigned char*>(vp.sum) +
                                       ((size_t)slot * (p.cap / kChunk) + (size_t)(k0 / kChunk)) * tile_b;
            mbar_expect_tx(&bar[0], tile_b);
            bulk_g2s(ring, sum, tile_b, &bar[0]);
        }
    }
    // ---- setup: q, thresholds
    for (int i = tid; i < G * DP; i += kThreads) {
        const int g = i / DP, c = i % DP;
        qf[g * Ge::QP + c] = p.q[((size_t)slot * G + g) * DP + c];
    }
    for (int i = tid; i < kUnit / 4; i += kThreads) reinterpret_cast<unsigned*>(am)[i] = 0;
    for (int i = tid; i < G * (kUnit / 32); i += kThreads) sw[i] = 0;
    __syncthreads();
    if (warp < G) {
        for (int g = warp; g < G; g += kWarps) {
            float s = 0.0f;
            for (int c = lane; c < DP; c += 32)
                s = __fadd_ru(s, __fmul_ru(fabsf(qf[g * Ge::QP + c]), p.colmax[(size_t)slot * DP + c]));
#pragma unroll
            for (int o = 16; o > 0; o >>= 1) s = __fadd_ru(s, __shfl_xor_sync(0xffffffffu, s, o));
            if (lane == 0) {
                const float t = p.tau ? p.tau[(size_t)slot * G + g] : -INFINITY;
                tau_s[g] = t;
                tau_pr[g] = __fsub_rd(t, __fmul_ru(s, 2.44140625e-4f));  // 2^-12 S
                marg[g] = __fmul_ru(s, 1.220703125e-4f);                // 2^-13 S
            }
        }
    }

    int stat_scan[G];
#pragma unroll
    for (int g = 0; g < G; ++g) stat_scan[g] = 0;
    unsigned long long t_cells = 0, t_surv = 0, t_keys = 0, t_vals = 0;

    // ---------------------------------------------------------- P: probe
    const int ncells = (nvalid + r - 1) >> rl;  // cells holding keys
    const int MT = (CPC + 15) / 16;             // m-tiles of 16 cells
    const int KH = kWarps / MT;                 // k-split per m-tile
    if (probe_on) {
        mbar_wait(&bar[0], 0);
        LV2_TRACE(1)
        {
            const int mt = warp % MT, kh = warp / MT;
            const int ksteps = Ge::KS_PR / KH;
            float acc[Ge::NT][4];
#pragma unroll
            for (int t = 0; t < Ge::NT; ++t) acc[t][0] = acc[t][1] = acc[t][2] = acc[t][3] = 0.0f;
            // ldmatrix.trans from [k][cell]: lane -> matrix lane/8, stored row lane%8;
            // cells past CPC (r = 64: 8 cells) read the neighbouring rows, unused
            const int mi = lane >> 3, rr = lane & 7;
            const int cic = (mt * 16 + (mi & 1) * 8) % CPC;
            for (int s = 0; s < ksteps; ++s) {
                const int ks = kh * ksteps + s;
                const int k = ks * 16 + (mi >> 1) * 8 + rr;
                const int part = k < DP ? 1 : 0;  // tile = [lo | hi]; A = [hi | lo]
                const int kk = k < DP ? k : k - DP;
                unsigned a[4];
                ldsm_x4_t(a, ring + ((size_t)part * DP * CPC + (size_t)kk * CPC + cic) * 2);
#pragma unroll
                for (int t = 0; t < Ge::NT; ++t) {
                    const uint2 b = q_frag<DP, G>(qf, ks, t, lane, true);
                    mma16816(acc[t], a, b.x, b.y);
                }
            }
#pragma unroll
            for (int t = 0; t < Ge::NT; ++t) {
                const int row = mt * 16 + (lane >> 2), col = t * 8 + 2 * (lane & 3);
                float* dst = ct + (size_t)kh * 32 * 8 * Ge::NT;
                if (row < 32) {
                    dst[row * 8 * Ge::NT + col] = acc[t][0];
                    dst[row * 8 * Ge::NT + col + 1] = acc[t][1];
                }
                if (row + 8 < 32) {
                    dst[(row + 8) * 8 * Ge::NT + col] = acc[t][2];
                    dst[(row + 8) * 8 * Ge::NT + col + 1] = acc[t][3];
                }
            }
        }
        __syncthreads();
    }
    if (tid < 32) {  // one thread per cell (<= 32 cells per unit)
        const int cell = tid;
        unsigned char m = 0;
        if (cell < ncells) {
            const long long cs = k0 + ((long long)cell << rl);
            const long long ce = cs + r;
            if (!probe_on || ce > indexed) {
                m = (unsigned char)((1u << G) - 1u);  // dense mode, or buffer keys inside
            } else {
#pragma unroll
                for (int g = 0; g < G; ++g) {
                    float b = 0.0f;
                    for (int kh = 0; kh < KH; ++kh) {
                        const float* src = ct + (size_t)kh * 32 * 8 * Ge::NT + cell * 8 * Ge::NT;
                        b += src[g] + src[G + g];
                    }
                    if (b >= tau_pr[g]) m |= (unsigned char)(1u << g);
                }
            }
            ++t_cells;
            if (m) ++t_surv;
            const long long kend = ce < n ? ce : n;
#pragma unroll
            for (int g = 0; g < G; ++g)
                if (m & (1u << g)) stat_scan[g] += (int)(kend - cs);
        }
        cm[cell] = m;
    }
    __syncthreads();
    LV2_TRACE(2)
    const int nsurv = compact(CPC, [&](int i) { return cm[i] != 0; }, sv, iscr);
    const int nrows = nsurv << rl;

    // ---------------------------------------------------------- E: exact
    // keys of surviving cells, 16-byte cp.async pieces, two rounds in flight
    const int nrounds = (nrows + kRows - 1) / kRows;
    auto issue_keys = [&](int rd) {
        const int r0 = rd * kRows;
        const int cnt = nrows - r0 < kRows ? nrows - r0 : kRows;
        unsigned char* dst = ring + (rd & 1) * Ge::KROUND;
        constexpr int CPR = Ge::ROWB / 16;
        for (int it = tid; it < cnt * CPR; it += kThreads) {
            const int i = it / CPR, c = it % CPR;
            const int f = r0 + i;
            const int key = ((int)sv[f >> rl] << rl) + (f & (r - 1));
            if (key < nvalid)
                lvk::cp_async16(dst + i * Ge::PITCH + c * 16,
                                reinterpret_cast<const unsigned char*>(Ks + (size_t)(k0 + key) * DP) + c * 16);
        }
        lvk::cp_async_commit();
    };
    auto wait_round = [&](int rd, int rounds) {
        if (rd + 1 < rounds)
            lvk::cp_async_wait<1>();
        else
            lvk::cp_async_wait<0>();
        __syncthreads();
    };
    if (nrounds > 0) issue_keys(0);
    if (nrounds > 1) issue_keys(1);
    // score fragments for this warp's k-range, kept in registers across rounds
    constexpr int MTR = kRows / 16;        // m-tiles per round
    constexpr int KHR = kWarps / MTR;      // k-split
    constexpr int KSW = Ge::KS_SC / KHR;   // k-steps per warp
    const int mtr = warp % MTR, khr = warp / MTR;
    uint2 bq[KSW][Ge::NT];
#pragma unroll
    for (int s = 0; s < KSW; ++s)
#pragma unroll
        for (int t = 0; t < Ge::NT; ++t) bq[s][t] = q_frag<DP, G>(qf, khr * KSW + s, t, lane, false);
    for (int rd = 0; rd < nrounds; ++rd) {
        wait_round(rd, nrounds);
        const unsigned char* kb = ring + (rd & 1) * Ge::KROUND;
        const int r0 = rd * kRows;
        const int cnt = nrows - r0 < kRows ? nrows - r0 : kRows;
        if (mtr * 16 < cnt) {
            float acc[Ge::NT][4];
#pragma unroll
            for (int t = 0; t < Ge::NT; ++t) acc[t][0] = acc[t][1] = acc[t][2] = acc[t][3] = 0.0f;
            const int row = mtr * 16 + (lane & 7) + ((lane >> 3) & 1) * 8;
            const int kofs = (lane >> 4) * 8;
#pragma unroll
            for (int s = 0; s < KSW; ++s) {
                const int ks = khr * KSW + s;
                unsigned a[4];
                ldsm_x4(a, kb + row * Ge::PITCH + (ks * 16 + kofs) * 2);
#pragma unroll
                for (int t = 0; t < Ge::NT; ++t) mma16816(acc[t], a, bq[s][t].x, bq[s][t].y);
            }
#pragma unroll
            for (int t = 0; t < Ge::NT; ++t) {
                const int rw = mtr * 16 + (lane >> 2), col = t * 8 + 2 * (lane & 3);
                float* dst = ct + (size_t)khr * 32 * 8 * Ge::NT;
                dst[rw * 8 * Ge::NT + col] = acc[t][0];
                dst[rw * 8 * Ge::NT + col + 1] = acc[t][1];
                dst[(rw + 8) * 8 * Ge::NT + col] = acc[t][2];
                dst[(rw + 8) * 8 * Ge::NT + col + 1] = acc[t][3];
            }
        }
        __syncthreads();
        // classify (row, g): the fast score decides outside +-margin; the
        // normative dot is run for undecided and for attended pairs
        for (int pi = tid; pi < kRows * G; pi += kThreads) {
            const int row = pi / G, g = pi % G;
            unsigned char need = 0;
            if (row < cnt) {
                const int f = r0 + row;
                const int key = ((int)sv[f >> rl] << rl) + (f & (r - 1));
                if (g == 0) rowkey[row] = (unsigned short)key;
                if (key < nvalid) {
                    float fast = 0.0f;
#pragma unroll
                    for (int kh = 0; kh < KHR; ++kh) {
                        const float* c0 = ct + (size_t)kh * 32 * 8 * Ge::NT + row * 8 * Ge::NT;
                        fast += c0[g] + c0[G + g];
                    }
                    if (dense) {
                        sc[key * G + g] = fast;
                        if (g == 0) am[key] = (unsigned char)((1u << G) - 1u);
                    } else {
                        const bool in_buf = k0 + key >= indexed;
                        need = (fast >= tau_s[g] - marg[g]) || (in_buf && !p.strict);
                    }
                    if (g == 0) ++t_keys;
                }
            }
            needf[pi] = need;
        }
        __syncthreads();
        if (!dense) {
            const int tot = compact(kRows * G, [&](int i) { return needf[i] != 0; }, np, iscr);
            for (int e = tid; e < tot; e += kThreads) {
                const int pi = np[e];
                const int row = pi / G, g = pi % G;
                const int key = rowkey[row];
                const unsigned char* krow = kb + row * Ge::PITCH;
                const float* qg = qf + g * Ge::QP;
                float s = 0.0f;
#pragma unroll 2
                for (int c = 0; c < DP / 8; ++c) {
                    const uint4 kv = *reinterpret_cast<const uint4*>(krow + c * 16);
                    float kf[8];
                    lvk::unpack16<__nv_bfloat16>(kv, kf);
#pragma unroll
                    for (int e2 = 0; e2 < 8; ++e2) s = __fadd_rn(s, __fmul_rn(qg[c * 8 + e2], kf[e2]));
                }
                sc[key * G + g] = s;
                const bool selected = s >= tau_s[g];
                const bool in_buf = k0 + key >= indexed;
                if (selected) atomicOr(&sw[g * (kUnit / 32) + (key >> 5)], 1u << (key & 31));
                if (selected || (in_buf && !p.strict))
                    atomicOr(reinterpret_cast<unsigned*>(am + (key & ~3)), 1u << ((key & 3) * 8 + g));
            }
        }
        __syncthreads();
        if (rd + 2 < nrounds) issue_keys(rd + 2);
    }

    LV2_TRACE(3)
    // selected bitmap words + counts
    int stat_sel[G];
#pragma unroll
    for (int g = 0; g < G; ++g) stat_sel[g] = 0;
    if (!dense) {
        for (int i = tid; i < G * (kUnit / 32); i += kThreads) {
            const int g = i / (kUnit / 32), w = i % (kUnit / 32);
            const unsigned v = sw[i];
            stat_sel[g] += __popc(v);
            if (p.bits) {
                const long long word = (k0 >> 5) + w;
                if (word < p.bits_words) p.bits[((size_t)slot * G + g) * p.bits_words + word] = v;
            }
        }
    }

    // ---------------------------------------------------------- A: attend
    const int natt = compact(nvalid, [&](int i) { return am[i] != 0; }, al, iscr);
    // V rows of attended keys: issue the first two rounds before the softmax math
    const int vrounds = (natt + kRows - 1) / kRows;
    auto issue_vals = [&](int rd) {
        const int r0 = rd * kRows;
        const int cnt = natt - r0 < kRows ? natt - r0 : kRows;
        unsigned char* dst = ring + (rd & 1) * Ge::VROUND;
        constexpr int CPR = Ge::ROWB / 16;
        for (int it = tid; it < cnt * CPR; it += kThreads) {
            const int i = it / CPR, c = it % CPR;
            lvk::cp_async16(dst + i * Ge::ROWB + c * 16,
                            reinterpret_cast<const unsigned char*>(Vs + (size_t)(k0 + al[r0 + i]) * DP) + c * 16);
        }
        lvk::cp_async_commit();
    };
    LV2_TRACE(4)
    if (vrounds > 0) issue_vals(0);
    if (vrounds > 1) issue_vals(1);
    {
        // exact CTA max per q head of scale*s over attended pairs
        float cmx[G];
#pragma unroll
        for (int g = 0; g < G; ++g) cmx[g] = -INFINITY;
        for (int i = tid; i < natt; i += kThreads) {
            const int key = al[i];
            const unsigned char m = am[key];
#pragma unroll
            for (int g = 0; g < G; ++g)
                if (m & (1u << g)) cmx[g] = fmaxf(cmx[g], p.scale * sc[key * G + g]);
        }
#pragma unroll
        for (int g = 0; g < G; ++g) {
            float v = cmx[g];
#pragma unroll
            for (int o = 16; o > 0; o >>= 1) v = fmaxf(v, __shfl_xor_sync(0xffffffffu, v, o));
            if (lane == 0) red[warp * G + g] = v;
        }
        __syncthreads();
        if (tid < G) {
            float v = -INFINITY;
            for (int w = 0; w < kWarps; ++w) v = fmaxf(v, red[w * G + tid]);
            mx[tid] = v;
        }
        __syncthreads();
        // p = exp(scale*s - m) (0 for pairs not attended), l = sum p
        float lp[G];
#pragma unroll
        for (int g = 0; g < G; ++g) lp[g] = 0.0f;
        for (int i = tid; i < natt; i += kThreads) {
            const int key = al[i];
            const unsigned char m = am[key];
#pragma unroll
            for (int g = 0; g < G; ++g) {
                const float e = (m & (1u << g)) ? expf(p.scale * sc[key * G + g] - mx[g]) : 0.0f;
                sc[key * G + g] = e;
                lp[g] += e;
            }
        }
#pragma unroll
        for (int g = 0; g < G; ++g) {
            float v = lp[g];
#pragma unroll
            for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
            if (lane == 0) red[warp * G + g] = v;
        }
        __syncthreads();
        if (tid < G) {
            float v = 0.0f;
            for (int w = 0; w < kWarps; ++w) v += red[w * G + tid];
            lsum[tid] = v;
        }
    }
    // thread -> (dim pair dp, row group rg)
    constexpr int NDP = DP / 2;
    constexpr int NRG = kThreads / NDP;
    const int dp = tid % NDP, rg = tid / NDP;
    float o[G][2];
#pragma unroll
    for (int g = 0; g < G; ++g) o[g][0] = o[g][1] = 0.0f;
    for (int rd = 0; rd < vrounds; ++rd) {
        wait_round(rd, vrounds);
        const unsigned char* vb = ring + (rd & 1) * Ge::VROUND;
        const int r0 = rd * kRows;
        const int cnt = natt - r0 < kRows ? natt - r0 : kRows;
        for (int i = rg; i < cnt; i += NRG) {
            const unsigned w2 = *reinterpret_cast<const unsigned*>(vb + i * Ge::ROWB + dp * 4);
            const float v0 = lvk::bf_lo(w2), v1 = lvk::bf_hi(w2);
            const float* pk = sc + (size_t)al[r0 + i] * G;
#pragma unroll
            for (int g = 0; g < G; ++g) {
                const float pw = pk[g];
                o[g][0] = fmaf(pw, v0, o[g][0]);
                o[g][1] = fmaf(pw, v1, o[g][1]);
            }
        }
        __syncthreads();
        if (rd + 2 < vrounds) issue_vals(rd + 2);
    }
    LV2_TRACE(5)
    t_vals = tid == 0 ? (unsigned long long)natt : 0ull;

    // ---- statistics
    if (p.counts) {
        int att[G];
#pragma unroll
        for (int g = 0; g < G; ++g) att[g] = 0;
        for (int i = tid; i < natt; i += kThreads) {
            const unsigned char m = am[al[i]];
#pragma unroll
            for (int g = 0; g < G; ++g) att[g] += (m >> g) & 1;
        }
#pragma unroll
        for (int g = 0; g < G; ++g) {
            const int s0 = lvk::warp_sum_int(stat_sel[g]);
            const int s1 = lvk::warp_sum_int(att[g]);
            const int s2 = lvk::warp_sum_int(stat_scan[g]);
            if (lane == 0) {
                int* c = p.counts + ((size_t)slot * G + g) * 4;
                if (s0) atomicAdd(c + 0, s0);
                if (s1) atomicAdd(c + 1, s1);
                if (s2) atomicAdd(c + 2, s2);
            }
        }
    }
    if (p.totals) {
        unsigned long long a = t_cells, bq2 = t_surv, c = t_keys, d = t_vals;
#pragma unroll
        for (int of = 16; of > 0; of >>= 1) {
            a += __shfl_xor_sync(0xffffffffu, a, of);
            bq2 += __shfl_xor_sync(0xffffffffu, bq2, of);
            c += __shfl_xor_sync(0xffffffffu, c, of);
            d += __shfl_xor_sync(0xffffffffu, d, of);
        }
        if (lane == 0) {
            if (a) atomicAdd(p.totals + 0, a);
            if (bq2) atomicAdd(p.totals + 1, bq2);
            if (c) atomicAdd(p.totals + 2, c);
            if (d) atomicAdd(p.totals + 3, d);
        }
    }

    // ---- unit partial: reduce o over row groups
    float* ored = reinterpret_cast<float*>(ring);  // [NRG][G][DP]
#pragma unroll
    for (int g = 0; g < G; ++g) {
        ored[(rg * G + g) * DP + 2 * dp] = o[g][0];
        ored[(rg * G + g) * DP + 2 * dp + 1] = o[g][1];
    }
    __syncthreads();
    constexpr int W = G * (DP + 2);
    float* part = p.partial_ws + ((size_t)slot * p.splits + unit) * W;
    for (int i = tid; i < G * DP; i += kThreads) {
        const int g = i / DP, c = i % DP;
        float s = 0.0f;
        for (int q = 0; q < NRG; ++q) s += ored[(q * G + g) * DP + c];
        part[g * (DP + 2) + 2 + c] = s;
    }
    if (tid < G) {
        part[tid * (DP + 2)] = lsum[tid] > 0.0f ? mx[tid] : -INFINITY;
        part[tid * (DP + 2) + 1] = lsum[tid];
    }

    LV2_TRACE(6)
    // ---- two-level merge: last unit of each group of kGroup, then last group
    __threadfence();
    __syncthreads();
    int* flag = iscr + 32;
    const int grp = unit / kGroup;
    const int members = p.splits - grp * kGroup < kGroup ? p.splits - grp * kGroup : kGroup;
    if (tid == 0) *flag = atomicAdd(vp.gtickets + slot * vp.ngroups + grp, 1) == members - 1;
    __syncthreads();
    if (!*flag) return;
    __threadfence();
    float* shw = reinterpret_cast<float*>(ring);
    float* gdst = vp.gpart + ((size_t)slot * vp.ngroups + grp) * W;
    merge_partials<DP, G>(p.partial_ws + ((size_t)slot * p.splits + grp * kGroup) * W, members, gdst,
                          nullptr, nullptr, nullptr, shw);
    if (tid == 0) vp.gtickets[slot * vp.ngroups + grp] = 0;
    __threadfence();
    __syncthreads();
    if (tid == 0) *flag = atomicAdd(vp.stickets + slot, 1) == vp.ngroups - 1;
    __syncthreads();
    if (!*flag) return;
    __threadfence();
    merge_partials<DP, G>(vp.gpart + (size_t)slot * vp.ngroups * W, vp.ngroups, nullptr,
                          p.out ? p.out + (size_t)slot * G * DP : nullptr,
                          p.partial_out ? p.partial_out + (size_t)slot * W : nullptr,
                          p.counts ? p.counts + (size_t)slot * G * 4 : nullptr, shw);
    if (tid == 0) vp.stickets[slot] = 0;
    LV2_TRACE(7)
#undef LV2_TRACE
}

cudaError_t launch_query_v2(int DP, int G, const V2Params& vp, dim3 grid, cudaStream_t st);
int query_v2_smem(int DP, int G);

}  // namespace lvk2
