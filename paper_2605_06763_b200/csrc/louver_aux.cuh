// Index build / insert / data-movement / merge kernels (sm_100a).
#pragma once

#include "louver_kernels.cuh"

namespace lvk {

template <typename T>
__device__ __forceinline__ float to_f(T x);
template <>
__device__ __forceinline__ float to_f<float>(float x) { return x; }
template <>
__device__ __forceinline__ float to_f<__nv_bfloat16>(__nv_bfloat16 x) { return __bfloat162float(x); }

template <typename T>
__device__ __forceinline__ T from_f(float x);
template <>
__device__ __forceinline__ float from_f<float>(float x) { return x; }
template <>
__device__ __forceinline__ __nv_bfloat16 from_f<__nv_bfloat16>(float x) { return __float2bfloat16_rn(x); }

// Copy src rows [slots][n][d] (S = fp32 or T) into the arena rows
// [slots][cap][DP] starting at row `first`, zero-filling columns d..DP.
template <typename S, typename T>
__global__ void convert_rows_kernel(const S* __restrict__ src, T* __restrict__ dst, long long slots,
                                    long long n, int d, int DP, long long cap, long long first) {
    const long long total = slots * n * DP;
    for (long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x; i < total;
         i += (long long)gridDim.x * blockDim.x) {
        const int c = (int)(i % DP);
        const long long row = i / DP;
        const long long s = row / n, j = row % n;
        const float v = c < d ? to_f<S>(src[(s * n + j) * d + c]) : 0.0f;
        dst[(s * cap + first + j) * DP + c] = from_f<T>(v);
    }
}

// Cell AABBs for cells [cell_begin, cell_end) of every slot over keys [0, n):
// summary row [slot][cell] = [hi (DP) | lo (DP)], per-coordinate max/min of the cell's keys
// (exactly representable in T: they are stored key values). Also folds
// max |k_c| into colmax[slot][DP]. One CTA = 32 cells (16 at DP=256) of one slot.
template <typename T, int DP>
__global__ void __launch_bounds__(256) summarize_kernel(const T* __restrict__ K, T* __restrict__ lo,
                                                        T* __restrict__ hi, float* __restrict__ colmax,
                                                        long long cap, long long cap_cells, int r_log2,
                                                        long long n, long long cell_begin,
                                                        long long cell_end) {
    constexpr int NPAIR = DP / 2;
    constexpr int NSG = 256 / NPAIR;  // cell subgroups
    constexpr int CB = DP > 128 ? 16 : 32;  // cells per CTA
    __shared__ float slo[DP][CB + 1];
    __shared__ float shi[DP][CB + 1];
    __shared__ float cmax[DP];
    const int slot = blockIdx.y;
    const long long c0 = cell_begin + (long long)blockIdx.x * CB;
    const int tid = threadIdx.x;
    const int dp = tid % NPAIR, sg = tid / NPAIR;
    const int r = 1 << r_log2;
    for (int i = tid; i < DP; i += 256) cmax[i] = 0.0f;
    __syncthreads();
    const T* Ks = K + (size_t)slot * cap * DP;
    float am0 = 0.0f, am1 = 0.0f;
    for (int cl = sg; cl < CB; cl += NSG) {
        const long long cell = c0 + cl;
        float l0 = INFINITY, l1 = INFINITY, h0 = -INFINITY, h1 = -INFINITY;
        if (cell < cell_end) {
            const long long ks = cell << r_log2;
            const long long ke = ks + r < n ? ks + r : n;
            for (long long j = ks; j < ke; ++j) {
                const float x0 = to_f<T>(Ks[(size_t)j * DP + 2 * dp]);
                const float x1 = to_f<T>(Ks[(size_t)j * DP + 2 * dp + 1]);
                l0 = fminf(l0, x0);
                h0 = fmaxf(h0, x0);
                l1 = fminf(l1, x1);
                h1 = fmaxf(h1, x1);
            }
            if (ke > ks) {
                am0 = fmaxf(am0, fmaxf(fabsf(l0), fabsf(h0)));
                am1 = fmaxf(am1, fmaxf(fabsf(l1), fabsf(h1)));
            }
        }
        slo[2 * dp][cl] = l0;
        slo[2 * dp + 1][cl] = l1;
        shi[2 * dp][cl] = h0;
        shi[2 * dp + 1][cl] = h1;
    }
    atomicMax(reinterpret_cast<int*>(&cmax[2 * dp]), __float_as_int(am0));
    atomicMax(reinterpret_cast<int*>(&cmax[2 * dp + 1]), __float_as_int(am1));
    __syncthreads();
    // cell-major layout: one row per cell = [hi (DP) | lo (DP)]
    (void)hi;
    for (int i = tid; i < 2 * DP * CB; i += 256) {
        const int cl = i / (2 * DP), e = i % (2 * DP);
        const long long cell = c0 + cl;
        if (cell < cell_end && (cell << r_log2) < n) {
            const size_t at = ((size_t)slot * cap_cells + (size_t)cell) * 2 * DP + (size_t)e;
            lo[at] = from_f<T>(e < DP ? shi[e][cl] : slo[e - DP][cl]);
        }
    }
    for (int c = tid; c < DP; c += 256)
        atomicMax(reinterpret_cast<int*>(colmax + (size_t)slot * DP + c), __float_as_int(cmax[c]));
}

// Host-mapped (zero-copy) input staging for lv_query_layers: dst[i] = src[i] for the q
// block and the tau block, read over the bus by many CTAs in one launch (a copy-engine
// transfer costs ~10 us of fixed latency inside a graph; this costs one bus round trip).
__global__ void stage_in_kernel(const float* __restrict__ q, float* __restrict__ qd, long long nq,
                                const float* __restrict__ tau, float* __restrict__ td, long long nt) {
    // the first layer kernel may launch now: it prefetches sealed summaries, then waits for this grid
    asm volatile("griddepcontrol.launch_dependents;\n" ::: "memory");
    for (long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x; i < nq + nt;
         i += (long long)gridDim.x * blockDim.x) {
        if (i < nq)
            qd[i] = __ldcv(q + i);
        else
            td[i - nq] = __ldcv(tau + (i - nq));
    }
}

// One decode step's insert for every slot (cache.cpp:7-10 on the device):
// append k/v at row n, fold k into cell n/r's box (opening it when n % r == 0),
// raise colmax; the last CTA advances n and applies the flush-at-B rule
// (indexed = n when n - indexed >= B). Counters stay on the device, so a
// decode loop of query -> insert can be captured in one CUDA graph.
template <typename S, typename T>
__global__ void insert_kernel(const S* __restrict__ k, const S* __restrict__ v, T* __restrict__ K,
                              T* __restrict__ V, T* __restrict__ lo, T* __restrict__ hi,
                              float* __restrict__ colmax, Counters* ctr, int* ticket, int d, int DP,
                              long long cap, long long cap_cells, int r_log2, long long B,
                              int nslots) {
    const int slot = blockIdx.x;
    const long long pos = ctr->n;
    const long long cell = pos >> r_log2;
    const bool open = (pos & ((1 << r_log2) - 1)) == 0;
    for (int c = threadIdx.x; c < DP; c += blockDim.x) {
        const float kx = c < d ? to_f<S>(k[(size_t)slot * d + c]) : 0.0f;
        const float vx = c < d ? to_f<S>(v[(size_t)slot * d + c]) : 0.0f;
        const T kt = from_f<T>(kx);
        K[((size_t)slot * cap + pos) * DP + c] = kt;
        V[((size_t)slot * cap + pos) * DP + c] = from_f<T>(vx);
        const float kr = to_f<T>(kt);
        // cell-major summary row [hi (DP) | lo (DP)]
        T* hp = lo + ((size_t)slot * cap_cells + (size_t)cell) * 2 * DP + (size_t)c;
        T* lp = hp + DP;
        (void)hi;
        if (open) {
            *lp = kt;
            *hp = kt;
        } else {
            if (kr < to_f<T>(*lp)) *lp = kt;
            if (kr > to_f<T>(*hp)) *hp = kt;
        }
        float* cm = colmax + (size_t)slot * DP + c;
        if (fabsf(kr) > *cm) *cm = fabsf(kr);
    }
    __threadfence();
    __syncthreads();
    if (threadIdx.x == 0) {
        const int t = atomicAdd(ticket, 1);
        if (t == nslots - 1) {
            const long long nn = pos + 1;
            ctr->n = nn;
            if (nn - ctr->indexed >= B) {
                ctr->indexed = nn;
                ctr->flushes += 1;
            }
            *ticket = 0;
            __threadfence();
        }
    }
}

// Normative scores for an explicit token list (sparse_attention, query.cpp:349-354).
template <typename T, int DP>
__global__ void token_scores_kernel(const T* __restrict__ Ks, const unsigned* __restrict__ ids,
                                    long long ntok, const float* __restrict__ q, float scale,
                                    float* __restrict__ scores) {
    __shared__ float qs[DP];
    for (int c = threadIdx.x; c < DP; c += blockDim.x) qs[c] = q[c];
    __syncthreads();
    const long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x;
    if (i >= ntok) return;
    const T* row = Ks + (size_t)ids[i] * DP;
    float s = 0.0f;
    for (int c = 0; c < DP; ++c) s = __fadd_rn(s, __fmul_rn(qs[c], to_f<T>(row[c])));
    scores[i] = scale * s;
}

// Per-split softmax partials over scored tokens: (m, l, o[DP]) unnormalised.
template <typename T, int DP>
__global__ void token_partials_kernel(const T* __restrict__ Vs, const unsigned* __restrict__ ids,
                                      const float* __restrict__ scores, long long ntok, int per,
                                      float* __restrict__ part) {
    __shared__ float red[8];
    __shared__ float acc[DP];
    const long long b = (long long)blockIdx.x * per;
    const long long e = b + per < ntok ? b + per : ntok;
    float m = -INFINITY;
    for (long long i = b + threadIdx.x; i < e; i += blockDim.x) m = fmaxf(m, scores[i]);
    m = warp_max(m);
    if ((threadIdx.x & 31) == 0) red[threadIdx.x >> 5] = m;
    for (int c = threadIdx.x; c < DP; c += blockDim.x) acc[c] = 0.0f;
    __syncthreads();
    m = -INFINITY;
    for (int w = 0; w < (int)(blockDim.x >> 5); ++w) m = fmaxf(m, red[w]);
    // each thread owns coordinates c = tid, tid + blockDim ...; l is summed by all
    float l = 0.0f;
    for (long long i = b; i < e; ++i) {
        const float p = expf(scores[i] - m);
        l += p;
        const T* row = Vs + (size_t)ids[i] * DP;
        for (int c = threadIdx.x; c < DP; c += blockDim.x) acc[c] = fmaf(p, to_f<T>(row[c]), acc[c]);
    }
    __syncthreads();
    float* out = part + (size_t)blockIdx.x * (DP + 2);
    if (threadIdx.x == 0) {
        out[0] = m;
        out[1] = l;
    }
    for (int c = threadIdx.x; c < DP; c += blockDim.x) out[2 + c] = acc[c];
}

// out[row][c] = sum_p o_p e^{m_p - M} / sum_p l_p e^{m_p - M}; optionally (M, L).
__global__ void lse_merge_kernel(const float* __restrict__ part, int P, long long rows, int d,
                                 int in_stride, float* __restrict__ out, int out_stride,
                                 float* __restrict__ ml) {
    const long long row = blockIdx.x;
    __shared__ float w[64];
    __shared__ float ML[2];
    if (threadIdx.x == 0) {
        float M = -INFINITY;
        for (int p = 0; p < P; ++p) M = fmaxf(M, part[((size_t)p * rows + row) * in_stride]);
        float L = 0.0f;
        for (int p = 0; p < P; ++p) {
            const float mp = part[((size_t)p * rows + row) * in_stride];
            const float wp = mp == -INFINITY ? 0.0f : expf(mp - M);
            w[p] = wp;
            L += wp * part[((size_t)p * rows + row) * in_stride + 1];
        }
        ML[0] = M;
        ML[1] = L;
    }
    __syncthreads();
    for (int c = threadIdx.x; c < d; c += blockDim.x) {
        float acc = 0.0f;
        for (int p = 0; p < P; ++p)
            if (w[p] != 0.0f) acc = fmaf(w[p], part[((size_t)p * rows + row) * in_stride + 2 + c], acc);
        out[(size_t)row * out_stride + c] = ML[1] > 0.0f ? acc / ML[1] : 0.0f;
    }
    if (ml && threadIdx.x == 0) {
        ml[2 * row] = ML[0];
        ml[2 * row + 1] = ML[1];
    }
}

// derive_subspace_thresholds (query.cpp:305-336) over the device cells: block s computes,
// over cells [0, ncells), M_s = max of the AABB bound sum_{c in s} max(q_c lo_c, q_c hi_c)
// (gate_bounds' order, float) and the norm bound max ||max(|lo|, |hi|)||_s (double,
// append_gate_entry index.cpp:147-154)
template <typename T, int DP>
__global__ void subspace_peaks_kernel(const T* __restrict__ rows, long long ncells, const float* __restrict__ q,
                                      const int* __restrict__ offs, double* __restrict__ peak,
                                      double* __restrict__ nb) {
    __shared__ double red[2][8];
    const int s = blockIdx.x, b = offs[s], e = offs[s + 1];
    double pk = -INFINITY, nq = 0.0;
    for (long long cell = threadIdx.x; cell < ncells; cell += blockDim.x) {
        const T* row = rows + (size_t)cell * 2 * DP;  // [hi (DP) | lo (DP)]
        float f = 0.0f;
        double sq = 0.0;
        for (int c = b; c < e; ++c) {
            const float h = to_f<T>(row[c]), l = to_f<T>(row[DP + c]);
            f = __fadd_rn(f, fmaxf(__fmul_rn(q[c], l), __fmul_rn(q[c], h)));
            const double m = fmax(fabs((double)l), fabs((double)h));
            sq += m * m;
        }
        pk = fmax(pk, (double)f);
        nq = fmax(nq, sqrt(sq));
    }
    for (int o = 16; o > 0; o >>= 1) {
        pk = fmax(pk, __shfl_xor_sync(0xffffffffu, pk, o));
        nq = fmax(nq, __shfl_xor_sync(0xffffffffu, nq, o));
    }
    if ((threadIdx.x & 31) == 0) {
        red[0][threadIdx.x >> 5] = pk;
        red[1][threadIdx.x >> 5] = nq;
    }
    __syncthreads();
    if (threadIdx.x == 0) {
        for (int w = 1; w < (int)(blockDim.x >> 5); ++w) {
            pk = fmax(pk, red[0][w]);
            nq = fmax(nq, red[1][w]);
        }
        peak[s] = fmax(pk, red[0][0]);
        nb[s] = fmax(nq, red[1][0]);
    }
}

// exact_check (query.cpp:22-31): flag[i] = normative dot(q, k_ids[i]) >= tau
template <typename T, int DP>
__global__ void exact_flags_kernel(const T* __restrict__ Ks, const unsigned* __restrict__ ids, long long nids,
                                   const float* __restrict__ q, float tau, unsigned char* __restrict__ flags) {
    __shared__ float qs[DP];
    for (int c = threadIdx.x; c < DP; c += blockDim.x) qs[c] = q[c];
    __syncthreads();
    const long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x;
    if (i >= nids) return;
    const T* row = Ks + (size_t)ids[i] * DP;
    float s = 0.0f;
    for (int c = 0; c < DP; ++c) s = __fadd_rn(s, __fmul_rn(qs[c], to_f<T>(row[c])));
    flags[i] = s >= tau ? 1 : 0;
}

// weights_i = exp(s_i - m) / l for a query's own (m, l)
__global__ void attn_weights_kernel(float* __restrict__ s, long long n, float m, float l) {
    const long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x;
    if (i < n) s[i] = expf(s[i] - m) / l;
}

// weights_i = exp(s_i - M) / L  (query.cpp:359-365)
__global__ void token_weights_kernel(const float* __restrict__ scores, long long ntok,
                                     const float* __restrict__ ml, float* __restrict__ w) {
    const long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x;
    if (i < ntok) w[i] = expf(scores[i] - ml[0]) / ml[1];
}

// Ascending id lists from bitmaps: one CTA per row.
__global__ void bitmap_ids_kernel(const unsigned* __restrict__ bits, long long words,
                                  long long limit, unsigned* __restrict__ ids, long long stride,
                                  int* __restrict__ count) {
    __shared__ int wsum[32];
    __shared__ int base_s;
    const long long row = blockIdx.x;
    const unsigned* b = bits + row * words;
    unsigned* out = ids + row * stride;
    const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5, nw = blockDim.x >> 5;
    if (tid == 0) base_s = 0;
    __syncthreads();
    const long long lw = (limit + 31) >> 5;
    for (long long w0 = 0; w0 < lw; w0 += blockDim.x) {
        const long long w = w0 + tid;
        unsigned v = w < lw ? b[w] : 0u;
        if (w == lw - 1 && (limit & 31)) v &= (1u << (limit & 31)) - 1u;
        const int c = __popc(v);
        int incl = c;
#pragma unroll
        for (int o = 1; o < 32; o <<= 1) {
            const int t = __shfl_up_sync(0xffffffffu, incl, o);
            if (lane >= o) incl += t;
        }
        if (lane == 31) wsum[warp] = incl;
        __syncthreads();
        int off = base_s;
        for (int i = 0; i < warp; ++i) off += wsum[i];
        off += incl - c;
        while (v) {
            const int bit = __ffs(v) - 1;
            out[off++] = (unsigned)(w * 32 + bit);
            v &= v - 1;
        }
        __syncthreads();
        if (tid == 0) {
            int tot = 0;
            for (int i = 0; i < nw; ++i) tot += wsum[i];
            base_s += tot;
        }
        __syncthreads();
    }
    if (tid == 0) count[row] = base_s;
}

}  // namespace lvk
