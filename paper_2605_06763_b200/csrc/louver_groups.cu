// Grouped index on the device (see louver_groups.h): the reference's BuildConfig
// groupings and enclosures over the HBM key arena, with the exact floating-point
// operation order of index.cpp / query.cpp, so assignments, enclosures, candidate sets
// and statistics equal the reference's (checked against the compiled reference and the
// oracle in tests/test_groups.py).
//
// Grouping shapes (group count, member count per group, the PCA tree's segments) depend
// only on the block size m and r, so the host plans them and the device fills the
// data-dependent parts: the PCA split axes and orders, the member ids, the enclosures.
#include "louver_groups.h"

#include <cuda_bf16.h>

#include <algorithm>
#include <cmath>
#include <cstring>
#include <numeric>
#include <random>

#include <cub/device/device_segmented_sort.cuh>

namespace lvg {

namespace {

__device__ __forceinline__ float kval(const ArenaView& a, int slot, long long row, int col) {
    const size_t i = ((size_t)slot * a.cap + (size_t)row) * a.DP + col;
    return a.bf16 ? __bfloat162float(reinterpret_cast<const __nv_bfloat16*>(a.K)[i])
                  : reinterpret_cast<const float*>(a.K)[i];
}

// float order as an unsigned key; -0 and +0 compare equal in pca_split's sort (index.cpp:45-49)
__device__ __forceinline__ unsigned ord_key(float x) {
    unsigned b = __float_as_uint(x);
    if (b == 0x80000000u) b = 0u;
    return (b & 0x80000000u) ? ~b : (b | 0x80000000u);
}
// rank_key (query.cpp:125-128): signed zeros stay distinct
__device__ __forceinline__ unsigned rank_key(float x) {
    const unsigned b = __float_as_uint(x);
    return (b & 0x80000000u) ? ~b : (b | 0x80000000u);
}

struct Dev {  // kernel-side view of a GroupIndex
    int S, r, enclosure, wmax;
    long long cap, kcap;
    unsigned *assign, *moff, *mids;
    float *ga, *gb, *grad;
    unsigned long long* nbound;
    int off[65];
};

Dev view(const GroupIndex& gi) {
    Dev v{};
    v.S = gi.S;
    v.r = gi.r;
    v.enclosure = gi.enclosure;
    v.wmax = gi.wmax;
    v.cap = gi.cap;
    v.kcap = gi.kcap;
    v.assign = gi.assign;
    v.moff = gi.moff;
    v.mids = gi.mids;
    v.ga = gi.ga;
    v.gb = gi.gb;
    v.grad = gi.grad;
    v.nbound = gi.nbound;
    for (int s = 0; s <= gi.S; ++s) v.off[s] = gi.off[s];
    return v;
}

// ---- PCA tree (index.cpp:15-56), one level of every pair's tree at a time -------------

// Block (segment, pair): thread c computes coordinate c's mean and variance over the
// segment in its current order, in double, exactly as pca_split's loops; the block keeps
// the largest variance, ties toward the lowest coordinate.
__global__ void pca_axis_kernel(ArenaView a, Dev g, const unsigned* ids, int m, long long first, const int2* segs,
                                int* axis) {
    const int p = blockIdx.y, slot = p / g.S, s = p % g.S, c = threadIdx.x;
    const int w = g.off[s + 1] - g.off[s];
    const int2 sg = segs[blockIdx.x];
    const unsigned* id = ids + (size_t)p * m + sg.x;
    double var = -1.0;
    if (c < w) {
        const int col = g.off[s] + c;
        double mean = 0.0;
        for (int i = 0; i < sg.y; ++i) mean = __dadd_rn(mean, (double)kval(a, slot, first + id[i], col));
        mean = __ddiv_rn(mean, (double)sg.y);
        var = 0.0;
        for (int i = 0; i < sg.y; ++i) {
            const double dv = __dsub_rn((double)kval(a, slot, first + id[i], col), mean);
            var = __dadd_rn(var, __dmul_rn(dv, dv));
        }
    }
    __shared__ double sv[256];
    __shared__ int sc[256];
    sv[c] = var;
    sc[c] = c;
    __syncthreads();
    for (int h = blockDim.x / 2; h > 0; h >>= 1) {
        if (c < h) {
            const double v2 = sv[c + h];
            const int c2 = sc[c + h];
            if (v2 > sv[c] || (v2 == sv[c] && c2 < sc[c])) {
                sv[c] = v2;
                sc[c] = c2;
            }
        }
        __syncthreads();
    }
    if (c == 0) axis[(size_t)p * gridDim.x + blockIdx.x] = sc[0];
}

// Sort keys of one level: active segments by (coordinate on their axis, id) — the
// comparator of index.cpp:45-49 —, every other segment by id (its order is irrelevant).
__global__ void pca_keys_kernel(ArenaView a, Dev g, const unsigned* ids, int m, long long first, const int* seg_of_pos,
                                const int* axis, int nact, unsigned long long* keys) {
    const int p = blockIdx.y, slot = p / g.S, s = p % g.S;
    const int pos = blockIdx.x * blockDim.x + threadIdx.x;
    if (pos >= m) return;
    const unsigned id = ids[(size_t)p * m + pos];
    const int si = seg_of_pos[pos];
    unsigned long long k = id;
    if (si >= 0) {
        const int col = g.off[s] + axis[(size_t)p * nact + si];
        k |= (unsigned long long)ord_key(kval(a, slot, first + id, col)) << 32;
    }
    keys[(size_t)p * m + pos] = k;
}

__global__ void low32_kernel(const unsigned long long* keys, unsigned* ids, long long total) {
    const long long i = (long long)blockIdx.x * blockDim.x + threadIdx.x;
    if (i < total) ids[i] = (unsigned)keys[i];
}

// ids in group order for the shapes that need no data: contiguous (identity),
// interleaved (group gg holds gg, gg + K, ...), random (the host's permutation)
__global__ void order_kernel(int grouping, int m, int Kl, const unsigned* perm, const unsigned* gstart,
                             unsigned long long* keys, int S) {
    const int p = blockIdx.y;
    const int pos = blockIdx.x * blockDim.x + threadIdx.x;
    if (pos >= m) return;
    unsigned id = pos;
    if (grouping == 1) {  // interleaved
        int lo = 0, hi = Kl;  // group of position pos: last gg with gstart[gg] <= pos
        while (hi - lo > 1) {
            const int mid = (lo + hi) / 2;
            if ((int)gstart[mid] <= pos) lo = mid; else hi = mid;
        }
        id = (unsigned)lo + (unsigned)(pos - (int)gstart[lo]) * (unsigned)Kl;
    } else if (grouping == 2) {  // random: perm of subspace s
        id = perm[(size_t)(p % S) * m + pos];
    }
    keys[(size_t)p * m + pos] = id;
}

// group-ordered ids (ascending within each group) -> member lists and assignments
__global__ void members_kernel(Dev g, const unsigned* ids, const unsigned* pos_group, int m, long long first,
                               long long gbase) {
    const int p = blockIdx.y;
    const int pos = blockIdx.x * blockDim.x + threadIdx.x;
    if (pos >= m) return;
    const unsigned id = ids[(size_t)p * m + pos];
    g.mids[(size_t)p * g.cap + first + pos] = (unsigned)(first + id);
    g.assign[(size_t)p * g.cap + first + id] = (unsigned)(gbase + pos_group[pos]);
}

__global__ void moff_kernel(Dev g, const unsigned* loc, int Kl, long long first, long long gbase) {
    const int p = blockIdx.y;
    const int i = blockIdx.x * blockDim.x + threadIdx.x;
    if (i <= Kl) g.moff[(size_t)p * (g.kcap + 1) + gbase + i] = (unsigned)(first + loc[i]);
}

// enclose_group (index.cpp:104-137) + append_gate_entry's packed arrays and norm bound
// (index.cpp:139-168): one warp per group, lanes over coordinates; every reduction runs
// in the reference's member order (ascending ids).
__global__ void enclose_kernel(ArenaView a, Dev g, long long gbase) {
    const int p = blockIdx.y, slot = p / g.S, s = p % g.S, lane = threadIdx.x;
    const long long gg = gbase + blockIdx.x;
    const int w = g.off[s + 1] - g.off[s], col0 = g.off[s];
    const unsigned t0 = g.moff[(size_t)p * (g.kcap + 1) + gg], t1 = g.moff[(size_t)p * (g.kcap + 1) + gg + 1];
    const unsigned* mem = g.mids + (size_t)p * g.cap;
    const int cnt = (int)(t1 - t0);
    extern __shared__ float sh[];
    float* ctr = sh;        // [w]
    float* slo = sh + w;    // [w]
    float* shi = sh + 2 * w;
    const size_t gi = (size_t)p * g.wmax * g.kcap;
    for (int c = lane; c < w; c += 32) {
        float lo = kval(a, slot, mem[t0], col0 + c), hi = lo;
        for (int t = 1; t < cnt; ++t) {  // colwise min/max: std::min/std::max keep the first on ties
            const float x = kval(a, slot, mem[t0 + t], col0 + c);
            lo = x < lo ? x : lo;
            hi = hi < x ? x : hi;
        }
        slo[c] = lo;
        shi[c] = hi;
        float cv;
        if (g.enclosure == 1) {  // AABB
            g.ga[gi + (size_t)c * g.kcap + gg] = lo;
            g.gb[gi + (size_t)c * g.kcap + gg] = hi;
            continue;
        } else if (g.enclosure == 0) {  // ball: mean accumulated in double, cast to float
            double acc = 0.0;
            for (int t = 0; t < cnt; ++t) acc = __dadd_rn(acc, (double)kval(a, slot, mem[t0 + t], col0 + c));
            cv = (float)__ddiv_rn(acc, (double)cnt);
        } else {  // span_ball: 0.5f * (lo + hi)
            cv = __fmul_rn(0.5f, __fadd_rn(lo, hi));
        }
        ctr[c] = cv;
        g.ga[gi + (size_t)c * g.kcap + gg] = cv;
    }
    __syncwarp();
    double b = 0.0;
    if (g.enclosure == 1) {
        if (lane == 0) {
            double sq = 0.0;
            for (int c = 0; c < w; ++c) {
                const double x = fabs((double)slo[c]), y = fabs((double)shi[c]);
                const double mx = x < y ? y : x;
                sq = __dadd_rn(sq, __dmul_rn(mx, mx));
            }
            b = __dsqrt_rn(sq);
        }
    } else {
        float rad = 0.0f;  // max over members of norm2(p - center), core.hpp:29-31 (sequential dot)
        for (int t = lane; t < cnt; t += 32) {
            float acc = 0.0f;
            for (int c = 0; c < w; ++c) {
                const float df = __fsub_rn(kval(a, slot, mem[t0 + t], col0 + c), ctr[c]);
                acc = __fadd_rn(acc, __fmul_rn(df, df));
            }
            const float nr = __fsqrt_rn(acc);
            rad = rad < nr ? nr : rad;
        }
#pragma unroll
        for (int o = 16; o > 0; o >>= 1) rad = fmaxf(rad, __shfl_xor_sync(0xffffffffu, rad, o));
        if (lane == 0) {
            if (rad > 0.0f) rad = nextafterf(rad, INFINITY);  // one ulp of headroom
            g.grad[(size_t)p * g.kcap + gg] = rad;
            float sq = 0.0f;
            for (int c = 0; c < w; ++c) sq = __fadd_rn(sq, __fmul_rn(ctr[c], ctr[c]));
            b = __dadd_rn((double)__fsqrt_rn(sq), (double)rad);
        }
    }
    if (lane == 0) atomicMax(g.nbound + p, (unsigned long long)__double_as_longlong(b));
}

// ---- queries -----------------------------------------------------------------------

// gate_bounds (query.cpp:47-68) for every group of every subspace of one slot
__global__ void bounds_kernel(Dev g, int slot, long long K, const float* q, float* out) {
    const int s = blockIdx.y, p = slot * g.S + s;
    const long long i = (long long)blockIdx.x * blockDim.x + threadIdx.x;
    if (i >= K) return;
    const int w = g.off[s + 1] - g.off[s];
    const float* qs = q + g.off[s];
    const size_t gi = (size_t)p * g.wmax * g.kcap;
    float acc = 0.0f;
    if (g.enclosure == 1) {
        for (int c = 0; c < w; ++c) {
            const float x = __fmul_rn(qs[c], g.ga[gi + (size_t)c * g.kcap + i]);
            const float y = __fmul_rn(qs[c], g.gb[gi + (size_t)c * g.kcap + i]);
            acc = __fadd_rn(acc, x < y ? y : x);  // std::max(q*lo, q*hi)
        }
    } else {
        for (int c = 0; c < w; ++c) acc = __fadd_rn(acc, __fmul_rn(qs[c], g.ga[gi + (size_t)c * g.kcap + i]));
        float qq = 0.0f;
        for (int c = 0; c < w; ++c) qq = __fadd_rn(qq, __fmul_rn(qs[c], qs[c]));
        acc = __fadd_rn(acc, __fmul_rn(g.grad[(size_t)p * g.kcap + i], __fsqrt_rn(qq)));
    }
    out[(size_t)s * K + i] = acc;
}

// members of the groups with bound >= tau_s set their bit in the subspace's bitmap
__global__ void mark_kernel(Dev g, int slot, long long K, const float* bounds, const float* tau_s, unsigned* bits,
                            long long words) {
    const int s = blockIdx.y, p = slot * g.S + s;
    const long long i = (long long)blockIdx.x * blockDim.x + threadIdx.x;
    if (i >= K || bounds[(size_t)s * K + i] < tau_s[s]) return;  // inclusive predicate
    const unsigned* off = g.moff + (size_t)p * (g.kcap + 1);
    const unsigned* mem = g.mids + (size_t)p * g.cap;
    for (unsigned t = off[i]; t < off[i + 1]; ++t) atomicOr(bits + (size_t)s * words + (mem[t] >> 5), 1u << (mem[t] & 31));
}

__global__ void and_kernel(const unsigned* bits, int S, long long words, unsigned* live) {
    const long long i = (long long)blockIdx.x * blockDim.x + threadIdx.x;
    if (i >= words) return;
    unsigned x = bits[i];
    for (int s = 1; s < S; ++s) x &= bits[(size_t)s * words + i];
    live[i] = x;
}

// TA scan order: bound descending, ties by ascending group id (query.cpp:213-221)
__global__ void ta_keys_kernel(const float* bounds, long long K, int S, unsigned long long* keys) {
    const long long i = (long long)blockIdx.x * blockDim.x + threadIdx.x;
    if (i >= K * S) return;
    keys[i] = ((unsigned long long)(~rank_key(bounds[i])) << 32) | (unsigned)(i % K);
}

// U(d) = sum over subspaces of the d-th ranked bound, in double, subspace order; the
// first d with U(d) < tau halts the scan (query.cpp:238-251)
__global__ void ta_upper_kernel(const unsigned long long* sorted, const float* bounds, long long K, int S, float tau,
                                double* U, unsigned long long* dstar) {
    const long long d = (long long)blockIdx.x * blockDim.x + threadIdx.x + 1;
    if (d > K) return;
    double u = 0.0;
    for (int s = 0; s < S; ++s) u = __dadd_rn(u, (double)bounds[(size_t)s * K + (unsigned)sorted[(size_t)s * K + d - 1]]);
    U[d - 1] = u;
    if (u < (double)tau) atomicMin(dstar, (unsigned long long)d);
}

__global__ void ta_mark_kernel(Dev g, int slot, long long K, const unsigned long long* sorted, long long depth,
                               unsigned* live) {
    const int s = blockIdx.y, p = slot * g.S + s;
    const long long i = (long long)blockIdx.x * blockDim.x + threadIdx.x;
    if (i >= depth) return;
    const unsigned gg = (unsigned)sorted[(size_t)s * K + i];
    const unsigned* off = g.moff + (size_t)p * (g.kcap + 1);
    const unsigned* mem = g.mids + (size_t)p * g.cap;
    for (unsigned t = off[gg]; t < off[gg + 1]; ++t) atomicOr(live + (mem[t] >> 5), 1u << (mem[t] & 31));
}

__global__ void popc_kernel(const unsigned* bits, long long words, unsigned long long* out) {
    unsigned long long c = 0;
    for (long long i = (long long)blockIdx.x * blockDim.x + threadIdx.x; i < words; i += (long long)gridDim.x * blockDim.x)
        c += __popc(bits[i]);
    for (int o = 16; o > 0; o >>= 1) c += __shfl_xor_sync(0xffffffffu, c, o);
    if ((threadIdx.x & 31) == 0 && c) atomicAdd(out, c);
}

__global__ void peaks_kernel(const float* bounds, long long K, double* peak) {
    const int s = blockIdx.x;
    double m = -INFINITY;
    for (long long i = threadIdx.x; i < K; i += blockDim.x) m = fmax(m, (double)bounds[(size_t)s * K + i]);
    __shared__ double sm[256];
    sm[threadIdx.x] = m;
    __syncthreads();
    for (int h = blockDim.x / 2; h > 0; h >>= 1) {
        if (threadIdx.x < h) sm[threadIdx.x] = fmax(sm[threadIdx.x], sm[threadIdx.x + h]);
        __syncthreads();
    }
    if (threadIdx.x == 0) peak[s] = sm[0];
}

// ---- host-side planning of the data-independent shapes -------------------------------

struct Plan {
    int Kl = 0;                        // groups of the block
    std::vector<unsigned> gstart;      // [Kl + 1] position offsets of the groups
    std::vector<unsigned> pos_group;   // [m]
    std::vector<std::vector<int2>> levels;  // PCA: every level's segments (start, len)
};

Plan plan_block(int grouping, int m, int r) {
    Plan pl;
    if (grouping == 3) {  // PCA tree: median bisection until segments hold <= r points
        std::vector<int2> seg{{0, m}};
        for (;;) {
            pl.levels.push_back(seg);
            bool any = false;
            std::vector<int2> nx;
            for (const int2& x : seg) {
                if (x.y > r) {
                    const int left = x.y / 2;
                    nx.push_back({x.x, left});
                    nx.push_back({x.x + left, x.y - left});
                    any = true;
                } else {
                    nx.push_back(x);
                }
            }
            seg.swap(nx);
            if (!any) break;
        }
        pl.levels.push_back(seg);  // final: every segment a leaf (sorted by id)
        pl.Kl = (int)seg.size();
        pl.gstart.resize(pl.Kl + 1);
        for (int i = 0; i < pl.Kl; ++i) pl.gstart[i] = seg[i].x;
        pl.gstart[pl.Kl] = m;
    } else if (grouping == 1) {  // interleaved: K = ceil(m / r), group gg = {j : j % K == gg}
        pl.Kl = (m + r - 1) / r;
        pl.gstart.resize(pl.Kl + 1);
        unsigned acc = 0;
        for (int gg = 0; gg < pl.Kl; ++gg) {
            pl.gstart[gg] = acc;
            acc += (unsigned)((m - gg + pl.Kl - 1) / pl.Kl);
        }
        pl.gstart[pl.Kl] = acc;
    } else {  // contiguous, random: groups of r positions
        pl.Kl = (m + r - 1) / r;
        pl.gstart.resize(pl.Kl + 1);
        for (int gg = 0; gg <= pl.Kl; ++gg) pl.gstart[gg] = (unsigned)std::min<long long>((long long)gg * r, m);
    }
    pl.pos_group.resize(m);
    for (int gg = 0; gg < pl.Kl; ++gg)
        for (unsigned i = pl.gstart[gg]; i < pl.gstart[gg + 1]; ++i) pl.pos_group[i] = gg;
    return pl;
}

// assign_groups' Random case (index.cpp:84-94): the permutation depends only on the
// seed, the subspace and the block's first id, never on the keys
std::vector<unsigned> random_perm(unsigned long long seed, int s, unsigned base_id, int m) {
    std::seed_seq seq{static_cast<std::uint32_t>(seed), static_cast<std::uint32_t>(seed >> 32),
                      static_cast<std::uint32_t>(s), static_cast<std::uint32_t>(base_id)};
    std::mt19937_64 rng(seq);
    std::vector<unsigned> perm(m);
    std::iota(perm.begin(), perm.end(), 0u);
    std::shuffle(perm.begin(), perm.end(), rng);
    return perm;
}

template <class T>
cudaError_t dalloc(T** p, size_t n) {
    return cudaMalloc(reinterpret_cast<void**>(p), sizeof(T) * std::max<size_t>(n, 1));
}

}  // namespace

#define LVG_TRY(x)                               \
    do {                                         \
        cudaError_t e_ = (x);                    \
        if (e_ != cudaSuccess) return e_;        \
    } while (0)

cudaError_t create(GroupIndex& gi, int d, int S, int r, int grouping, int enclosure, unsigned long long seed,
                   int slots, long long cap) {
    if (S > 64) return cudaErrorInvalidValue;
    gi.S = S;
    gi.d = d;
    gi.r = r;
    gi.grouping = grouping;
    gi.enclosure = enclosure;
    gi.seed = seed;
    gi.slots = slots;
    gi.off.assign(S + 1, 0);
    for (int s = 0; s < S; ++s) gi.off[s + 1] = gi.off[s] + d / S + (s < d % S ? 1 : 0);  // core.hpp:41-50
    gi.wmax = d / S + (d % S ? 1 : 0);
    gi.indexed = 0;
    gi.K = 0;
    gi.cap = 0;
    return reserve(gi, cap, 0);
}

void destroy(GroupIndex& gi) {
    cudaFree(gi.assign);
    cudaFree(gi.moff);
    cudaFree(gi.mids);
    cudaFree(gi.ga);
    cudaFree(gi.gb);
    cudaFree(gi.grad);
    cudaFree(gi.nbound);
    gi.assign = gi.moff = gi.mids = nullptr;
    gi.ga = gi.gb = gi.grad = nullptr;
    gi.nbound = nullptr;
}

cudaError_t reserve(GroupIndex& gi, long long cap, cudaStream_t st) {
    if (cap <= gi.cap) return cudaSuccess;
    const size_t P = (size_t)gi.slots * gi.S;
    const long long kcap = cap;  // groups never outnumber keys
    GroupIndex nw = gi;
    nw.cap = cap;
    nw.kcap = kcap;
    nw.assign = nw.moff = nw.mids = nullptr;
    nw.ga = nw.gb = nw.grad = nullptr;
    nw.nbound = nullptr;
    auto undo = [&](cudaError_t e) {
        destroy(nw);
        return e;
    };
    cudaError_t e;
    if ((e = dalloc(&nw.assign, P * cap)) != cudaSuccess) return undo(e);
    if ((e = dalloc(&nw.moff, P * (kcap + 1))) != cudaSuccess) return undo(e);
    if ((e = dalloc(&nw.mids, P * cap)) != cudaSuccess) return undo(e);
    if ((e = dalloc(&nw.ga, P * gi.wmax * kcap)) != cudaSuccess) return undo(e);
    if (gi.enclosure == 1 && (e = dalloc(&nw.gb, P * gi.wmax * kcap)) != cudaSuccess) return undo(e);
    if (gi.enclosure != 1 && (e = dalloc(&nw.grad, P * kcap)) != cudaSuccess) return undo(e);
    if ((e = dalloc(&nw.nbound, P)) != cudaSuccess) return undo(e);
    LVG_TRY(cudaMemsetAsync(nw.nbound, 0, sizeof(unsigned long long) * P, st));
    LVG_TRY(cudaMemsetAsync(nw.moff, 0, sizeof(unsigned) * P * (kcap + 1), st));
    if (gi.cap > 0) {  // keep the contents
        LVG_TRY(cudaMemcpy2DAsync(nw.assign, sizeof(unsigned) * cap, gi.assign, sizeof(unsigned) * gi.cap,
                                  sizeof(unsigned) * gi.cap, P, cudaMemcpyDeviceToDevice, st));
        LVG_TRY(cudaMemcpy2DAsync(nw.mids, sizeof(unsigned) * cap, gi.mids, sizeof(unsigned) * gi.cap,
                                  sizeof(unsigned) * gi.cap, P, cudaMemcpyDeviceToDevice, st));
        LVG_TRY(cudaMemcpy2DAsync(nw.moff, sizeof(unsigned) * (kcap + 1), gi.moff, sizeof(unsigned) * (gi.kcap + 1),
                                  sizeof(unsigned) * (gi.kcap + 1), P, cudaMemcpyDeviceToDevice, st));
        LVG_TRY(cudaMemcpy2DAsync(nw.ga, sizeof(float) * kcap, gi.ga, sizeof(float) * gi.kcap, sizeof(float) * gi.kcap,
                                  P * gi.wmax, cudaMemcpyDeviceToDevice, st));
        if (gi.gb)
            LVG_TRY(cudaMemcpy2DAsync(nw.gb, sizeof(float) * kcap, gi.gb, sizeof(float) * gi.kcap,
                                      sizeof(float) * gi.kcap, P * gi.wmax, cudaMemcpyDeviceToDevice, st));
        if (gi.grad)
            LVG_TRY(cudaMemcpy2DAsync(nw.grad, sizeof(float) * kcap, gi.grad, sizeof(float) * gi.kcap,
                                      sizeof(float) * gi.kcap, P, cudaMemcpyDeviceToDevice, st));
        LVG_TRY(cudaMemcpyAsync(nw.nbound, gi.nbound, sizeof(unsigned long long) * P, cudaMemcpyDeviceToDevice, st));
        LVG_TRY(cudaStreamSynchronize(st));
        destroy(gi);
    }
    gi = nw;
    return cudaSuccess;
}

cudaError_t index_range(GroupIndex& gi, const ArenaView& a, long long first, long long count, cudaStream_t st) {
    if (count <= 0) return cudaSuccess;
    if (first != gi.indexed || first + count > gi.cap || count >= (1LL << 31)) return cudaErrorInvalidValue;
    const int m = (int)count, S = gi.S, P = gi.slots * S;
    const Plan pl = plan_block(gi.grouping, m, gi.r);
    if (gi.K + pl.Kl > gi.kcap) return cudaErrorInvalidValue;
    const Dev dv = view(gi);
    const size_t PM = (size_t)P * m;
    // scratch: two key buffers, ids, plan arrays
    unsigned long long *k0 = nullptr, *k1 = nullptr;
    unsigned *ids = nullptr, *pg = nullptr, *gs = nullptr, *perm = nullptr;
    LVG_TRY(cudaMallocAsync(&k0, sizeof(unsigned long long) * PM, st));
    LVG_TRY(cudaMallocAsync(&k1, sizeof(unsigned long long) * PM, st));
    LVG_TRY(cudaMallocAsync(&ids, sizeof(unsigned) * PM, st));
    LVG_TRY(cudaMallocAsync(&pg, sizeof(unsigned) * m, st));
    LVG_TRY(cudaMallocAsync(&gs, sizeof(unsigned) * (pl.Kl + 1), st));
    LVG_TRY(cudaMemcpyAsync(pg, pl.pos_group.data(), sizeof(unsigned) * m, cudaMemcpyHostToDevice, st));
    LVG_TRY(cudaMemcpyAsync(gs, pl.gstart.data(), sizeof(unsigned) * (pl.Kl + 1), cudaMemcpyHostToDevice, st));
    std::vector<unsigned> hperm;
    if (gi.grouping == 2) {
        hperm.resize((size_t)S * m);
        for (int s = 0; s < S; ++s) {
            const auto pr = random_perm(gi.seed, s, (unsigned)first, m);
            std::copy(pr.begin(), pr.end(), hperm.begin() + (size_t)s * m);
        }
        LVG_TRY(cudaMallocAsync(&perm, sizeof(unsigned) * S * m, st));
        LVG_TRY(cudaMemcpyAsync(perm, hperm.data(), sizeof(unsigned) * S * m, cudaMemcpyHostToDevice, st));
    }
    const dim3 gpos((m + 255) / 256, P);
    // segmented sort of every pair's positions by key over the given segments
    std::vector<int> hb, he;
    auto seg_sort = [&](const std::vector<int2>& segs) -> cudaError_t {
        const int ns = (int)segs.size();
        hb.resize((size_t)P * ns);
        he.resize((size_t)P * ns);
        for (int p = 0; p < P; ++p)
            for (int i = 0; i < ns; ++i) {
                hb[(size_t)p * ns + i] = p * m + segs[i].x;
                he[(size_t)p * ns + i] = p * m + segs[i].x + segs[i].y;
            }
        int *db = nullptr, *de = nullptr;
        LVG_TRY(cudaMallocAsync(&db, sizeof(int) * hb.size(), st));
        LVG_TRY(cudaMallocAsync(&de, sizeof(int) * he.size(), st));
        LVG_TRY(cudaMemcpyAsync(db, hb.data(), sizeof(int) * hb.size(), cudaMemcpyHostToDevice, st));
        LVG_TRY(cudaMemcpyAsync(de, he.data(), sizeof(int) * he.size(), cudaMemcpyHostToDevice, st));
        size_t tb = 0;
        LVG_TRY(cub::DeviceSegmentedSort::SortKeys(nullptr, tb, k0, k1, (int)PM, (int)hb.size(), db, de, st));
        void* tmp = nullptr;
        LVG_TRY(cudaMallocAsync(&tmp, std::max<size_t>(tb, 1), st));
        LVG_TRY(cub::DeviceSegmentedSort::SortKeys(tmp, tb, k0, k1, (int)PM, (int)hb.size(), db, de, st));
        LVG_TRY(cudaFreeAsync(tmp, st));
        LVG_TRY(cudaFreeAsync(db, st));
        LVG_TRY(cudaFreeAsync(de, st));
        low32_kernel<<<(unsigned)((PM + 255) / 256), 256, 0, st>>>(k1, ids, (long long)PM);
        return cudaGetLastError();
    };
    if (gi.grouping == 3) {
        // balanced PCA tree: ids start as the identity; each level computes the split axis of
        // every segment larger than r and sorts it by (coordinate, id)
        order_kernel<<<gpos, 256, 0, st>>>(0, m, pl.Kl, nullptr, gs, k0, S);
        low32_kernel<<<(unsigned)((PM + 255) / 256), 256, 0, st>>>(k0, ids, (long long)PM);
        int* seg_of_pos = nullptr;
        int* axis = nullptr;
        int2* dsegs = nullptr;
        LVG_TRY(cudaMallocAsync(&seg_of_pos, sizeof(int) * m, st));
        std::vector<int> hsp(m);
        for (size_t L = 0; L < pl.levels.size(); ++L) {
            const auto& segs = pl.levels[L];
            std::vector<int2> act;
            std::fill(hsp.begin(), hsp.end(), -1);
            for (const int2& x : segs)
                if (x.y > gi.r) {
                    for (int i = 0; i < x.y; ++i) hsp[x.x + i] = (int)act.size();
                    act.push_back(x);
                }
            const int nact = (int)act.size();
            LVG_TRY(cudaMemcpyAsync(seg_of_pos, hsp.data(), sizeof(int) * m, cudaMemcpyHostToDevice, st));
            if (nact > 0) {
                LVG_TRY(cudaMallocAsync(&dsegs, sizeof(int2) * nact, st));
                LVG_TRY(cudaMallocAsync(&axis, sizeof(int) * (size_t)P * nact, st));
                LVG_TRY(cudaMemcpyAsync(dsegs, act.data(), sizeof(int2) * nact, cudaMemcpyHostToDevice, st));
                int thr = 32;  // a power of two >= the subspace width (block tree reduction)
                while (thr < gi.wmax) thr *= 2;
                pca_axis_kernel<<<dim3(nact, P), thr, 0, st>>>(a, dv, ids, m, first, dsegs, axis);
                LVG_TRY(cudaGetLastError());
            }
            pca_keys_kernel<<<gpos, 256, 0, st>>>(a, dv, ids, m, first, seg_of_pos, axis, nact, k0);
            LVG_TRY(cudaGetLastError());
            LVG_TRY(seg_sort(segs));
            if (nact > 0) {
                LVG_TRY(cudaFreeAsync(dsegs, st));
                LVG_TRY(cudaFreeAsync(axis, st));
                dsegs = nullptr;
                axis = nullptr;
            }
            // the last level lists only leaves: every segment sorted by id -> member order
        }
        LVG_TRY(cudaFreeAsync(seg_of_pos, st));
    } else {
        order_kernel<<<gpos, 256, 0, st>>>(gi.grouping, m, pl.Kl, perm, gs, k0, S);
        LVG_TRY(cudaGetLastError());
        std::vector<int2> groups(pl.Kl);
        for (int gg = 0; gg < pl.Kl; ++gg) groups[gg] = {(int)pl.gstart[gg], (int)(pl.gstart[gg + 1] - pl.gstart[gg])};
        LVG_TRY(seg_sort(groups));  // members ascending within each group
    }
    members_kernel<<<gpos, 256, 0, st>>>(dv, ids, pg, m, first, gi.K);
    moff_kernel<<<dim3((pl.Kl + 1 + 255) / 256, P), 256, 0, st>>>(dv, gs, pl.Kl, first, gi.K);
    LVG_TRY(cudaGetLastError());
    enclose_kernel<<<dim3(pl.Kl, P), 32, sizeof(float) * 3 * gi.wmax, st>>>(a, dv, gi.K);
    LVG_TRY(cudaGetLastError());
    LVG_TRY(cudaFreeAsync(k0, st));
    LVG_TRY(cudaFreeAsync(k1, st));
    LVG_TRY(cudaFreeAsync(ids, st));
    LVG_TRY(cudaFreeAsync(pg, st));
    LVG_TRY(cudaFreeAsync(gs, st));
    if (perm) LVG_TRY(cudaFreeAsync(perm, st));
    gi.K += pl.Kl;
    gi.indexed = first + count;
    return cudaSuccess;
}

cudaError_t candidates(const GroupIndex& gi, int slot, const float* q, float tau, const float* tau_s, int algo,
                       unsigned* live_bits, Stats* stats, cudaStream_t st) {
    const long long n = gi.indexed, K = gi.K;
    const int S = gi.S;
    const long long words = (n + 31) / 32;
    Stats res;
    res.groups_tested = (long long)S * K;
    if (n > 0) {
        const Dev dv = view(gi);
        float *qd = nullptr, *bnd = nullptr, *ts = nullptr;
        unsigned* bits = nullptr;
        unsigned long long* cnt = nullptr;
        LVG_TRY(cudaMallocAsync(&qd, sizeof(float) * gi.d, st));
        LVG_TRY(cudaMallocAsync(&bnd, sizeof(float) * S * K, st));
        LVG_TRY(cudaMallocAsync(&cnt, sizeof(unsigned long long) * 2, st));
        LVG_TRY(cudaMemcpyAsync(qd, q, sizeof(float) * gi.d, cudaMemcpyHostToDevice, st));
        LVG_TRY(cudaMemsetAsync(cnt, 0, sizeof(unsigned long long) * 2, st));
        LVG_TRY(cudaMemsetAsync(live_bits, 0, sizeof(unsigned) * words, st));
        const dim3 gk((unsigned)((K + 255) / 256), S);
        bounds_kernel<<<gk, 256, 0, st>>>(dv, slot, K, qd, bnd);
        LVG_TRY(cudaGetLastError());
        if (algo == 0) {  // query_full_subspace: AND over subspaces of the groups at or above tau_s
            LVG_TRY(cudaMallocAsync(&ts, sizeof(float) * S, st));
            LVG_TRY(cudaMallocAsync(&bits, sizeof(unsigned) * S * words, st));
            LVG_TRY(cudaMemcpyAsync(ts, tau_s, sizeof(float) * S, cudaMemcpyHostToDevice, st));
            LVG_TRY(cudaMemsetAsync(bits, 0, sizeof(unsigned) * S * words, st));
            mark_kernel<<<gk, 256, 0, st>>>(dv, slot, K, bnd, ts, bits, words);
            and_kernel<<<(unsigned)((words + 255) / 256), 256, 0, st>>>(bits, S, words, live_bits);
            LVG_TRY(cudaGetLastError());
            LVG_TRY(cudaFreeAsync(ts, st));
            LVG_TRY(cudaFreeAsync(bits, st));
        } else {  // query_ta
            unsigned long long *k0 = nullptr, *k1 = nullptr;
            double* U = nullptr;
            int *db = nullptr, *de = nullptr;
            LVG_TRY(cudaMallocAsync(&k0, sizeof(unsigned long long) * S * K, st));
            LVG_TRY(cudaMallocAsync(&k1, sizeof(unsigned long long) * S * K, st));
            LVG_TRY(cudaMallocAsync(&U, sizeof(double) * K, st));
            LVG_TRY(cudaMallocAsync(&db, sizeof(int) * S * 2, st));
            de = db + S;
            std::vector<int> hb(2 * S);
            for (int s = 0; s < S; ++s) {
                hb[s] = (int)(s * K);
                hb[S + s] = (int)((s + 1) * K);
            }
            LVG_TRY(cudaMemcpyAsync(db, hb.data(), sizeof(int) * 2 * S, cudaMemcpyHostToDevice, st));
            ta_keys_kernel<<<(unsigned)((S * K + 255) / 256), 256, 0, st>>>(bnd, K, S, k0);
            size_t tb = 0;
            LVG_TRY(cub::DeviceSegmentedSort::SortKeys(nullptr, tb, k0, k1, (int)(S * K), S, db, de, st));
            void* tmp = nullptr;
            LVG_TRY(cudaMallocAsync(&tmp, std::max<size_t>(tb, 1), st));
            LVG_TRY(cub::DeviceSegmentedSort::SortKeys(tmp, tb, k0, k1, (int)(S * K), S, db, de, st));
            LVG_TRY(cudaFreeAsync(tmp, st));
            const unsigned long long none = ~0ull;
            LVG_TRY(cudaMemcpyAsync(cnt + 1, &none, sizeof(none), cudaMemcpyHostToDevice, st));
            ta_upper_kernel<<<(unsigned)((K + 255) / 256), 256, 0, st>>>(k1, bnd, K, S, tau, U, cnt + 1);
            unsigned long long dstar = 0;
            LVG_TRY(cudaMemcpyAsync(&dstar, cnt + 1, sizeof(dstar), cudaMemcpyDeviceToHost, st));
            LVG_TRY(cudaStreamSynchronize(st));
            const long long depth = dstar == none ? K : (long long)dstar;
            if (dstar != none) {
                res.ta_stop_depth = (int)dstar;
                LVG_TRY(cudaMemcpyAsync(&res.ta_stop_upper, U + dstar - 1, sizeof(double), cudaMemcpyDeviceToHost, st));
            }
            ta_mark_kernel<<<dim3((unsigned)((depth + 255) / 256), S), 256, 0, st>>>(dv, slot, K, k1, depth, live_bits);
            LVG_TRY(cudaGetLastError());
            LVG_TRY(cudaFreeAsync(k0, st));
            LVG_TRY(cudaFreeAsync(k1, st));
            LVG_TRY(cudaFreeAsync(U, st));
            LVG_TRY(cudaFreeAsync(db, st));
        }
        popc_kernel<<<64, 256, 0, st>>>(live_bits, words, cnt);
        unsigned long long kc = 0;
        LVG_TRY(cudaMemcpyAsync(&kc, cnt, sizeof(kc), cudaMemcpyDeviceToHost, st));
        LVG_TRY(cudaFreeAsync(qd, st));
        LVG_TRY(cudaFreeAsync(bnd, st));
        LVG_TRY(cudaFreeAsync(cnt, st));
        LVG_TRY(cudaStreamSynchronize(st));
        res.keys_scanned = (long long)kc;
    }
    // finalize_stats (query.cpp:70-78)
    res.f_scan = n ? (double)res.keys_scanned / (double)n : 0.0;
    const int gate = gi.enclosure == 1 ? 2 : 1;
    res.gate_cost_equiv = (double)gate * (double)res.groups_tested / gi.r;
    *stats = res;
    return cudaSuccess;
}

cudaError_t thresholds(const GroupIndex& gi, int slot, const float* q, float tau, float* out, cudaStream_t st) {
    const int S = gi.S;
    const long long K = gi.K;
    std::vector<double> peak(S, 0.0);
    std::vector<unsigned long long> nbb(S, 0);
    if (K > 0) {
        const Dev dv = view(gi);
        float *qd = nullptr, *bnd = nullptr;
        double* pk = nullptr;
        LVG_TRY(cudaMallocAsync(&qd, sizeof(float) * gi.d, st));
        LVG_TRY(cudaMallocAsync(&bnd, sizeof(float) * S * K, st));
        LVG_TRY(cudaMallocAsync(&pk, sizeof(double) * S, st));
        LVG_TRY(cudaMemcpyAsync(qd, q, sizeof(float) * gi.d, cudaMemcpyHostToDevice, st));
        bounds_kernel<<<dim3((unsigned)((K + 255) / 256), S), 256, 0, st>>>(dv, slot, K, qd, bnd);
        peaks_kernel<<<S, 256, 0, st>>>(bnd, K, pk);
        LVG_TRY(cudaGetLastError());
        LVG_TRY(cudaMemcpyAsync(peak.data(), pk, sizeof(double) * S, cudaMemcpyDeviceToHost, st));
        LVG_TRY(cudaMemcpyAsync(nbb.data(), gi.nbound + (size_t)slot * S, sizeof(unsigned long long) * S,
                                cudaMemcpyDeviceToHost, st));
        LVG_TRY(cudaFreeAsync(qd, st));
        LVG_TRY(cudaFreeAsync(bnd, st));
        LVG_TRY(cudaFreeAsync(pk, st));
        LVG_TRY(cudaStreamSynchronize(st));
    }
    // query.cpp:313-335: slack and tau_s, in double; q.norm() is a float norm
    double nbsq = 0.0;
    for (int s = 0; s < S; ++s) {
        double v;
        std::memcpy(&v, &nbb[s], sizeof(v));
        nbsq += v * v;
    }
    float qq = 0.0f;
    for (int i = 0; i < gi.d; ++i) qq += q[i] * q[i];
    const double eps = 1.1920928955078125e-07;
    const double slack = S == 1 ? 0.0 : 4.0 * gi.d * eps * double(std::sqrt(qq)) * std::sqrt(nbsq);
    double total = 0.0;
    for (int s = 0; s < S; ++s) total += peak[s];
    for (int s = 0; s < S; ++s) out[s] = static_cast<float>(double(tau) - (total - peak[s]) - slack);
    return cudaSuccess;
}

cudaError_t export_subspace(const GroupIndex& gi, int slot, int s, unsigned* assign, unsigned* moff, unsigned* mids,
                            float* a, float* b, float* radii, double* norm_bound) {
    const size_t p = (size_t)slot * gi.S + s;
    const long long n = gi.indexed, K = gi.K;
    const int w = gi.off[s + 1] - gi.off[s];
    if (assign && n) LVG_TRY(cudaMemcpy(assign, gi.assign + p * gi.cap, sizeof(unsigned) * n, cudaMemcpyDeviceToHost));
    if (mids && n) LVG_TRY(cudaMemcpy(mids, gi.mids + p * gi.cap, sizeof(unsigned) * n, cudaMemcpyDeviceToHost));
    if (moff) {
        if (K) LVG_TRY(cudaMemcpy(moff, gi.moff + p * (gi.kcap + 1), sizeof(unsigned) * (K + 1), cudaMemcpyDeviceToHost));
        else moff[0] = 0;
    }
    if (a && K)
        LVG_TRY(cudaMemcpy2D(a, sizeof(float) * K, gi.ga + p * gi.wmax * gi.kcap, sizeof(float) * gi.kcap,
                             sizeof(float) * K, w, cudaMemcpyDeviceToHost));
    if (b && K && gi.gb)
        LVG_TRY(cudaMemcpy2D(b, sizeof(float) * K, gi.gb + p * gi.wmax * gi.kcap, sizeof(float) * gi.kcap,
                             sizeof(float) * K, w, cudaMemcpyDeviceToHost));
    if (radii && K && gi.grad)
        LVG_TRY(cudaMemcpy(radii, gi.grad + p * gi.kcap, sizeof(float) * K, cudaMemcpyDeviceToHost));
    if (norm_bound) {
        unsigned long long nb = 0;
        LVG_TRY(cudaMemcpy(&nb, gi.nbound + p, sizeof(nb), cudaMemcpyDeviceToHost));
        std::memcpy(norm_bound, &nb, sizeof(double));
    }
    return cudaSuccess;
}

cudaError_t import_subspace(GroupIndex& gi, int slot, int s, long long indexed, long long K, const unsigned* assign,
                            const unsigned* moff, const unsigned* mids, const float* a, const float* b,
                            const float* radii, double norm_bound) {
    if (indexed > gi.cap || K > gi.kcap) return cudaErrorInvalidValue;
    const size_t p = (size_t)slot * gi.S + s;
    const int w = gi.off[s + 1] - gi.off[s];
    if (indexed) {
        LVG_TRY(cudaMemcpy(gi.assign + p * gi.cap, assign, sizeof(unsigned) * indexed, cudaMemcpyHostToDevice));
        LVG_TRY(cudaMemcpy(gi.mids + p * gi.cap, mids, sizeof(unsigned) * indexed, cudaMemcpyHostToDevice));
    }
    LVG_TRY(cudaMemcpy(gi.moff + p * (gi.kcap + 1), moff, sizeof(unsigned) * (K + 1), cudaMemcpyHostToDevice));
    if (K) {
        LVG_TRY(cudaMemcpy2D(gi.ga + p * gi.wmax * gi.kcap, sizeof(float) * gi.kcap, a, sizeof(float) * K,
                             sizeof(float) * K, w, cudaMemcpyHostToDevice));
        if (gi.gb && b)
            LVG_TRY(cudaMemcpy2D(gi.gb + p * gi.wmax * gi.kcap, sizeof(float) * gi.kcap, b, sizeof(float) * K,
                                 sizeof(float) * K, w, cudaMemcpyHostToDevice));
        if (gi.grad && radii)
            LVG_TRY(cudaMemcpy(gi.grad + p * gi.kcap, radii, sizeof(float) * K, cudaMemcpyHostToDevice));
    }
    unsigned long long nb;
    std::memcpy(&nb, &norm_bound, sizeof(nb));
    LVG_TRY(cudaMemcpy(gi.nbound + p, &nb, sizeof(nb), cudaMemcpyHostToDevice));
    gi.indexed = indexed;
    gi.K = K;
    return cudaSuccess;
}

}  // namespace lvg
