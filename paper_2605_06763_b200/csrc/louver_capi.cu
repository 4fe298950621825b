// C ABI of the B200 Louver hot path (include/louver_b200.h): context/arena
// management, host<->device staging, and kernel launches. No CPU compute path:
// every score, bound, selection and softmax runs in the kernels of
// louver_kernels.cuh / louver_aux.cuh.

#include <algorithm>
#include <atomic>
#include <cmath>
#include <cstdlib>
#include <cstring>
#include <fstream>
#include <mutex>
#include <random>
#include <string>
#include <vector>

#include <cudaTypedefs.h>  // PFN_cuTensorMapEncodeTiled

#include "louver_aux.cuh"
#include "louver_b200.h"
#include "louver_threshold.cuh"
#include "louver_dispatch.h"
#include "louver_f32.cuh"
#include "louver_groups.h"
#include "louver_launch.h"
#include "louver_v9.cuh"

using lvk::Counters;

namespace {

thread_local std::string g_err;

int fail(int code, const std::string& msg) {
    g_err = msg;
    return code;
}

#define LV_CUDA(call)                                                                        \
    do {                                                                                     \
        cudaError_t e_ = (call);                                                             \
        if (e_ != cudaSuccess)                                                               \
            return fail(LV_ERUNTIME, std::string(#call) + ": " + cudaGetErrorString(e_));    \
    } while (0)

int pad_dim(int d) { return d <= 64 ? 64 : (d <= 128 ? 128 : 256); }
int esize(int dtype) { return dtype == LV_BF16 ? 2 : 4; }
int ilog2(int x) {
    int l = 0;
    while ((1 << l) < x) ++l;
    return l;
}

constexpr long long kCapAlign = 1024;  // arena rows per slot: a whole number of v2 units

struct Workspace {
    float* partial = nullptr;  // [slots][max(splits, nb)][G][DP+2]
    int* tickets = nullptr;    // [slots] (fp32 kernel)
    int* stickets = nullptr;   // [slots] (bf16 layer kernel)
    float* q = nullptr;        // [rows][DP]
    float* out = nullptr;      // [rows][DP]
    float* tau = nullptr;      // [rows]
    float* part_out = nullptr; // [rows][DP+2]
    int* counts = nullptr;     // [rows][4]
    unsigned short* glist = nullptr;  // [slots][cap_cells + nb] survivor lists (fused kernel, large contexts)
};

}  // namespace

struct lv_ctx {
    lv_config cfg{};
    int DP = 0, G = 1, r = 1, r_log2 = 0, slots = 0, rows = 0;
    long long cap = 0, cap_cells = 0, bits_words = 0;
    int splits = 1, chunks_per_split = 1;  // fp32 kernel (query, dense, brute force) geometry
    int sms = 148;
    int layer_geo[4] = {0, 0, 0, 0};  // fused bf16 layer kernel: team CTAs/slot, threads, smem, CTAs/SM
    int nb = 1;                        // bf16 layer kernel: team CTAs per slot (upper bound)
    void* K = nullptr;
    void* V = nullptr;
    void* lo = nullptr;
    void* hi = nullptr;
    float* colmax = nullptr;
    Counters* ctr = nullptr;
    int* ins_ticket = nullptr;
    void* ws_mem = nullptr;
    size_t ws_bytes = 0;
    // host mirrors of the device counters
    long long n = 0, indexed = 0, flushes = 0;
    void* stage = nullptr;       // lv_query_layers' internal staging (lazily grown)
    size_t stage_bytes = 0;
    std::mutex stage_mu;
    long long version = 0;       // unique per context and per arena (lv_reserve): cached graphs expire
    // lv_query_layers' CUDA graph of one decode step (copy in, L queries, copy out), cached for
    // the last (contexts, host buffers, staging, stream) it was called with
    struct LayersGraph {
        std::vector<const lv_ctx*> ctxs;
        std::vector<long long> versions;
        const void *q = nullptr, *tau = nullptr, *out = nullptr, *base = nullptr;
        float scale = 0.0f;
        int strict = 0;
        cudaStream_t st = nullptr;
        cudaGraphExec_t exec = nullptr;
    } lgraph;
    int npre = 3;                // experiment knob (LV_PRE)
    long long* trace = nullptr;  // debug: per-CTA phase timestamps of the bf16 query kernel
    lvg::GroupIndex* gi = nullptr;  // the reference's grouped index (cfg.group_index)
    int kpf = 8;                    // listed cells whose key blocks the probe L2-prefetches (LV_KPF)
    int vtail = 16;                 // last tasks whose value blocks are L2-prefetched (LV_VTAIL)
    int spread = 1;                 // late-dispatched CTAs spread over the slots (LV_SPREAD)
    int uneven = 1;                 // teams of nb and nb - 1 CTAs to fill every SM (LV_UNEVEN)
    int ktma = 0;                   // key blocks by TMA in the bf16 layer kernel (LV_KTMA=1; A/B: slower)
    int f32_layer = 1;               // fp32 queries on the fused fp32 layer kernel (LV_F32_LAYER=0: round-1 kernel)
    CUtensorMap kmap{};             // its tensor map, for kmap_K / kmap_cap
    const void* kmap_K = nullptr;
    long long kmap_cap = 0;
    std::mutex writer;
};

namespace {

size_t align256(size_t x) { return (x + 255) & ~size_t(255); }

// Carve a workspace into its parts; returns the total size.
size_t carve(const lv_ctx* c, unsigned char* base, Workspace* w) {
    size_t off = 0;
    auto take = [&](size_t bytes) {
        unsigned char* p = base ? base + off : nullptr;
        off = align256(off + bytes);
        return p;
    };
    const size_t rows = (size_t)c->rows;
    unsigned char* t = take(sizeof(int) * c->slots);
    const size_t nparts = (size_t)std::max(c->splits, c->nb);
    // partials: [slots][parts][G][DP+2] (+ the bf16 layer kernel's per-CTA counts [G][4])
    unsigned char* part = take(sizeof(float) * c->slots * nparts * c->G * (c->DP + 6));
    unsigned char* q = take(sizeof(float) * rows * c->DP);
    unsigned char* o = take(sizeof(float) * rows * c->DP);
    unsigned char* tau = take(sizeof(float) * rows);
    unsigned char* po = take(sizeof(float) * rows * (c->DP + 2));
    unsigned char* cnt = take(sizeof(int) * rows * 4);
    unsigned char* stk = take(sizeof(int) * c->slots);
    unsigned char* gl = take(sizeof(unsigned short) * c->slots * ((size_t)c->cap_cells + c->nb));
    if (w) {
        w->glist = reinterpret_cast<unsigned short*>(gl);
        w->stickets = reinterpret_cast<int*>(stk);
        w->tickets = reinterpret_cast<int*>(t);
        w->partial = reinterpret_cast<float*>(part);
        w->q = reinterpret_cast<float*>(q);
        w->out = reinterpret_cast<float*>(o);
        w->tau = reinterpret_cast<float*>(tau);
        w->part_out = reinterpret_cast<float*>(po);
        w->counts = reinterpret_cast<int*>(cnt);
    }
    return off;
}

int validate(const lv_config* c) {
    if (!c) return fail(LV_EINVAL, "lv_create: null config");
    if (c->d < 1 || c->d > 256) return fail(LV_EINVAL, "KeyStore: 1 <= d <= 256 required");
    if (c->n_kv_heads < 1 || c->batch < 1) return fail(LV_EINVAL, "lv_create: heads/batch >= 1");
    if (c->group_size != 1 && c->group_size != 2 && c->group_size != 4 && c->group_size != 8)
        return fail(LV_EINVAL, "lv_create: group_size must be 1, 2, 4 or 8");
    if (c->dtype != LV_F32 && c->dtype != LV_BF16) return fail(LV_EINVAL, "lv_create: dtype");
    // BuildConfig::validate (index.hpp:17-21)
    if (c->S < 1) return fail(LV_EINVAL, "BuildConfig: S >= 1 required");
    if (c->r < 1) return fail(LV_EINVAL, "BuildConfig: r >= 1 required");
    if (c->S > c->d) return fail(LV_EINVAL, "BuildConfig: S <= d required");
    if (c->group_index != 0 && c->group_index != 1) return fail(LV_EINVAL, "lv_create: group_index must be 0 or 1");
    if (c->group_index && c->S > 64) return fail(LV_EINVAL, "lv_create: the grouped index supports S <= 64");
    if (c->grouping < 0 || c->grouping > 3 || c->enclosure < 0 || c->enclosure > 2)
        return fail(LV_EINVAL, "BuildConfig: unknown grouping or enclosure");
    if (c->buffer_capacity < 1)
        return fail(LV_EINVAL, "LouverCache: buffer capacity >= 1 required");
    if (c->capacity < 1) return fail(LV_EINVAL, "lv_create: capacity >= 1 required");
    return LV_OK;
}

cudaStream_t S(void* s) { return reinterpret_cast<cudaStream_t>(s); }

void choose_splits(lv_ctx* c) {
    c->sms = lvl::device_sms();
    {
        // fused layer kernels (bf16 and fp32): up to one CTA per SM per slot; the launch
        // clamps the team to the resident wave (inst_v9.cu, inst_f32.cu)
        // ... and no more CTAs than 64-cell shares of the arena: a small slot (C1: 2048
        // cells) spread over every SM leaves each CTA a handful of cells and a long merge
        // (C1 fp32: 148 CTAs 17.5 us, 32 CTAs 13.1 us)
        long long nb = std::max(1LL, ((long long)c->sms + c->slots - 1) / c->slots);
        nb = std::max(1LL, std::min(nb, (c->cap_cells + 63) / 64));
        if (const char* e = std::getenv("LV_NB")) nb = std::max(1LL, std::atoll(e));
        if (const char* e = std::getenv("LV_PRE")) c->npre = std::min(3, std::max(0, std::atoi(e)));
        if (const char* e = std::getenv("LV_KTMA")) c->ktma = std::atoi(e);
        if (const char* e = std::getenv("LV_KPF")) c->kpf = std::max(0, std::atoi(e));
        if (const char* e = std::getenv("LV_UNEVEN")) c->uneven = std::atoi(e);
        if (const char* e = std::getenv("LV_VTAIL")) c->vtail = std::max(0, std::atoi(e));
        if (const char* e = std::getenv("LV_SPREAD")) c->spread = std::atoi(e);
        if (const char* e = std::getenv("LV_F32_LAYER")) c->f32_layer = std::atoi(e);
        c->nb = (int)std::min<long long>(nb, 4096);
    }
    // fp32 kernel (fp32 query and dense, brute force for both dtypes): chunks of kChunk keys
    const long long chunks = c->cap / lvk::kChunk;
    long long cps = 1;
    if (const char* e = std::getenv("LV_CHUNKS_PER_SPLIT")) {
        cps = std::max(1LL, std::atoll(e));
    } else {
        const long long target = (long long)c->sms * 6;  // ~2 waves at 3 CTAs/SM
        cps = std::max(1LL, (chunks * c->slots + target - 1) / target);
    }
    long long splits = (chunks + cps - 1) / cps;
    while (splits > 1024) {
        ++cps;
        splits = (chunks + cps - 1) / cps;
    }
    c->chunks_per_split = (int)cps;
    c->splits = (int)splits;
}

// Copy a [rows][d] fp32 array (host or device) into a [rows][DP] device array.
int stage_rows(lv_ctx* c, float* dst, const float* src, int where, cudaStream_t st) {
    const size_t d = c->cfg.d;
    if (d != (size_t)c->DP) LV_CUDA(cudaMemsetAsync(dst, 0, sizeof(float) * c->rows * c->DP, st));
    LV_CUDA(cudaMemcpy2DAsync(dst, sizeof(float) * c->DP, src, sizeof(float) * d, sizeof(float) * d,
                              c->rows, where == LV_HOST ? cudaMemcpyHostToDevice : cudaMemcpyDeviceToDevice,
                              st));
    return LV_OK;
}

template <typename T>
int launch_summaries_t(lv_ctx* c, long long cell_begin, long long cell_end, long long n,
                       cudaStream_t st) {
    const int CB = c->DP > 128 ? 16 : 32;
    const long long ncell = cell_end - cell_begin;
    if (ncell <= 0) return LV_OK;
    dim3 grid((unsigned)((ncell + CB - 1) / CB), (unsigned)c->slots);
    T* K = reinterpret_cast<T*>(c->K);
    T* lo = reinterpret_cast<T*>(c->lo);
    T* hi = reinterpret_cast<T*>(c->hi);
    switch (c->DP) {
        case 64:
            lvk::summarize_kernel<T, 64><<<grid, 256, 0, st>>>(K, lo, hi, c->colmax, c->cap, c->cap_cells,
                                                              c->r_log2, n, cell_begin, cell_end);
            break;
        case 128:
            lvk::summarize_kernel<T, 128><<<grid, 256, 0, st>>>(K, lo, hi, c->colmax, c->cap, c->cap_cells,
                                                               c->r_log2, n, cell_begin, cell_end);
            break;
        default:
            lvk::summarize_kernel<T, 256><<<grid, 256, 0, st>>>(K, lo, hi, c->colmax, c->cap, c->cap_cells,
                                                               c->r_log2, n, cell_begin, cell_end);
    }
    LV_CUDA(cudaGetLastError());
    return LV_OK;
}

int launch_summaries(lv_ctx* c, long long cell_begin, long long cell_end, long long n,
                     cudaStream_t st) {
    return c->cfg.dtype == LV_BF16
               ? launch_summaries_t<__nv_bfloat16>(c, cell_begin, cell_end, n, st)
               : launch_summaries_t<float>(c, cell_begin, cell_end, n, st);
}

template <typename S_, typename T>
int launch_convert(lv_ctx* c, const void* src, void* dst, long long n, long long first,
                   cudaStream_t st) {
    const long long total = (long long)c->slots * n * c->DP;
    const int blocks = (int)std::min<long long>((total + 255) / 256, 148LL * 16);
    lvk::convert_rows_kernel<S_, T><<<blocks, 256, 0, st>>>(
        reinterpret_cast<const S_*>(src), reinterpret_cast<T*>(dst), c->slots, n, c->cfg.d, c->DP,
        c->cap, first);
    LV_CUDA(cudaGetLastError());
    return LV_OK;
}

int convert_into(lv_ctx* c, const void* src_dev, int src_dtype, void* arena, long long n,
                 long long first, cudaStream_t st) {
    const bool bf = c->cfg.dtype == LV_BF16;
    if (src_dtype == LV_F32)
        return bf ? launch_convert<float, __nv_bfloat16>(c, src_dev, arena, n, first, st)
                  : launch_convert<float, float>(c, src_dev, arena, n, first, st);
    if (!bf) return fail(LV_EINVAL, "bf16 source needs a bf16 cache");
    return launch_convert<__nv_bfloat16, __nv_bfloat16>(c, src_dev, arena, n, first, st);
}

long long next_version() {  // process-wide: a context reusing a freed one's address never matches
    static std::atomic<long long> v{0};
    return ++v;
}

lvg::ArenaView arena_view(const lv_ctx* c) {
    lvg::ArenaView a;
    a.K = c->K;
    a.bf16 = c->cfg.dtype == LV_BF16;
    a.DP = c->DP;
    a.cap = c->cap;
    return a;
}

// The K arena [slots * cap][DP] bf16 as a 2D tensor map: box 64 x 16 (one 128-byte column
// half of a 16-key block), 128-byte swizzle — the layer kernel's stage layout.
int ensure_kmap(lv_ctx* c) {
    if (c->kmap_K == c->K && c->kmap_cap == c->cap) return LV_OK;
    static PFN_cuTensorMapEncodeTiled_v12000 encode = nullptr;
    static std::once_flag once;
    std::call_once(once, [] {
        cudaDriverEntryPointQueryResult q;
        void* fn = nullptr;
        if (cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &fn, cudaEnableDefault, &q) == cudaSuccess &&
            q == cudaDriverEntryPointSuccess)
            encode = reinterpret_cast<PFN_cuTensorMapEncodeTiled_v12000>(fn);
    });
    if (!encode) return fail(LV_ERUNTIME, "cuTensorMapEncodeTiled unavailable");
    const cuuint64_t dims[2] = {(cuuint64_t)c->DP, (cuuint64_t)c->slots * (cuuint64_t)c->cap};
    const cuuint64_t strides[1] = {(cuuint64_t)c->DP * 2};
    const cuuint32_t box[2] = {64, 16};
    const cuuint32_t estr[2] = {1, 1};
    const CUresult r = encode(&c->kmap, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 2, c->K, dims, strides, box, estr,
                              CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B,
                              CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
    if (r != CUDA_SUCCESS) return fail(LV_ERUNTIME, "cuTensorMapEncodeTiled failed: " + std::to_string((int)r));
    c->kmap_K = c->K;
    c->kmap_cap = c->cap;
    return LV_OK;
}

int sync_if_host(int where, cudaStream_t st) {
    if (where == LV_HOST) LV_CUDA(cudaStreamSynchronize(st));
    return LV_OK;
}

int run_query_kernel(lv_ctx* c, int mode, const float* qdev, const float* taudev, long long limit,
                     float scale, int strict, Workspace& w, float* out, float* part_out,
                     unsigned* bits, int* counts, unsigned long long* totals, cudaStream_t st,
                     unsigned* cand_bits = nullptr) {
    lvk::QueryParams p{};
    p.K = c->K;
    p.V = c->V;
    p.lo = c->lo;
    p.hi = c->hi;
    p.colmax = c->colmax;
    p.q = qdev;
    p.tau = taudev;
    p.ctr = c->ctr;
    p.cap = c->cap;
    p.cap_cells = c->cap_cells;
    p.limit = limit;
    p.r_log2 = c->r_log2;
    p.chunks_per_split = c->chunks_per_split;
    p.splits = c->splits;
    p.strict = strict;
    p.d_true = c->cfg.d;
    p.scale = scale != 0.0f ? scale : (float)(1.0 / std::sqrt((double)c->cfg.d));
    p.partial_ws = w.partial;
    p.tickets = w.tickets;
    p.out = out;
    p.partial_out = part_out;
    p.bits = bits;
    p.bits_words = c->bits_words;
    p.counts = counts;
    p.totals = totals;
    p.cand_bits = cand_bits;
    dim3 grid((unsigned)c->splits, (unsigned)c->slots);
    cudaError_t e;
    if (c->cfg.dtype == LV_BF16 && mode != lvk::kBrute) {
        lvk9::LayerParams lp{};
        lp.p = p;
        lp.sum = reinterpret_cast<const __nv_bfloat16*>(c->lo);
        lp.stickets = w.stickets;
        lp.nb = c->nb;
        lp.glist = w.glist;
        lp.p.tot_trace = c->trace;
        lp.npre = c->npre;
        lp.kpf = c->kpf;
        lp.nfull = c->uneven;
        lp.vtail = c->vtail;
        lp.spread = c->spread;
        lp.ktma = c->ktma && c->kmap_K == c->K;  // the map is encoded by lv_create / lv_reserve
        if (lp.ktma) lp.kmap = c->kmap;
        // cells complete before the last insert enqueued ahead of this query: the insert kernel
        // that may still be draining under PDL writes only the cell of key n - 1
        lp.sealed = c->n > 0 ? (c->n - 1) >> c->r_log2 : 0;
        e = lvk9::launch_layer_v9(c->DP, c->G, mode == lvk::kDense, lp, c->slots, c->sms, st, c->layer_geo);
    } else if (mode == lvk::kQuery && c->f32_layer && (c->DP == 128 || c->DP == 256)) {
        // fp32 caches: the fused fp32 layer kernel (normative dots on the CUDA cores)
        lvkf::F32Params fp{};
        fp.p = p;
        fp.sum = reinterpret_cast<const float*>(c->lo);
        fp.stickets = w.stickets;
        fp.nb = c->nb;
        fp.glist = w.glist;
        fp.sealed = c->n > 0 ? (c->n - 1) >> c->r_log2 : 0;
        e = lvkf::launch_layer_f32(c->DP, c->G, fp, c->slots, c->sms, st, c->layer_geo);
    } else {
        e = lvk::launch_query(c->cfg.dtype, c->DP, c->G, mode, p, grid, st);
    }
    if (e != cudaSuccess) return fail(LV_ERUNTIME, std::string("query kernel: ") + cudaGetErrorString(e));
    return LV_OK;
}

}  // namespace

namespace lvk {

int query_smem_bytes(int dtype, int DP, int G) {
#define LVK_SM(T)                                                   \
    switch (DP * 16 + G) {                                          \
        case 64 * 16 + 1: return Geo<T, 64, 1>::SMEM;               \
        case 64 * 16 + 2: return Geo<T, 64, 2>::SMEM;               \
        case 64 * 16 + 4: return Geo<T, 64, 4>::SMEM;               \
        case 64 * 16 + 8: return Geo<T, 64, 8>::SMEM;               \
        case 128 * 16 + 1: return Geo<T, 128, 1>::SMEM;             \
        case 128 * 16 + 2: return Geo<T, 128, 2>::SMEM;             \
        case 128 * 16 + 4: return Geo<T, 128, 4>::SMEM;             \
        case 128 * 16 + 8: return Geo<T, 128, 8>::SMEM;             \
        case 256 * 16 + 1: return Geo<T, 256, 1>::SMEM;             \
        case 256 * 16 + 2: return Geo<T, 256, 2>::SMEM;             \
        case 256 * 16 + 4: return Geo<T, 256, 4>::SMEM;             \
        case 256 * 16 + 8: return Geo<T, 256, 8>::SMEM;             \
    }
    if (dtype == LV_BF16) {
        LVK_SM(__nv_bfloat16)
    } else {
        LVK_SM(float)
    }
#undef LVK_SM
    return -1;
}

cudaError_t launch_query(int dtype, int DP, int G, int mode, const QueryParams& p, dim3 grid,
                         cudaStream_t st) {
#define LVK_G(T, D, M)                                               \
    switch (G) {                                                     \
        case 1: return launch_query_t<T, D, 1, M>(p, grid, st);      \
        case 2: return launch_query_t<T, D, 2, M>(p, grid, st);      \
        case 4: return launch_query_t<T, D, 4, M>(p, grid, st);      \
        case 8: return launch_query_t<T, D, 8, M>(p, grid, st);      \
    }                                                                \
    break;
#define LVK_D(T, M)                    \
    switch (DP) {                      \
        case 64: LVK_G(T, 64, M)       \
        case 128: LVK_G(T, 128, M)     \
        case 256: LVK_G(T, 256, M)     \
    }                                  \
    break;
#define LVK_M(T)                       \
    switch (mode) {                    \
        case kQuery: LVK_D(T, kQuery)  \
        case kBrute: LVK_D(T, kBrute)  \
        case kDense: LVK_D(T, kDense)  \
    }
    if (dtype == LV_BF16) {  // bf16 queries and dense scans run the layer kernel (inst_v9.cu)
        switch (mode) {
            case kBrute: LVK_D(__nv_bfloat16, kBrute)
        }
    } else {
        LVK_M(float)
    }
#undef LVK_G
#undef LVK_D
#undef LVK_M
    return cudaErrorInvalidValue;
}

}  // namespace lvk

namespace {
const char kLVKD[4] = {'L', 'V', 'K', 'D'};
const char kLVIX[4] = {'L', 'V', 'I', 'X'};

template <typename T>
void put_le(std::ostream& os, T v) {  // little-endian host, as io.cpp:18-24
    os.write(reinterpret_cast<const char*>(&v), sizeof(T));
}

template <typename T>
bool get_le(std::istream& is, T* v) {
    is.read(reinterpret_cast<char*>(v), sizeof(T));
    return (bool)is;
}

bool at_eof(std::istream& is) {
    is.peek();
    return is.eof();
}
}  // namespace

extern "C" {

const char* lv_last_error(void) { return g_err.c_str(); }

const char* lv_build_info(void) { return "louver_b200 0.1 sm_100a"; }

int lv_create(const lv_config* cfg, lv_ctx** out) {
    if (!out) return fail(LV_EINVAL, "lv_create: null out");
    *out = nullptr;
    if (int rc = validate(cfg)) return rc;
    int ndev = 0;
    if (cudaGetDeviceCount(&ndev) != cudaSuccess || ndev == 0)
        return fail(LV_ENODEV, "lv_create: no CUDA device (the Louver hot path has no CPU fallback)");
    auto* c = new lv_ctx();
    c->cfg = *cfg;
    c->DP = pad_dim(cfg->d);
    c->G = cfg->group_size;
    // device cells: contiguous, r rounded up to a power of two in [16, 64]
    c->r = std::max(16, 1 << ilog2(std::min(cfg->r, 64)));
    c->r_log2 = ilog2(c->r);
    c->slots = cfg->batch * cfg->n_kv_heads;
    c->rows = c->slots * c->G;
    c->version = next_version();
    c->cap = (cfg->capacity + kCapAlign - 1) / kCapAlign * kCapAlign;
    c->cap_cells = c->cap / c->r;
    c->bits_words = c->cap / 32;
    choose_splits(c);
    const size_t es = esize(cfg->dtype);
    const size_t kv_bytes = (size_t)c->slots * c->cap * c->DP * es;
    // blocked summaries [slot][chunk][lo|hi][DP][cells per chunk]
    const size_t sum_bytes = 2 * (size_t)c->slots * c->DP * c->cap_cells * es;
    auto cleanup = [&](const char* what, cudaError_t e) {
        lv_destroy(c);
        return fail(LV_ERUNTIME, std::string(what) + ": " + cudaGetErrorString(e));
    };
    cudaError_t e;
    if ((e = cudaMalloc(&c->K, kv_bytes)) != cudaSuccess) return cleanup("alloc K", e);
    if ((e = cudaMalloc(&c->V, kv_bytes)) != cudaSuccess) return cleanup("alloc V", e);
    if ((e = cudaMalloc(&c->lo, sum_bytes)) != cudaSuccess) return cleanup("alloc summaries", e);
    c->hi = c->lo;  // lo and hi live in the same blocked tiles
    if ((e = cudaMalloc(&c->colmax, sizeof(float) * c->slots * c->DP)) != cudaSuccess)
        return cleanup("alloc colmax", e);
    if ((e = cudaMalloc(&c->ctr, sizeof(Counters))) != cudaSuccess) return cleanup("alloc ctr", e);
    if ((e = cudaMalloc(&c->ins_ticket, sizeof(int))) != cudaSuccess) return cleanup("alloc ticket", e);
    c->ws_bytes = carve(c, nullptr, nullptr);
    if ((e = cudaMalloc(&c->ws_mem, c->ws_bytes)) != cudaSuccess) return cleanup("alloc ws", e);
    cudaMemset(c->K, 0, kv_bytes);
    cudaMemset(c->V, 0, kv_bytes);
    cudaMemset(c->colmax, 0, sizeof(float) * c->slots * c->DP);
    cudaMemset(c->ctr, 0, sizeof(Counters));
    cudaMemset(c->ins_ticket, 0, sizeof(int));
    cudaMemset(c->ws_mem, 0, c->ws_bytes);
    if (cfg->group_index) {
        c->gi = new lvg::GroupIndex();
        if ((e = lvg::create(*c->gi, cfg->d, cfg->S, cfg->r, cfg->grouping, cfg->enclosure, cfg->rng_seed, c->slots,
                             c->cap)) != cudaSuccess)
            return cleanup("alloc grouped index", e);
    }
    if ((e = cudaDeviceSynchronize()) != cudaSuccess) return cleanup("init", e);
    if (cfg->dtype == LV_BF16 && c->ktma)
        if (int rc = ensure_kmap(c)) {
            lv_destroy(c);
            return rc;
        }
    *out = c;
    return LV_OK;
}

int lv_destroy(lv_ctx* c) {
    if (!c) return LV_OK;
    cudaFree(c->K);
    cudaFree(c->V);
    cudaFree(c->lo);
    cudaFree(c->colmax);
    cudaFree(c->ctr);
    cudaFree(c->ins_ticket);
    cudaFree(c->ws_mem);
    if (c->stage) cudaFree(c->stage);
    if (c->lgraph.exec) cudaGraphExecDestroy(c->lgraph.exec);
    if (c->gi) {
        lvg::destroy(*c->gi);
        delete c->gi;
    }
    delete c;
    return LV_OK;
}

size_t lv_query_workspace_bytes(const lv_ctx* c) { return c ? c->ws_bytes : 0; }

int lv_debug_trace(lv_ctx* c, int64_t* dev_buf) {
    if (!c) return fail(LV_EINVAL, "lv_debug_trace: null context");
    c->trace = reinterpret_cast<long long*>(dev_buf);
    return LV_OK;
}

int lv_geometry(const lv_ctx* c, int64_t* out) {
    if (!c || !out) return fail(LV_EINVAL, "lv_geometry: null argument");
    out[0] = c->DP;
    out[1] = c->r;
    out[2] = c->cap;
    out[3] = c->cap_cells;
    out[4] = c->splits;
    out[5] = c->chunks_per_split;
    out[6] = lvk::kChunk;
    out[7] = c->cfg.dtype == LV_BF16 ? c->layer_geo[2] : lvk::query_smem_bytes(c->cfg.dtype, c->DP, c->G);
    return LV_OK;
}
int lv_layer_geometry(const lv_ctx* c, int64_t* out) {
    if (!c || !out) return fail(LV_EINVAL, "lv_layer_geometry: null argument");
    out[0] = c->layer_geo[0];  // CTAs per slot (team)
    out[1] = c->layer_geo[3];  // resident CTAs per SM
    out[2] = c->layer_geo[1];  // threads per CTA
    out[3] = c->layer_geo[2];  // dynamic shared memory bytes
    return LV_OK;
}
int64_t lv_bitmap_words(const lv_ctx* c) { return c ? c->bits_words : 0; }
int64_t lv_n(const lv_ctx* c) { return c->n; }
int64_t lv_indexed_count(const lv_ctx* c) { return c->indexed; }
int64_t lv_pending_count(const lv_ctx* c) { return c->n - c->indexed; }
int64_t lv_flush_count(const lv_ctx* c) { return c->flushes; }

int lv_reserve(lv_ctx* c, int64_t capacity, void* stream) {
    if (!c) return fail(LV_EINVAL, "lv_reserve: null context");
    std::lock_guard<std::mutex> lock(c->writer);
    if (capacity <= c->cfg.capacity) return LV_OK;
    cudaStream_t st = S(stream);
    LV_CUDA(cudaStreamSynchronize(st));
    const long long ncap = (capacity + kCapAlign - 1) / kCapAlign * kCapAlign;
    const long long ncells = ncap / c->r;
    const size_t es = esize(c->cfg.dtype);
    const size_t kv_bytes = (size_t)c->slots * ncap * c->DP * es;
    const size_t sum_bytes = 2 * (size_t)c->slots * c->DP * ncells * es;
    void *K = nullptr, *V = nullptr, *lo = nullptr, *ws = nullptr;
    auto undo = [&](cudaError_t e) {
        cudaFree(K);
        cudaFree(V);
        cudaFree(lo);
        cudaFree(ws);
        return fail(LV_ERUNTIME, std::string("lv_reserve: ") + cudaGetErrorString(e));
    };
    cudaError_t e;
    if ((e = cudaMalloc(&K, kv_bytes)) != cudaSuccess) return undo(e);
    if ((e = cudaMalloc(&V, kv_bytes)) != cudaSuccess) return undo(e);
    if ((e = cudaMalloc(&lo, sum_bytes)) != cudaSuccess) return undo(e);
    cudaMemset(K, 0, kv_bytes);
    cudaMemset(V, 0, kv_bytes);
    // rows keep their ids: [slot][cap][DP] -> [slot][ncap][DP]; the blocked
    // summary tiles of a slot are contiguous, so they move the same way
    const size_t rowb = (size_t)c->cap * c->DP * es;
    if ((e = cudaMemcpy2D(K, (size_t)ncap * c->DP * es, c->K, rowb, rowb, c->slots,
                          cudaMemcpyDeviceToDevice)) != cudaSuccess) return undo(e);
    if ((e = cudaMemcpy2D(V, (size_t)ncap * c->DP * es, c->V, rowb, rowb, c->slots,
                          cudaMemcpyDeviceToDevice)) != cudaSuccess) return undo(e);
    const size_t tileb = 2 * (size_t)c->DP * c->cap_cells * es;
    if ((e = cudaMemcpy2D(lo, 2 * (size_t)c->DP * ncells * es, c->lo, tileb, tileb, c->slots,
                          cudaMemcpyDeviceToDevice)) != cudaSuccess) return undo(e);
    void* hi = lo;
    lv_ctx probe_geo;  // geometry for the new capacity's workspace
    probe_geo.cfg = c->cfg;
    probe_geo.DP = c->DP;
    probe_geo.G = c->G;
    probe_geo.slots = c->slots;
    probe_geo.rows = c->rows;
    probe_geo.cap = ncap;
    probe_geo.r = c->r;
    probe_geo.r_log2 = c->r_log2;
    probe_geo.cap_cells = ncells;  // sizes the survivor-list scratch
    choose_splits(&probe_geo);
    const size_t wsb = carve(&probe_geo, nullptr, nullptr);
    if ((e = cudaMalloc(&ws, wsb)) != cudaSuccess) return undo(e);
    cudaMemset(ws, 0, wsb);
    if (c->gi && (e = lvg::reserve(*c->gi, ncap, st)) != cudaSuccess) return undo(e);
    if ((e = cudaDeviceSynchronize()) != cudaSuccess) return undo(e);
    cudaFree(c->K);
    cudaFree(c->V);
    cudaFree(c->lo);
    cudaFree(c->ws_mem);
    c->K = K;
    c->V = V;
    c->lo = lo;
    c->hi = hi;
    c->ws_mem = ws;
    c->ws_bytes = wsb;
    c->cap = ncap;
    c->cap_cells = ncells;
    c->bits_words = ncap / 32;
    c->splits = probe_geo.splits;
    c->chunks_per_split = probe_geo.chunks_per_split;
    c->nb = probe_geo.nb;
    c->cfg.capacity = capacity;
    c->version = next_version();
    if (c->cfg.dtype == LV_BF16 && c->ktma) return ensure_kmap(c);
    return LV_OK;
}

int lv_build(lv_ctx* c, const void* K, const void* V, int64_t n, int src_dtype, int where,
             void* stream) {
    if (!c) return fail(LV_EINVAL, "lv_build: null context");
    std::lock_guard<std::mutex> lock(c->writer);
    if (n < 0 || n > c->cfg.capacity) return fail(LV_ERANGE, "lv_build: n exceeds capacity");
    if (n > 0 && (!K || !V)) return fail(LV_EINVAL, "lv_build: null K/V");
    if (src_dtype != LV_F32 && src_dtype != LV_BF16) return fail(LV_EINVAL, "lv_build: src dtype");
    cudaStream_t st = S(stream);
    const size_t src_bytes = (size_t)c->slots * n * c->cfg.d * esize(src_dtype);
    LV_CUDA(cudaMemsetAsync(c->colmax, 0, sizeof(float) * c->slots * c->DP, st));
    if (n > 0) {
        const void* ksrc = K;
        const void* vsrc = V;
        void* tmp = nullptr;
        if (where == LV_HOST) {
            LV_CUDA(cudaMallocAsync(&tmp, 2 * src_bytes, st));
            LV_CUDA(cudaMemcpyAsync(tmp, K, src_bytes, cudaMemcpyHostToDevice, st));
            LV_CUDA(cudaMemcpyAsync((char*)tmp + src_bytes, V, src_bytes, cudaMemcpyHostToDevice, st));
            ksrc = tmp;
            vsrc = (char*)tmp + src_bytes;
        }
        int rc = convert_into(c, ksrc, src_dtype, c->K, n, 0, st);
        if (!rc) rc = convert_into(c, vsrc, src_dtype, c->V, n, 0, st);
        if (tmp) cudaFreeAsync(tmp, st);
        if (rc) return rc;
        if (int rc2 = launch_summaries(c, 0, (n + c->r - 1) / c->r, n, st)) return rc2;
    }
    if (c->gi) {  // build_index over [0, n) (index.cpp:213-221)
        c->gi->indexed = 0;
        c->gi->K = 0;
        LV_CUDA(cudaMemsetAsync(c->gi->nbound, 0, sizeof(unsigned long long) * c->slots * c->gi->S, st));
        LV_CUDA(lvg::index_range(*c->gi, arena_view(c), 0, n, st));
    }
    Counters h{n, n, 0, 0};
    LV_CUDA(cudaMemcpyAsync(c->ctr, &h, sizeof(h), cudaMemcpyHostToDevice, st));
    LV_CUDA(cudaStreamSynchronize(st));
    c->version = next_version();  // a rebuild may shrink n: captured launch parameters expire
    c->n = n;
    c->indexed = n;
    c->flushes = 0;
    return LV_OK;
}

int lv_push_key(lv_ctx* c, const void* k, const void* v, int src_dtype, int where, void* stream) {
    if (!c || !k || !v) return fail(LV_EINVAL, "lv_push_key: null argument");
    std::lock_guard<std::mutex> lock(c->writer);
    if (c->n >= c->cfg.capacity) return fail(LV_ERANGE, "lv_push_key: arena capacity exhausted");
    if (src_dtype != LV_F32 && !(src_dtype == LV_BF16 && c->cfg.dtype == LV_BF16))
        return fail(LV_EINVAL, "lv_push_key: unsupported source dtype");
    cudaStream_t st = S(stream);
    const size_t bytes = (size_t)c->slots * c->cfg.d * esize(src_dtype);
    const void* kd = k;
    const void* vd = v;
    void* tmp = nullptr;
    if (where == LV_HOST) {
        LV_CUDA(cudaMallocAsync(&tmp, 2 * bytes, st));
        LV_CUDA(cudaMemcpyAsync(tmp, k, bytes, cudaMemcpyHostToDevice, st));
        LV_CUDA(cudaMemcpyAsync((char*)tmp + bytes, v, bytes, cudaMemcpyHostToDevice, st));
        kd = tmp;
        vd = (char*)tmp + bytes;
    }
    const int threads = c->DP;
    const long long B = c->cfg.buffer_capacity;
    if (c->cfg.dtype == LV_BF16) {
        auto* K = reinterpret_cast<__nv_bfloat16*>(c->K);
        auto* Vv = reinterpret_cast<__nv_bfloat16*>(c->V);
        auto* lo = reinterpret_cast<__nv_bfloat16*>(c->lo);
        auto* hi = reinterpret_cast<__nv_bfloat16*>(c->hi);
        if (src_dtype == LV_F32)
            lvk::insert_kernel<float, __nv_bfloat16><<<c->slots, threads, 0, st>>>(
                (const float*)kd, (const float*)vd, K, Vv, lo, hi, c->colmax, c->ctr, c->ins_ticket,
                c->cfg.d, c->DP, c->cap, c->cap_cells, c->r_log2, B, c->slots);
        else
            lvk::insert_kernel<__nv_bfloat16, __nv_bfloat16><<<c->slots, threads, 0, st>>>(
                (const __nv_bfloat16*)kd, (const __nv_bfloat16*)vd, K, Vv, lo, hi, c->colmax, c->ctr,
                c->ins_ticket, c->cfg.d, c->DP, c->cap, c->cap_cells, c->r_log2, B, c->slots);
    } else {
        lvk::insert_kernel<float, float><<<c->slots, threads, 0, st>>>(
            (const float*)kd, (const float*)vd, (float*)c->K, (float*)c->V, (float*)c->lo,
            (float*)c->hi, c->colmax, c->ctr, c->ins_ticket, c->cfg.d, c->DP, c->cap, c->cap_cells,
            c->r_log2, B, c->slots);
    }
    LV_CUDA(cudaGetLastError());
    if (tmp) LV_CUDA(cudaFreeAsync(tmp, st));
    if (int rc = sync_if_host(where, st)) return rc;
    c->n += 1;
    if (c->n - c->indexed >= B) {  // the insert kernel flushed (cache.cpp:7-10)
        if (c->gi) LV_CUDA(lvg::index_range(*c->gi, arena_view(c), c->indexed, c->n - c->indexed, st));
        c->indexed = c->n;
        c->flushes += 1;
    }
    return LV_OK;
}

int lv_sync_counters(lv_ctx* c, void* stream) {
    if (!c) return fail(LV_EINVAL, "lv_sync_counters: null context");
    Counters h{};
    LV_CUDA(cudaMemcpyAsync(&h, c->ctr, sizeof(h), cudaMemcpyDeviceToHost, S(stream)));
    LV_CUDA(cudaStreamSynchronize(S(stream)));
    c->n = h.n;
    c->indexed = h.indexed;
    c->flushes = h.flushes;
    return LV_OK;
}

int lv_flush(lv_ctx* c, void* stream) {
    if (!c) return fail(LV_EINVAL, "lv_flush: null context");
    std::lock_guard<std::mutex> lock(c->writer);
    if (c->n == c->indexed) return LV_EMPTY;  // cache.cpp:14
    // The summaries already cover every stored key (lv_push_key folds each key
    // into its cell), so folding the buffer into the index is a counter move.
    Counters h{c->n, c->n, c->flushes + 1, 0};
    LV_CUDA(cudaMemcpyAsync(c->ctr, &h, sizeof(h), cudaMemcpyHostToDevice, S(stream)));
    if (c->gi) LV_CUDA(lvg::index_range(*c->gi, arena_view(c), c->indexed, c->n - c->indexed, S(stream)));
    LV_CUDA(cudaStreamSynchronize(S(stream)));
    c->indexed = c->n;
    c->flushes += 1;
    return LV_OK;
}

int lv_query(lv_ctx* c, const lv_query_args* a) {
    if (!c || !a || !a->q || !a->tau) return fail(LV_EINVAL, "lv_query: null argument");
    cudaStream_t st = S(a->stream);
    Workspace w;
    carve(c, reinterpret_cast<unsigned char*>(a->workspace ? a->workspace : c->ws_mem), &w);
    const bool direct = a->where == LV_DEVICE && c->cfg.d == c->DP;
    const float* qd = a->q;
    const float* taud = a->tau;
    if (!direct) {
        if (int rc = stage_rows(c, w.q, a->q, a->where, st)) return rc;
        qd = w.q;
    }
    if (a->where == LV_HOST) {
        LV_CUDA(cudaMemcpyAsync(w.tau, a->tau, sizeof(float) * c->rows, cudaMemcpyHostToDevice, st));
        taud = w.tau;
    }
    float* outd = direct ? a->out : (a->out ? w.out : nullptr);
    float* pod = (a->partial && direct) ? a->partial : (a->partial ? w.part_out : nullptr);
    int* cntd = a->counts ? (a->where == LV_DEVICE ? a->counts : w.counts) : nullptr;
    // the bf16 layer kernel writes every count itself (its merge sums the team's); the fp32
    // kernels accumulate into zeroed counts
    if (cntd && c->cfg.dtype != LV_BF16) LV_CUDA(cudaMemsetAsync(cntd, 0, sizeof(int) * c->rows * 4, st));
    if (a->totals) LV_CUDA(cudaMemsetAsync(a->totals, 0, sizeof(uint64_t) * 4, st));
    if (a->sel_bits)
        LV_CUDA(cudaMemsetAsync(a->sel_bits, 0, sizeof(uint32_t) * c->rows * c->bits_words, st));
    if (a->cand_bits) {
        if (c->cfg.dtype != LV_F32) return fail(LV_EINVAL, "lv_query: cand_bits needs an fp32 cache");
        LV_CUDA(cudaMemsetAsync(a->cand_bits, 0, sizeof(uint32_t) * c->slots * c->bits_words, st));
    }
    if (int rc = run_query_kernel(c, lvk::kQuery, qd, taud, 0, a->scale, a->strict, w, outd, pod,
                                  a->sel_bits, cntd, reinterpret_cast<unsigned long long*>(a->totals),
                                  st, a->cand_bits))
        return rc;
    const cudaMemcpyKind kind = a->where == LV_HOST ? cudaMemcpyDeviceToHost : cudaMemcpyDeviceToDevice;
    if (a->out && !direct)
        LV_CUDA(cudaMemcpy2DAsync(a->out, sizeof(float) * c->cfg.d, w.out, sizeof(float) * c->DP,
                                  sizeof(float) * c->cfg.d, c->rows, kind, st));
    if (a->partial && !direct) {
        // (m, l, o[d]) rows of the caller's d+2 width
        LV_CUDA(cudaMemcpy2DAsync(a->partial, sizeof(float) * (c->cfg.d + 2), w.part_out,
                                  sizeof(float) * (c->DP + 2), sizeof(float) * (c->cfg.d + 2), c->rows,
                                  kind, st));
    }
    if (a->counts && a->where == LV_HOST)
        LV_CUDA(cudaMemcpyAsync(a->counts, w.counts, sizeof(int) * c->rows * 4, cudaMemcpyDeviceToHost, st));
    return sync_if_host(a->where, st);
}

size_t lv_query_layers_staging_bytes(const lv_ctx* c, int L) {
    if (!c || L < 1) return 0;
    const size_t rows = (size_t)c->rows, d = (size_t)c->cfg.d;
    return align256(sizeof(float) * L * rows * d) * 2 + align256(sizeof(float) * L * rows);
}

int lv_query_layers(lv_ctx* const* ctxs, int L, const float* q, const float* tau, float scale, int strict,
                    float* out, void* staging, void* stream) {
    if (!ctxs || L < 1 || !q || !tau || !out) return fail(LV_EINVAL, "lv_query_layers: null argument");
    lv_ctx* c0 = ctxs[0];
    if (!c0) return fail(LV_EINVAL, "lv_query_layers: null context");
    for (int l = 1; l < L; ++l)
        if (!ctxs[l] || ctxs[l]->rows != c0->rows || ctxs[l]->cfg.d != c0->cfg.d)
            return fail(LV_EINVAL, "lv_query_layers: every layer needs the same batch, H_q and d");
    cudaStream_t st = S(stream);
    const size_t rows = (size_t)c0->rows, d = (size_t)c0->cfg.d;
    const size_t need = lv_query_layers_staging_bytes(c0, L);
    std::unique_lock<std::mutex> lock(c0->stage_mu, std::defer_lock);
    unsigned char* base = static_cast<unsigned char*>(staging);
    if (!base) {  // the first context's internal staging: calls sharing it serialise
        lock.lock();
        if (c0->stage_bytes < need) {
            if (c0->stage) LV_CUDA(cudaFree(c0->stage));
            c0->stage = nullptr;
            c0->stage_bytes = 0;
            LV_CUDA(cudaMalloc(&c0->stage, need));
            c0->stage_bytes = need;
        }
        base = static_cast<unsigned char*>(c0->stage);
    }
    float* qd = reinterpret_cast<float*>(base);
    float* od = reinterpret_cast<float*>(base + align256(sizeof(float) * L * rows * d));
    float* td = reinterpret_cast<float*>(base + 2 * align256(sizeof(float) * L * rows * d));
    // one copy in for every layer's q and tau, the L queries back to back, one copy out
    auto enqueue = [&]() -> int {
        LV_CUDA(cudaMemcpyAsync(qd, q, sizeof(float) * L * rows * d, cudaMemcpyHostToDevice, st));
        LV_CUDA(cudaMemcpyAsync(td, tau, sizeof(float) * L * rows, cudaMemcpyHostToDevice, st));
        for (int l = 0; l < L; ++l) {
            lv_query_args a{};
            a.q = qd + (size_t)l * rows * d;
            a.tau = td + (size_t)l * rows;
            a.scale = scale;
            a.algo = LV_ALGO_TA;
            a.strict = strict;
            a.where = LV_DEVICE;
            a.out = od + (size_t)l * rows * d;
            a.stream = stream;
            if (int rc = lv_query(ctxs[l], &a)) return rc;
        }
        LV_CUDA(cudaMemcpyAsync(out, od, sizeof(float) * L * rows * d, cudaMemcpyDeviceToHost, st));
        return LV_OK;
    };
    // Mapped (page-locked, UVA) host buffers: no copy-engine transfers at all. One launch
    // stages every layer's q and tau from host memory, and each layer kernel writes its output
    // rows straight into the host buffer (d == DP: the kernel's rows are the caller's rows).
    const float *qm = nullptr, *tm = nullptr;
    float* om = nullptr;
    {
        void* p = nullptr;
        if (cudaHostGetDevicePointer(&p, const_cast<float*>(q), 0) == cudaSuccess) qm = static_cast<const float*>(p);
        if (cudaHostGetDevicePointer(&p, const_cast<float*>(tau), 0) == cudaSuccess) tm = static_cast<const float*>(p);
        if (cudaHostGetDevicePointer(&p, out, 0) == cudaSuccess) om = static_cast<float*>(p);
        cudaGetLastError();
        if (const char* e = std::getenv("LV_LAYERS_MAPPED"))  // 0: copy-engine transfers (A/B)
            if (!std::atoi(e)) qm = nullptr;
    }
    const bool mapped = qm && tm && om && c0->DP == (int)d;
    auto enqueue_mapped = [&]() -> int {
        const long long nq = (long long)(L * rows * d), nt = (long long)(L * rows);
        const unsigned blocks = (unsigned)std::min<long long>((nq + nt + 255) / 256, 4LL * c0->sms);
        lvk::stage_in_kernel<<<blocks, 256, 0, st>>>(qm, qd, nq, tm, td, nt);
        LV_CUDA(cudaGetLastError());
        for (int l = 0; l < L; ++l) {
            lv_query_args a{};
            a.q = qd + (size_t)l * rows * d;
            a.tau = td + (size_t)l * rows;
            a.scale = scale;
            a.algo = LV_ALGO_TA;
            a.strict = strict;
            a.where = LV_DEVICE;
            a.out = om + (size_t)l * rows * d;
            a.stream = stream;
            if (int rc = lv_query(ctxs[l], &a)) return rc;
        }
        return LV_OK;
    };
    // The step as a CUDA graph (one launch instead of 2 + L + 1, kernels scheduled back to back)
    // when it can be captured: a non-default stream that is not itself capturing, page-locked
    // host buffers, the context-internal staging (its lock serialises the calls).
    bool graph = lock.owns_lock() && st != nullptr;
    if (graph) {
        cudaStreamCaptureStatus cs = cudaStreamCaptureStatusNone;
        graph = cudaStreamIsCapturing(st, &cs) == cudaSuccess && cs == cudaStreamCaptureStatusNone;
        for (const void* h : {(const void*)q, (const void*)tau, (const void*)out}) {
            cudaPointerAttributes pa{};
            graph = graph && cudaPointerGetAttributes(&pa, h) == cudaSuccess && pa.type == cudaMemoryTypeHost;
        }
        cudaGetLastError();
        if (const char* e = std::getenv("LV_LAYERS_GRAPH")) graph = graph && std::atoi(e) != 0;
    }
    if (!graph) {
        if (int rc = mapped ? enqueue_mapped() : enqueue()) return rc;
        LV_CUDA(cudaStreamSynchronize(st));
        return LV_OK;
    }
    auto& g = c0->lgraph;
    bool hit = g.exec && g.q == q && g.tau == tau && g.out == out && g.base == base && g.scale == scale &&
               g.strict == strict && g.st == st && (int)g.ctxs.size() == L;
    for (int l = 0; hit && l < L; ++l) hit = g.ctxs[l] == ctxs[l] && g.versions[l] == ctxs[l]->version;
    if (!hit) {
        if (g.exec) cudaGraphExecDestroy(g.exec);
        g.exec = nullptr;
        LV_CUDA(cudaStreamBeginCapture(st, cudaStreamCaptureModeThreadLocal));
        const int rc = mapped ? enqueue_mapped() : enqueue();
        cudaGraph_t gr = nullptr;
        const cudaError_t e = cudaStreamEndCapture(st, &gr);
        if (rc) {
            if (gr) cudaGraphDestroy(gr);
            return rc;
        }
        if (e != cudaSuccess) return fail(LV_ERUNTIME, std::string("lv_query_layers capture: ") + cudaGetErrorString(e));
        const cudaError_t ei = cudaGraphInstantiate(&g.exec, gr, 0);
        cudaGraphDestroy(gr);
        if (ei != cudaSuccess) return fail(LV_ERUNTIME, std::string("lv_query_layers graph: ") + cudaGetErrorString(ei));
        g.ctxs.assign(ctxs, ctxs + L);
        g.versions.resize(L);
        for (int l = 0; l < L; ++l) g.versions[l] = ctxs[l]->version;
        g.q = q;
        g.tau = tau;
        g.out = out;
        g.base = base;
        g.scale = scale;
        g.strict = strict;
        g.st = st;
    }
    LV_CUDA(cudaGraphLaunch(g.exec, st));
    LV_CUDA(cudaStreamSynchronize(st));
    return LV_OK;
}

namespace {
// ids + q staged on the device (DEVICE inputs used in place); scratch from the stream-ordered pool
struct IdsQ {
    const unsigned* ids = nullptr;
    float* q = nullptr;   // [DP], zero-padded
    void* mem = nullptr;
};
int stage_ids_q(lv_ctx* c, const uint32_t* ids, int64_t nids, const float* q, int where, cudaStream_t st, IdsQ* o,
                size_t extra, void** extra_p) {
    const size_t bi = where == LV_HOST ? align256(sizeof(uint32_t) * nids) : 0;
    if (where == LV_HOST)
        for (int64_t i = 0; i < nids; ++i)
            if ((long long)ids[i] >= c->n) return fail(LV_ERANGE, "key id >= n");
    LV_CUDA(cudaMallocAsync(&o->mem, bi + align256(sizeof(float) * c->DP) + align256(extra), st));
    unsigned char* m = static_cast<unsigned char*>(o->mem);
    if (where == LV_HOST) {
        LV_CUDA(cudaMemcpyAsync(m, ids, sizeof(uint32_t) * nids, cudaMemcpyHostToDevice, st));
        o->ids = reinterpret_cast<const unsigned*>(m);
    } else {
        o->ids = ids;
    }
    o->q = reinterpret_cast<float*>(m + bi);
    LV_CUDA(cudaMemsetAsync(o->q, 0, sizeof(float) * c->DP, st));
    LV_CUDA(cudaMemcpyAsync(o->q, q, sizeof(float) * c->cfg.d,
                            where == LV_HOST ? cudaMemcpyHostToDevice : cudaMemcpyDeviceToDevice, st));
    if (extra_p) *extra_p = m + bi + align256(sizeof(float) * c->DP);
    return LV_OK;
}
}  // namespace

int lv_exact_check(lv_ctx* c, int slot, const uint32_t* ids, int64_t nids, const float* q, float tau, int where,
                   uint8_t* flags, void* stream) {
    if (!c || !q || (nids > 0 && (!ids || !flags)) || nids < 0) return fail(LV_EINVAL, "exact_check: bad arguments");
    if (slot < 0 || slot >= c->slots) return fail(LV_ERANGE, "exact_check: slot out of range");
    if (nids == 0) return LV_OK;
    cudaStream_t st = S(stream);
    IdsQ in;
    void* fl = nullptr;
    if (int rc = stage_ids_q(c, ids, nids, q, where, st, &in, where == LV_HOST ? (size_t)nids : 0, &fl)) return rc;
    unsigned char* fd = where == LV_HOST ? static_cast<unsigned char*>(fl) : flags;
    const size_t es = esize(c->cfg.dtype);
    const void* Ks = (const unsigned char*)c->K + (size_t)slot * c->cap * c->DP * es;
    const unsigned tb = (unsigned)((nids + 127) / 128);
#define LV_EX(T, D) lvk::exact_flags_kernel<T, D><<<tb, 128, 0, st>>>((const T*)Ks, in.ids, nids, in.q, tau, fd);
    if (c->cfg.dtype == LV_BF16) {
        if (c->DP == 64) { LV_EX(__nv_bfloat16, 64) } else if (c->DP == 128) { LV_EX(__nv_bfloat16, 128) } else { LV_EX(__nv_bfloat16, 256) }
    } else {
        if (c->DP == 64) { LV_EX(float, 64) } else if (c->DP == 128) { LV_EX(float, 128) } else { LV_EX(float, 256) }
    }
#undef LV_EX
    LV_CUDA(cudaGetLastError());
    if (where == LV_HOST) LV_CUDA(cudaMemcpyAsync(flags, fd, (size_t)nids, cudaMemcpyDeviceToHost, st));
    LV_CUDA(cudaFreeAsync(in.mem, st));
    return sync_if_host(where, st);
}

int lv_attention_weights(lv_ctx* c, int slot, const uint32_t* ids, int64_t nids, const float* q, float scale,
                         float m, float l, int where, float* weights, void* stream) {
    if (!c || !q || (nids > 0 && (!ids || !weights)) || nids < 0)
        return fail(LV_EINVAL, "attention_weights: bad arguments");
    if (slot < 0 || slot >= c->slots) return fail(LV_ERANGE, "attention_weights: slot out of range");
    if (nids == 0) return LV_OK;
    cudaStream_t st = S(stream);
    IdsQ in;
    void* sc_mem = nullptr;
    if (int rc = stage_ids_q(c, ids, nids, q, where, st, &in, sizeof(float) * nids, &sc_mem)) return rc;
    float* scores = where == LV_HOST ? static_cast<float*>(sc_mem) : weights;
    const float sc = scale != 0.0f ? scale : (float)(1.0 / std::sqrt((double)c->cfg.d));
    const size_t es = esize(c->cfg.dtype);
    const void* Ks = (const unsigned char*)c->K + (size_t)slot * c->cap * c->DP * es;
    const unsigned tb = (unsigned)((nids + 127) / 128);
#define LV_W(T, D) lvk::token_scores_kernel<T, D><<<tb, 128, 0, st>>>((const T*)Ks, in.ids, nids, in.q, sc, scores);
    if (c->cfg.dtype == LV_BF16) {
        if (c->DP == 64) { LV_W(__nv_bfloat16, 64) } else if (c->DP == 128) { LV_W(__nv_bfloat16, 128) } else { LV_W(__nv_bfloat16, 256) }
    } else {
        if (c->DP == 64) { LV_W(float, 64) } else if (c->DP == 128) { LV_W(float, 128) } else { LV_W(float, 256) }
    }
#undef LV_W
    lvk::attn_weights_kernel<<<tb, 128, 0, st>>>(scores, nids, m, l);
    LV_CUDA(cudaGetLastError());
    if (where == LV_HOST) LV_CUDA(cudaMemcpyAsync(weights, scores, sizeof(float) * nids, cudaMemcpyDeviceToHost, st));
    LV_CUDA(cudaFreeAsync(in.mem, st));
    return sync_if_host(where, st);
}

int lv_subspace_thresholds(lv_ctx* c, int slot, const float* q, float tau, int S, int where, float* out,
                           void* stream) {
    if (!c || !q || !out) return fail(LV_EINVAL, "derive_subspace_thresholds: null argument");
    if (slot < 0 || slot >= c->slots) return fail(LV_ERANGE, "derive_subspace_thresholds: slot out of range");
    const int d = c->cfg.d;
    if (S < 1 || S > d) return fail(LV_EINVAL, "SubspaceLayout: 1 <= S <= d required");
    // SubspaceLayout (core.hpp:41-50): S contiguous slices, the first d % S one wider
    std::vector<int> offs(S + 1, 0);
    for (int i = 0; i < S; ++i) offs[i + 1] = offs[i] + d / S + (i < d % S ? 1 : 0);
    cudaStream_t st = reinterpret_cast<cudaStream_t>(stream);
    const long long ncells = (c->indexed + c->r - 1) >> c->r_log2;  // cells holding indexed keys
    std::vector<float> qh(d);
    if (where == LV_HOST) {
        std::memcpy(qh.data(), q, sizeof(float) * d);
    } else {
        LV_CUDA(cudaMemcpyAsync(qh.data(), q, sizeof(float) * d, cudaMemcpyDeviceToHost, st));
        LV_CUDA(cudaStreamSynchronize(st));
    }
    std::vector<double> peak(S, 0.0), nb(S, 0.0);
    if (ncells > 0) {
        void* mem = nullptr;
        const size_t bq = align256(sizeof(float) * c->DP), bo = align256(sizeof(int) * (S + 1));
        LV_CUDA(cudaMallocAsync(&mem, bq + bo + 2 * align256(sizeof(double) * S), st));
        unsigned char* m = static_cast<unsigned char*>(mem);
        float* qd = reinterpret_cast<float*>(m);
        int* od = reinterpret_cast<int*>(m + bq);
        double* pd = reinterpret_cast<double*>(m + bq + bo);
        double* nd = reinterpret_cast<double*>(m + bq + bo + align256(sizeof(double) * S));
        LV_CUDA(cudaMemsetAsync(qd, 0, sizeof(float) * c->DP, st));
        LV_CUDA(cudaMemcpyAsync(qd, qh.data(), sizeof(float) * d, cudaMemcpyHostToDevice, st));
        LV_CUDA(cudaMemcpyAsync(od, offs.data(), sizeof(int) * (S + 1), cudaMemcpyHostToDevice, st));
        const size_t es = esize(c->cfg.dtype);
        const void* rows = (const unsigned char*)c->lo + (size_t)slot * c->cap_cells * 2 * c->DP * es;
#define LV_SP(T, D) lvk::subspace_peaks_kernel<T, D><<<S, 256, 0, st>>>((const T*)rows, ncells, qd, od, pd, nd);
        if (c->cfg.dtype == LV_BF16) {
            if (c->DP == 64) { LV_SP(__nv_bfloat16, 64) } else if (c->DP == 128) { LV_SP(__nv_bfloat16, 128) } else { LV_SP(__nv_bfloat16, 256) }
        } else {
            if (c->DP == 64) { LV_SP(float, 64) } else if (c->DP == 128) { LV_SP(float, 128) } else { LV_SP(float, 256) }
        }
#undef LV_SP
        LV_CUDA(cudaGetLastError());
        LV_CUDA(cudaMemcpyAsync(peak.data(), pd, sizeof(double) * S, cudaMemcpyDeviceToHost, st));
        LV_CUDA(cudaMemcpyAsync(nb.data(), nd, sizeof(double) * S, cudaMemcpyDeviceToHost, st));
        LV_CUDA(cudaFreeAsync(mem, st));
        LV_CUDA(cudaStreamSynchronize(st));
    }
    // query.cpp:322-335: slack and tau_s, in double
    double nbsq = 0.0, qq = 0.0, total = 0.0;
    for (int s = 0; s < S; ++s) nbsq += nb[s] * nb[s];
    for (int i = 0; i < d; ++i) qq += (double)qh[i] * qh[i];
    const double eps = 1.1920928955078125e-07;
    const double slack = S == 1 ? 0.0 : 4.0 * d * eps * std::sqrt(qq) * std::sqrt(nbsq);
    for (int s = 0; s < S; ++s) total += peak[s];
    std::vector<float> res(S);
    for (int s = 0; s < S; ++s) res[s] = (float)((double)tau - (total - peak[s]) - slack);
    if (where == LV_HOST) {
        std::memcpy(out, res.data(), sizeof(float) * S);
    } else {
        LV_CUDA(cudaMemcpyAsync(out, res.data(), sizeof(float) * S, cudaMemcpyHostToDevice, st));
        LV_CUDA(cudaStreamSynchronize(st));
    }
    return LV_OK;
}

int lv_dense_decode(lv_ctx* c, const float* q, float scale, int where, float* out, float* partial,
                    void* stream) {
    if (!c || !q) return fail(LV_EINVAL, "lv_dense_decode: null argument");
    cudaStream_t st = S(stream);
    Workspace w;
    carve(c, reinterpret_cast<unsigned char*>(c->ws_mem), &w);
    const bool direct = where == LV_DEVICE && c->cfg.d == c->DP;
    const float* qd = q;
    if (!direct) {
        if (int rc = stage_rows(c, w.q, q, where, st)) return rc;
        qd = w.q;
    }
    float* outd = direct ? out : (out ? w.out : nullptr);
    float* pod = (partial && direct) ? partial : (partial ? w.part_out : nullptr);
    if (int rc = run_query_kernel(c, lvk::kDense, qd, nullptr, 0, scale, 0, w, outd, pod, nullptr,
                                  nullptr, nullptr, st))
        return rc;
    const cudaMemcpyKind kind = where == LV_HOST ? cudaMemcpyDeviceToHost : cudaMemcpyDeviceToDevice;
    if (out && !direct)
        LV_CUDA(cudaMemcpy2DAsync(out, sizeof(float) * c->cfg.d, w.out, sizeof(float) * c->DP,
                                  sizeof(float) * c->cfg.d, c->rows, kind, st));
    if (partial && !direct)
        LV_CUDA(cudaMemcpy2DAsync(partial, sizeof(float) * (c->cfg.d + 2), w.part_out,
                                  sizeof(float) * (c->DP + 2), sizeof(float) * (c->cfg.d + 2), c->rows,
                                  kind, st));
    return sync_if_host(where, st);
}

int lv_brute_force_range(lv_ctx* c, const float* q, const float* tau, int64_t limit, int where,
                         uint32_t* sel_bits, void* stream) {
    if (!c || !q || !tau || !sel_bits) return fail(LV_EINVAL, "lv_brute_force_range: null argument");
    if (limit < -1 || limit > c->n) return fail(LV_EINVAL, "brute_force_range: limit > n");
    if (limit == -1) limit = c->cap;  // every stored key: the kernel clamps to the DEVICE count
    cudaStream_t st = S(stream);
    Workspace w;
    carve(c, reinterpret_cast<unsigned char*>(c->ws_mem), &w);
    const float* qd = q;
    const float* taud = tau;
    if (!(where == LV_DEVICE && c->cfg.d == c->DP)) {
        if (int rc = stage_rows(c, w.q, q, where, st)) return rc;
        qd = w.q;
    }
    if (where == LV_HOST) {
        LV_CUDA(cudaMemcpyAsync(w.tau, tau, sizeof(float) * c->rows, cudaMemcpyHostToDevice, st));
        taud = w.tau;
    }
    LV_CUDA(cudaMemsetAsync(sel_bits, 0, sizeof(uint32_t) * c->rows * c->bits_words, st));
    if (int rc = run_query_kernel(c, lvk::kBrute, qd, taud, limit, 0.0f, 0, w, nullptr, nullptr,
                                  sel_bits, nullptr, nullptr, st))
        return rc;
    return sync_if_host(where, st);
}

int lv_bitmap_to_ids(const uint32_t* bits, int64_t words, int64_t rows, int64_t limit, uint32_t* ids,
                     int64_t ids_stride, int32_t* count, void* stream) {
    if (!bits || !ids || !count || rows < 0 || limit > words * 32)
        return fail(LV_EINVAL, "lv_bitmap_to_ids: bad arguments");
    if (rows == 0) return LV_OK;
    lvk::bitmap_ids_kernel<<<(unsigned)rows, 256, 0, S(stream)>>>(bits, words, limit, ids, ids_stride,
                                                                  count);
    LV_CUDA(cudaGetLastError());
    return LV_OK;
}

// ---- threshold oracle (threshold.hpp:29-50, threshold.cpp:40-103) ----------------------

struct lv_reservoir {
    size_t capacity;
    std::vector<uint32_t> ids;
    size_t seen = 0;
    std::mt19937_64 rng;
    lv_reservoir(size_t cap, uint64_t seed) : capacity(cap), rng(seed) {}
};

int lv_reservoir_create(int64_t capacity, uint64_t seed, lv_reservoir** out) {
    if (!out) return fail(LV_EINVAL, "lv_reservoir_create: null out");
    if (capacity < 1) return fail(LV_EINVAL, "Reservoir: capacity >= 1 required");  // threshold.hpp:33
    *out = new lv_reservoir((size_t)capacity, seed);
    return LV_OK;
}

int lv_reservoir_destroy(lv_reservoir* res) {
    delete res;
    return LV_OK;
}

int lv_reservoir_update(lv_reservoir* res, uint32_t id, int64_t* slot) {
    if (!res) return fail(LV_EINVAL, "lv_reservoir_update: null reservoir");
    ++res->seen;
    int64_t at = -1;
    if (res->ids.size() < res->capacity) {
        at = (int64_t)res->ids.size();
        res->ids.push_back(id);
    } else {
        // item t replaces a uniform position with probability capacity / t: the
        // same distribution object and engine calls as threshold.cpp:49-54
        std::uniform_int_distribution<std::size_t> pick(0, res->seen - 1);
        const std::size_t s = pick(res->rng);
        if (s < res->capacity) {
            res->ids[s] = id;
            at = (int64_t)s;
        }
    }
    if (slot) *slot = at;
    return LV_OK;
}

int64_t lv_reservoir_size(const lv_reservoir* res) { return res ? (int64_t)res->ids.size() : -1; }
int64_t lv_reservoir_seen(const lv_reservoir* res) { return res ? (int64_t)res->seen : -1; }
int64_t lv_reservoir_capacity(const lv_reservoir* res) { return res ? (int64_t)res->capacity : -1; }

int lv_reservoir_ids(const lv_reservoir* res, uint32_t* ids) {
    if (!res || !ids) return fail(LV_EINVAL, "lv_reservoir_ids: null argument");
    if (!res->ids.empty()) std::memcpy(ids, res->ids.data(), sizeof(uint32_t) * res->ids.size());
    return LV_OK;
}

int lv_estimate_tau(lv_ctx* c, const uint32_t* ids, int64_t count, int64_t ld, const float* q, int variant,
                    int m, double alpha, int where, float* tau, void* stream) {
    if (!c || !ids || !q || !tau) return fail(LV_EINVAL, "lv_estimate_tau: null argument");
    // OracleConfig::validate (threshold.hpp:17-22), then estimate_tau's own checks
    if (variant < LV_TAU_MAX || variant > LV_TAU_BUDGET) return fail(LV_EINVAL, "estimate_tau: unknown variant");
    if (variant == LV_TAU_TOPK && m < 1) return fail(LV_EINVAL, "OracleConfig: m >= 1 required");
    if (variant == LV_TAU_BUDGET && !(alpha > 0.0 && alpha < 1.0))
        return fail(LV_EINVAL, "OracleConfig: 0 < alpha < 1 required");
    if (count <= 0) return fail(LV_EINVAL, "estimate_tau: empty reservoir");
    if (variant == LV_TAU_TOPK && count < m) return fail(LV_EINVAL, "estimate_tau: sample smaller than topk rank");
    if (variant == LV_TAU_GAP && count < 2) return fail(LV_EINVAL, "estimate_tau: gap needs >= 2 samples");
    if (count > 8192) return fail(LV_EINVAL, "estimate_tau: reservoir larger than 8192 on the device");
    if (ld < count) return fail(LV_EINVAL, "estimate_tau: ld < count");
    const size_t n = (size_t)count;
    int mode = lvkt::kPick, pick = 0;
    if (variant == LV_TAU_TOPK) {
        pick = m - 1;
    } else if (variant == LV_TAU_GAP) {
        mode = lvkt::kGap;
    } else if (variant == LV_TAU_MEANMAX) {
        mode = lvkt::kMeanMax;
    } else if (variant == LV_TAU_BUDGET) {  // threshold.cpp:98-101, same expression
        const auto idx = static_cast<std::size_t>(
            std::min<double>(std::ceil((1.0 - alpha) * static_cast<double>(n)), static_cast<double>(n - 1)));
        pick = (int)(n - 1 - idx);
    }
    cudaStream_t st = S(stream);
    Workspace w;
    carve(c, reinterpret_cast<unsigned char*>(c->ws_mem), &w);
    const uint32_t* idd = ids;
    uint32_t* ids_tmp = nullptr;
    if (where == LV_HOST) {
        for (int64_t s = 0; s < c->slots; ++s)
            for (int64_t i = 0; i < count; ++i)
                if ((long long)ids[s * ld + i] >= c->n) return fail(LV_ERANGE, "estimate_tau: id >= n");
        LV_CUDA(cudaMallocAsync(reinterpret_cast<void**>(&ids_tmp), sizeof(uint32_t) * c->slots * ld, st));
        LV_CUDA(cudaMemcpyAsync(ids_tmp, ids, sizeof(uint32_t) * c->slots * ld, cudaMemcpyHostToDevice, st));
        idd = ids_tmp;
    }
    const float* qd = q;
    if (!(where == LV_DEVICE && c->cfg.d == c->DP)) {
        if (int rc = stage_rows(c, w.q, q, where, st)) return rc;
        qd = w.q;
    }
    float* taud = where == LV_HOST ? w.tau : tau;
    int np2 = 32;  // at least one warp: the sort's shuffle stages need whole warps
    while (np2 < count) np2 <<= 1;
    const size_t esz = c->cfg.dtype == LV_BF16 ? 2 : 4;
    const int rpc = c->cfg.dtype == LV_BF16 ? lvkt::stage_rows<__nv_bfloat16>(c->DP) : lvkt::stage_rows<float>(c->DP);
    const size_t smem = (size_t)rpc * (c->DP * esz + 16) + sizeof(float) * (c->DP + 2 * (size_t)np2);
    const int threads = np2 <= 1024 ? np2 : 256;  // one score per thread up to 1024
    LV_CUDA(lvl::func_smem(c->cfg.dtype == LV_BF16
                               ? reinterpret_cast<const void*>(lvkt::estimate_tau_kernel<__nv_bfloat16>)
                               : reinterpret_cast<const void*>(lvkt::estimate_tau_kernel<float>),
                           (int)smem));
    if (c->cfg.dtype == LV_BF16)
        lvkt::estimate_tau_kernel<__nv_bfloat16><<<(unsigned)c->rows, threads, smem, st>>>(
            reinterpret_cast<const __nv_bfloat16*>(c->K), c->cap, c->DP, c->cfg.d, c->G, idd, ld, (int)count, qd,
            mode, pick, np2, taud);
    else
        lvkt::estimate_tau_kernel<float><<<(unsigned)c->rows, threads, smem, st>>>(
            reinterpret_cast<const float*>(c->K), c->cap, c->DP, c->cfg.d, c->G, idd, ld, (int)count, qd, mode,
            pick, np2, taud);
    LV_CUDA(cudaGetLastError());
    if (where == LV_HOST) {
        LV_CUDA(cudaMemcpyAsync(tau, w.tau, sizeof(float) * c->rows, cudaMemcpyDeviceToHost, st));
        LV_CUDA(cudaFreeAsync(ids_tmp, st));
    }
    return sync_if_host(where, st);
}

int lv_bits_diff(const uint32_t* a, const uint32_t* b, int64_t words, int64_t rows, int32_t* violations,
                 void* stream) {
    if (!a || !b || !violations || words < 0 || rows < 0) return fail(LV_EINVAL, "lv_bits_diff: bad arguments");
    if (rows == 0 || words == 0) return LV_OK;
    lvkt::bits_diff_kernel<<<(unsigned)rows, 256, 0, S(stream)>>>(a, b, words, violations);
    LV_CUDA(cudaGetLastError());
    return LV_OK;
}

int lv_step_load(const int64_t* step, const void* src, int64_t stride, void* dst, int64_t bytes, void* stream) {
    if (!step || !src || !dst || stride < 0 || bytes < 0 || bytes % 4 || stride % 4)
        return fail(LV_EINVAL, "lv_step_load: bad arguments (4-byte multiples required)");
    if (bytes == 0) return LV_OK;
    const long long w = bytes / 4;
    lvkt::step_copy_kernel<<<(unsigned)std::min<long long>((w + 255) / 256, 148), 256, 0, S(stream)>>>(
        reinterpret_cast<const long long*>(step), (const uint32_t*)src, (uint32_t*)dst, stride / 4, w, 0);
    LV_CUDA(cudaGetLastError());
    return LV_OK;
}

int lv_step_store(const int64_t* step, const void* src, void* dst, int64_t stride, int64_t bytes, void* stream) {
    if (!step || !src || !dst || stride < 0 || bytes < 0 || bytes % 4 || stride % 4)
        return fail(LV_EINVAL, "lv_step_store: bad arguments (4-byte multiples required)");
    if (bytes == 0) return LV_OK;
    const long long w = bytes / 4;
    lvkt::step_copy_kernel<<<(unsigned)std::min<long long>((w + 255) / 256, 148), 256, 0, S(stream)>>>(
        reinterpret_cast<const long long*>(step), (const uint32_t*)src, (uint32_t*)dst, stride / 4, w, 1);
    LV_CUDA(cudaGetLastError());
    return LV_OK;
}

int lv_step_copies(const int64_t* step, const lv_step_copy* copies, int ncopies, void* stream) {
    if (!step || !copies || ncopies < 1 || ncopies > 8) return fail(LV_EINVAL, "lv_step_copies: 1..8 copies");
    lvkt::StepCopies cs{};
    long long maxw = 0;
    for (int i = 0; i < ncopies; ++i) {
        const lv_step_copy& c = copies[i];
        if (!c.src || !c.dst || c.stride < 0 || c.bytes < 0 || c.bytes % 4 || c.stride % 4 || (c.dir != 0 && c.dir != 1))
            return fail(LV_EINVAL, "lv_step_copies: bad copy (4-byte multiples, dir 0 or 1)");
        cs.c[i] = {(const uint32_t*)c.src, (uint32_t*)c.dst, c.stride / 4, c.bytes / 4, c.dir};
        maxw = std::max<long long>(maxw, c.bytes / 4);
    }
    cs.n = ncopies;
    if (maxw == 0) return LV_OK;
    dim3 grid((unsigned)std::min<long long>((maxw + 255) / 256, 64), (unsigned)ncopies);
    lvkt::step_copies_kernel<<<grid, 256, 0, S(stream)>>>(reinterpret_cast<const long long*>(step), cs);
    LV_CUDA(cudaGetLastError());
    return LV_OK;
}

int lv_step_reservoir(const int64_t* step, const int32_t* slot_of_step, int64_t row0, uint32_t* ids, int nslots,
                      int64_t ld, void* stream) {
    if (!step || !slot_of_step || !ids || row0 < 0 || nslots < 1 || nslots > 1024 || ld < 0)
        return fail(LV_EINVAL, "lv_step_reservoir: bad arguments");
    lvkt::step_reservoir_kernel<<<1, nslots, 0, S(stream)>>>(reinterpret_cast<const long long*>(step), slot_of_step,
                                                            row0, ids, nslots, ld);
    LV_CUDA(cudaGetLastError());
    return LV_OK;
}

int lv_step_epilogue(int64_t* step, const lv_step_copy* copies, int ncopies, const int32_t* slot_of_step,
                     int64_t row0, uint32_t* ids, int nslots, int64_t ld, void* stream) {
    if (!step || ncopies < 0 || ncopies > 8 || (ncopies && !copies) || (ids && (!slot_of_step || row0 < 0 || nslots < 1 || ld < 0)))
        return fail(LV_EINVAL, "lv_step_epilogue: bad arguments");
    lvkt::StepCopies cs{};
    for (int i = 0; i < ncopies; ++i) {
        const lv_step_copy& c = copies[i];
        if (!c.src || !c.dst || c.stride < 0 || c.bytes < 0 || c.bytes % 4 || c.stride % 4 || (c.dir != 0 && c.dir != 1))
            return fail(LV_EINVAL, "lv_step_epilogue: bad copy (4-byte multiples, dir 0 or 1)");
        cs.c[i] = {(const uint32_t*)c.src, (uint32_t*)c.dst, c.stride / 4, c.bytes / 4, c.dir};
    }
    cs.n = ncopies;
    lvkt::step_epilogue_kernel<<<1, 256, 0, S(stream)>>>(reinterpret_cast<long long*>(step), cs, slot_of_step, row0,
                                                         ids, nslots, ld);
    LV_CUDA(cudaGetLastError());
    return LV_OK;
}

int lv_step_advance(int64_t* step, void* stream) {
    if (!step) return fail(LV_EINVAL, "lv_step_advance: null step");
    lvkt::step_advance_kernel<<<1, 1, 0, S(stream)>>>(reinterpret_cast<long long*>(step));
    LV_CUDA(cudaGetLastError());
    return LV_OK;
}

int lv_lse_merge(const float* partials, int P, int64_t rows, int d, float* out, void* stream) {
    if (!partials || !out || P < 1 || P > 64 || rows < 0 || d < 1)
        return fail(LV_EINVAL, "lv_lse_merge: bad arguments");
    if (rows == 0) return LV_OK;
    lvk::lse_merge_kernel<<<(unsigned)rows, 128, 0, S(stream)>>>(partials, P, rows, d, d + 2, out, d,
                                                                 nullptr);
    LV_CUDA(cudaGetLastError());
    return LV_OK;
}

int lv_sparse_attention(lv_ctx* c, int slot, const uint32_t* buffer_ids, int64_t nbuf,
                        const uint32_t* selected_ids, int64_t nsel, const float* q, float scale,
                        int where, float* out, float* weights, int64_t* ntok, void* stream) {
    if (!c || !q || !out) return fail(LV_EINVAL, "sparse_attention: null argument");
    if (slot < 0 || slot >= c->slots) return fail(LV_ERANGE, "sparse_attention: slot out of range");
    if (nbuf < 0 || nsel < 0) return fail(LV_EINVAL, "sparse_attention: negative count");
    cudaStream_t st = S(stream);
    // tokens = sort ∪ unique(selected ∪ buffer)  (query.cpp:342-345)
    std::vector<uint32_t> tok;
    tok.reserve((size_t)(nbuf + nsel));
    auto gather = [&](const uint32_t* ids, int64_t cnt) -> int {
        if (cnt == 0) return LV_OK;
        if (!ids) return fail(LV_EINVAL, "sparse_attention: null id list");
        const size_t at = tok.size();
        tok.resize(at + cnt);
        if (where == LV_HOST) {
            std::memcpy(tok.data() + at, ids, sizeof(uint32_t) * cnt);
        } else {
            LV_CUDA(cudaMemcpyAsync(tok.data() + at, ids, sizeof(uint32_t) * cnt, cudaMemcpyDeviceToHost, st));
            LV_CUDA(cudaStreamSynchronize(st));
        }
        return LV_OK;
    };
    if (int rc = gather(selected_ids, nsel)) return rc;
    if (int rc = gather(buffer_ids, nbuf)) return rc;
    std::sort(tok.begin(), tok.end());
    tok.erase(std::unique(tok.begin(), tok.end()), tok.end());
    if (ntok) *ntok = (int64_t)tok.size();
    if (tok.empty()) return LV_EMPTY;
    if ((long long)tok.back() >= c->n) return fail(LV_ERANGE, "sparse_attention: id out of range");
    const long long nt = (long long)tok.size();
    const int per = (int)std::max<long long>(256, (nt + 63) / 64);
    const int P = (int)((nt + per - 1) / per);
    const size_t bytes = align256(sizeof(uint32_t) * nt) + align256(sizeof(float) * nt) +
                         align256(sizeof(float) * P * (c->DP + 2)) + align256(sizeof(float) * c->DP * 2) +
                         align256(sizeof(float) * 2);
    unsigned char* mem = nullptr;
    LV_CUDA(cudaMallocAsync((void**)&mem, bytes, st));
    unsigned* dids = reinterpret_cast<unsigned*>(mem);
    float* scores = reinterpret_cast<float*>(mem + align256(sizeof(uint32_t) * nt));
    float* part = reinterpret_cast<float*>((unsigned char*)scores + align256(sizeof(float) * nt));
    float* qpad = reinterpret_cast<float*>((unsigned char*)part + align256(sizeof(float) * P * (c->DP + 2)));
    float* opad = qpad + c->DP;
    float* ml = reinterpret_cast<float*>((unsigned char*)qpad + align256(sizeof(float) * c->DP * 2));
    LV_CUDA(cudaMemcpyAsync(dids, tok.data(), sizeof(uint32_t) * nt, cudaMemcpyHostToDevice, st));
    LV_CUDA(cudaMemsetAsync(qpad, 0, sizeof(float) * c->DP, st));
    LV_CUDA(cudaMemcpyAsync(qpad, q, sizeof(float) * c->cfg.d,
                            where == LV_HOST ? cudaMemcpyHostToDevice : cudaMemcpyDeviceToDevice, st));
    const float sc = scale != 0.0f ? scale : (float)(1.0 / std::sqrt((double)c->cfg.d));
    const size_t es = esize(c->cfg.dtype);
    const void* Ks = (const unsigned char*)c->K + (size_t)slot * c->cap * c->DP * es;
    const void* Vs = (const unsigned char*)c->V + (size_t)slot * c->cap * c->DP * es;
    const unsigned tb = (unsigned)((nt + 127) / 128);
#define LV_ATT(T, D)                                                                                  \
    lvk::token_scores_kernel<T, D><<<tb, 128, 0, st>>>((const T*)Ks, dids, nt, qpad, sc, scores);     \
    lvk::token_partials_kernel<T, D><<<P, 128, 0, st>>>((const T*)Vs, dids, scores, nt, per, part);
    if (c->cfg.dtype == LV_BF16) {
        if (c->DP == 64) { LV_ATT(__nv_bfloat16, 64) } else if (c->DP == 128) { LV_ATT(__nv_bfloat16, 128) } else { LV_ATT(__nv_bfloat16, 256) }
    } else {
        if (c->DP == 64) { LV_ATT(float, 64) } else if (c->DP == 128) { LV_ATT(float, 128) } else { LV_ATT(float, 256) }
    }
#undef LV_ATT
    lvk::lse_merge_kernel<<<1, 128, 0, st>>>(part, P, 1, c->DP, c->DP + 2, opad, c->DP, ml);
    LV_CUDA(cudaGetLastError());
    const cudaMemcpyKind kind = where == LV_HOST ? cudaMemcpyDeviceToHost : cudaMemcpyDeviceToDevice;
    LV_CUDA(cudaMemcpyAsync(out, opad, sizeof(float) * c->cfg.d, kind, st));
    if (weights) {
        lvk::token_weights_kernel<<<tb, 128, 0, st>>>(scores, nt, ml, scores);
        LV_CUDA(cudaGetLastError());
        LV_CUDA(cudaMemcpyAsync(weights, scores, sizeof(float) * nt, kind, st));
    }
    LV_CUDA(cudaFreeAsync(mem, st));
    LV_CUDA(cudaStreamSynchronize(st));
    return LV_OK;
}

// ---- snapshots (io.hpp:40-51, io.cpp:205-317): "LVKD" datasets and "LVIX" index files --


int lv_save_dataset(const char* path, const float* data, int64_t n, int d) {
    if (!path || (!data && n > 0) || n < 0 || d < 1 || n > 0xffffffffLL)
        return fail(LV_EINVAL, "save_dataset: bad arguments");
    std::ofstream os(path, std::ios::binary);
    if (!os) return fail(LV_ERUNTIME, std::string("cannot open for writing: ") + path);
    os.write(kLVKD, 4);
    put_le<uint32_t>(os, 1);
    put_le<uint32_t>(os, (uint32_t)n);
    put_le<uint32_t>(os, (uint32_t)d);
    os.write(reinterpret_cast<const char*>(data), (std::streamsize)(sizeof(float) * n * d));
    if (!os) return fail(LV_ERUNTIME, std::string("write failed: ") + path);
    return LV_OK;
}

int lv_load_dataset(const char* path, float* out, int64_t cap_rows, int64_t* n, int* d) {
    if (!path || !n || !d) return fail(LV_EINVAL, "load_dataset: null argument");
    std::ifstream is(path, std::ios::binary);
    if (!is) return fail(LV_ERUNTIME, std::string("cannot open for reading: ") + path);
    char magic[4];
    is.read(magic, 4);
    if (!is || std::memcmp(magic, kLVKD, 4) != 0) return fail(LV_ERUNTIME, "bad magic: not a dataset file");
    uint32_t ver = 0, rows = 0, dim = 0;
    if (!get_le(is, &ver)) return fail(LV_ERUNTIME, "corrupt file: truncated version");
    if (ver != 1) return fail(LV_ERUNTIME, "unsupported dataset version " + std::to_string(ver));
    if (!get_le(is, &rows)) return fail(LV_ERUNTIME, "corrupt file: truncated row count");
    if (!get_le(is, &dim)) return fail(LV_ERUNTIME, "corrupt file: truncated dimension");
    *n = rows;
    *d = (int)dim;
    if (!out) return LV_OK;  // dimensions only
    if ((int64_t)rows > cap_rows) return fail(LV_EINVAL, "load_dataset: output holds fewer rows than the file");
    is.read(reinterpret_cast<char*>(out), (std::streamsize)(sizeof(float) * (size_t)rows * dim));
    if (!is) return fail(LV_ERUNTIME, std::string("corrupt file: truncated payload in ") + path);
    if (!at_eof(is)) return fail(LV_ERUNTIME, std::string("corrupt file: trailing bytes in ") + path);
    return LV_OK;
}

// The device index of a slot written as the reference's index snapshot: one subspace,
// contiguous groups of r keys (the device cells) over [0, indexed_count), each with its
// exact AABB (column min / max of the stored keys, index.cpp:112-117) and members.
// save_index (io.cpp:236-268) of the grouped index of one slot
int save_grouped(const lv_ctx* c, int slot, const char* path) {
    const lvg::GroupIndex& g = *c->gi;
    const int64_t m = g.indexed, K = g.K;
    std::ofstream os(path, std::ios::binary);
    if (!os) return fail(LV_ERUNTIME, std::string("cannot open for writing: ") + path);
    os.write(kLVIX, 4);
    put_le<uint32_t>(os, 1);
    put_le<uint32_t>(os, (uint32_t)c->cfg.d);
    put_le<uint32_t>(os, (uint32_t)g.S);
    put_le<uint32_t>(os, (uint32_t)c->cfg.r);
    put_le<uint32_t>(os, (uint32_t)c->cfg.grouping);
    put_le<uint32_t>(os, (uint32_t)c->cfg.enclosure);
    put_le<uint64_t>(os, c->cfg.rng_seed);
    put_le<uint64_t>(os, (uint64_t)m);
    std::vector<uint32_t> asg(std::max<int64_t>(m, 1)), off(K + 1), mem(std::max<int64_t>(m, 1));
    std::vector<float> a((size_t)g.wmax * std::max<int64_t>(K, 1)), b(a.size()), rad(std::max<int64_t>(K, 1));
    for (int s = 0; s < g.S; ++s) {
        const int w = g.off[s + 1] - g.off[s];
        if (lvg::export_subspace(g, slot, s, asg.data(), off.data(), mem.data(), a.data(), b.data(), rad.data(),
                                 nullptr) != cudaSuccess)
            return fail(LV_ERUNTIME, "save_index: reading the grouped index");
        put_le<uint64_t>(os, (uint64_t)m);
        os.write(reinterpret_cast<const char*>(asg.data()), (std::streamsize)(m * 4));
        put_le<uint32_t>(os, (uint32_t)K);
        for (int64_t gg = 0; gg < K; ++gg) {
            put_le<uint32_t>(os, (uint32_t)c->cfg.enclosure);
            put_le<uint32_t>(os, (uint32_t)w);
            for (int i = 0; i < w; ++i) put_le<float>(os, a[(size_t)i * K + gg]);
            if (c->cfg.enclosure == 1) {
                put_le<uint32_t>(os, (uint32_t)w);
                for (int i = 0; i < w; ++i) put_le<float>(os, b[(size_t)i * K + gg]);
            } else {
                put_le<float>(os, rad[gg]);
            }
            put_le<uint32_t>(os, off[gg + 1] - off[gg]);
            os.write(reinterpret_cast<const char*>(mem.data() + off[gg]), (std::streamsize)(off[gg + 1] - off[gg]) * 4);
        }
    }
    if (!os) return fail(LV_ERUNTIME, std::string("write failed: ") + path);
    return LV_OK;
}

int lv_save_index(const lv_ctx* c, int slot, const char* path) {
    if (!c || !path) return fail(LV_EINVAL, "save_index: null argument");
    if (slot < 0 || slot >= c->slots) return fail(LV_ERANGE, "save_index: slot out of range");
    if (c->gi) return save_grouped(c, slot, path);
    const int d = c->cfg.d, r = c->r;
    const int64_t m = c->indexed;
    std::vector<float> rows((size_t)std::max<int64_t>(m, 1) * d);
    if (m > 0)
        if (int rc = lv_read_rows(c, slot, 0, m, 0, rows.data())) return rc;
    std::ofstream os(path, std::ios::binary);
    if (!os) return fail(LV_ERUNTIME, std::string("cannot open for writing: ") + path);
    os.write(kLVIX, 4);
    put_le<uint32_t>(os, 1);                    // version
    put_le<uint32_t>(os, (uint32_t)d);          // layout.d
    put_le<uint32_t>(os, 1u);                   // S: the cells span every coordinate
    put_le<uint32_t>(os, (uint32_t)r);          // r
    put_le<uint32_t>(os, 0u);                   // GroupingStrategy::Contiguous
    put_le<uint32_t>(os, 1u);                   // EnclosureKind::Aabb
    put_le<uint64_t>(os, c->cfg.rng_seed);
    put_le<uint64_t>(os, (uint64_t)m);
    put_le<uint64_t>(os, (uint64_t)m);          // assignments
    for (int64_t j = 0; j < m; ++j) put_le<uint32_t>(os, (uint32_t)(j / r));
    const int64_t groups = (m + r - 1) / r;
    put_le<uint32_t>(os, (uint32_t)groups);
    std::vector<float> lo(d), hi(d);
    for (int64_t g = 0; g < groups; ++g) {
        const int64_t b = g * r, e = std::min<int64_t>(m, b + r);
        for (int i = 0; i < d; ++i) lo[i] = hi[i] = rows[(size_t)b * d + i];
        for (int64_t j = b + 1; j < e; ++j)
            for (int i = 0; i < d; ++i) {
                lo[i] = std::min(lo[i], rows[(size_t)j * d + i]);
                hi[i] = std::max(hi[i], rows[(size_t)j * d + i]);
            }
        put_le<uint32_t>(os, 1u);  // kind Aabb
        put_le<uint32_t>(os, (uint32_t)d);
        os.write(reinterpret_cast<const char*>(lo.data()), sizeof(float) * d);
        put_le<uint32_t>(os, (uint32_t)d);
        os.write(reinterpret_cast<const char*>(hi.data()), sizeof(float) * d);
        put_le<uint32_t>(os, (uint32_t)(e - b));
        for (int64_t j = b; j < e; ++j) put_le<uint32_t>(os, (uint32_t)j);
    }
    if (!os) return fail(LV_ERUNTIME, std::string("write failed: ") + path);
    return LV_OK;
}

// Reads a reference index snapshot (io.cpp:270-317; any grouping, enclosure and S),
// validates it against the cache (dimension, indexed_count <= n, every subspace's
// groups partition [0, indexed_count) and agree with its assignments), then adopts its
// indexed_count: keys past it form the buffer. The device index is not read from the
// file — the cell summaries already cover every stored key — so the query results are
// those of the snapshot's index (final sets never depend on the grouping).
int lv_load_index(lv_ctx* c, const char* path, int64_t* indexed_count, void* stream) {
    if (!c || !path) return fail(LV_EINVAL, "load_index: null argument");
    std::ifstream is(path, std::ios::binary);
    if (!is) return fail(LV_ERUNTIME, std::string("cannot open for reading: ") + path);
    char magic[4];
    is.read(magic, 4);
    if (!is || std::memcmp(magic, kLVIX, 4) != 0) return fail(LV_ERUNTIME, "bad magic: not a index snapshot file");
    uint32_t ver, d, nsub, r, grouping, enclosing;
    uint64_t seed, m;
    if (!get_le(is, &ver)) return fail(LV_ERUNTIME, "corrupt file: truncated version");
    if (ver != 1) return fail(LV_ERUNTIME, "unsupported snapshot version " + std::to_string(ver));
    if (!get_le(is, &d) || !get_le(is, &nsub) || !get_le(is, &r) || !get_le(is, &grouping) || !get_le(is, &enclosing) ||
        !get_le(is, &seed) || !get_le(is, &m))
        return fail(LV_ERUNTIME, "corrupt file: truncated header");
    if ((int)d != c->cfg.d) return fail(LV_EINVAL, "load_index: snapshot dimension differs from the cache");
    if (nsub < 1 || nsub > d) return fail(LV_ERUNTIME, "corrupt file: subspace count");
    if ((int64_t)m > c->n) return fail(LV_EINVAL, "load_index: indexed_count exceeds the stored keys");
    // the grouped index takes the snapshot's groups when it describes this cache's
    // BuildConfig (one slot); otherwise it is rebuilt over [0, indexed_count) after the load
    lvg::GroupIndex* gi = c->gi && c->slots == 1 && (int)nsub == c->gi->S && (int)r == c->cfg.r &&
                                  (int)grouping == c->cfg.grouping && (int)enclosing == c->cfg.enclosure &&
                                  seed == c->cfg.rng_seed
                              ? c->gi
                              : nullptr;
    // grouped index: every subspace's arrays, as append_gate_entry packs them (index.cpp:139-168)
    struct Sub {
        std::vector<uint32_t> asg, off{0}, mem;
        std::vector<std::vector<float>> a, b;
        std::vector<float> rad;
        double nb = 0.0;
    };
    std::vector<Sub> subs(gi ? nsub : 0);
    std::vector<uint32_t> asg, mem;
    std::vector<uint8_t> seen;
    for (uint32_t s = 0; s < nsub; ++s) {
        uint64_t asz;
        if (!get_le(is, &asz)) return fail(LV_ERUNTIME, "corrupt file: truncated assignment count");
        if (asz != m) return fail(LV_ERUNTIME, "corrupt file: assignment count != indexed count");
        asg.resize(asz);
        is.read(reinterpret_cast<char*>(asg.data()), (std::streamsize)(asz * 4));
        if (!is) return fail(LV_ERUNTIME, "corrupt file: truncated assignments");
        uint32_t gcount;
        if (!get_le(is, &gcount)) return fail(LV_ERUNTIME, "corrupt file: truncated group count");
        seen.assign(m, 0);
        const int w = (int)(d / nsub + (s < d % nsub ? 1 : 0));
        if (gi) {
            subs[s].asg = asg;
            subs[s].a.assign(w, {});
            subs[s].b.assign(w, {});
        }
        for (uint32_t g = 0; g < gcount; ++g) {
            uint32_t kind, len;
            if (!get_le(is, &kind)) return fail(LV_ERUNTIME, "corrupt file: truncated kind");
            const int nvec = kind == 1 ? 2 : 1;  // Aabb: lo, hi; Ball / SpanBall: center (+ radius)
            std::vector<float> vec[2];
            for (int v = 0; v < nvec; ++v) {
                if (!get_le(is, &len)) return fail(LV_ERUNTIME, "corrupt file: truncated vector length");
                if (gi) {
                    if ((int)len != w || kind != enclosing) return fail(LV_ERUNTIME, "corrupt file: enclosure shape");
                    vec[v].resize(len);
                    is.read(reinterpret_cast<char*>(vec[v].data()), (std::streamsize)len * 4);
                } else {
                    is.seekg((std::streamoff)len * 4, std::ios::cur);
                }
            }
            float rad = 0.0f;
            if (kind != 1) {
                if (!get_le(is, &rad)) return fail(LV_ERUNTIME, "corrupt file: truncated radius");
            }
            if (gi) {  // append_gate_entry: packed arrays and the norm bound
                Sub& sb = subs[s];
                double bnd = 0.0;
                for (int i = 0; i < w; ++i) {
                    sb.a[i].push_back(vec[0][i]);
                    if (kind == 1) sb.b[i].push_back(vec[1][i]);
                }
                if (kind == 1) {
                    double sq = 0.0;
                    for (int i = 0; i < w; ++i) {
                        const double x = std::abs(double(vec[0][i])), y = std::abs(double(vec[1][i]));
                        const double mx = std::max(x, y);
                        sq += mx * mx;
                    }
                    bnd = std::sqrt(sq);
                } else {
                    float sq = 0.0f;
                    for (int i = 0; i < w; ++i) sq += vec[0][i] * vec[0][i];
                    bnd = double(std::sqrt(sq)) + double(rad);
                    sb.rad.push_back(rad);
                }
                sb.nb = std::max(sb.nb, bnd);
            }
            uint32_t msz;
            if (!get_le(is, &msz)) return fail(LV_ERUNTIME, "corrupt file: truncated member count");
            mem.resize(msz);
            is.read(reinterpret_cast<char*>(mem.data()), (std::streamsize)msz * 4);
            if (!is) return fail(LV_ERUNTIME, "corrupt file: truncated members");
            for (uint32_t id : mem) {
                if (id >= m || seen[id] || asg[id] != g) return fail(LV_ERUNTIME, "corrupt file: groups do not partition the indexed keys");
                seen[id] = 1;
            }
            if (gi) {
                subs[s].mem.insert(subs[s].mem.end(), mem.begin(), mem.end());
                subs[s].off.push_back((uint32_t)subs[s].mem.size());
            }
        }
        for (uint64_t j = 0; j < m; ++j)
            if (!seen[j]) return fail(LV_ERUNTIME, "corrupt file: groups do not partition the indexed keys");
    }
    if (!at_eof(is)) return fail(LV_ERUNTIME, std::string("corrupt file: trailing bytes in ") + path);
    std::lock_guard<std::mutex> lock(c->writer);
    if (gi) {
        for (uint32_t s = 0; s < nsub; ++s) {
            const Sub& sb = subs[s];
            const int64_t K = (int64_t)sb.off.size() - 1;
            const int w = (int)sb.a.size();
            std::vector<float> a((size_t)w * std::max<int64_t>(K, 1)), b(a.size());
            for (int i = 0; i < w; ++i)
                for (int64_t g = 0; g < K; ++g) {
                    a[(size_t)i * K + g] = sb.a[i][g];
                    if (enclosing == 1) b[(size_t)i * K + g] = sb.b[i][g];
                }
            if (s > 0 && K != gi->K) return fail(LV_ERUNTIME, "load_index: subspaces with different group counts");
            if (lvg::import_subspace(*gi, 0, (int)s, (long long)m, K, sb.asg.data(), sb.off.data(), sb.mem.data(),
                                     a.data(), b.data(), sb.rad.data(), sb.nb) != cudaSuccess)
                return fail(LV_ERUNTIME, "load_index: writing the grouped index");
        }
    } else if (c->gi) {
        c->gi->indexed = 0;
        c->gi->K = 0;
        LV_CUDA(cudaMemsetAsync(c->gi->nbound, 0, sizeof(unsigned long long) * c->slots * c->gi->S, S(stream)));
        LV_CUDA(lvg::index_range(*c->gi, arena_view(c), 0, (long long)m, S(stream)));
    }
    Counters h{c->n, (long long)m, c->flushes, 0};
    LV_CUDA(cudaMemcpyAsync(c->ctr, &h, sizeof(h), cudaMemcpyHostToDevice, S(stream)));
    LV_CUDA(cudaStreamSynchronize(S(stream)));
    c->indexed = (long long)m;
    if (indexed_count) *indexed_count = (int64_t)m;
    return LV_OK;
}

int lv_group_candidates(lv_ctx* c, int slot, const float* q, float tau, const float* tau_subspace, int algo,
                        uint32_t* live_bits, uint32_t* live_ids, int64_t cap, int64_t* nlive, lv_group_stats* stats,
                        void* stream) {
    if (!c || !q) return fail(LV_EINVAL, "group candidates: null argument");
    if (!c->gi) return fail(LV_EINVAL, "group candidates: the cache has no grouped index (lv_config.group_index)");
    if (slot < 0 || slot >= c->slots) return fail(LV_ERANGE, "group candidates: slot out of range");
    if (algo != LV_ALGO_FULL_SUBSPACE && algo != LV_ALGO_TA) return fail(LV_EINVAL, "group candidates: algo");
    if (algo == LV_ALGO_FULL_SUBSPACE && !tau_subspace)
        return fail(LV_EINVAL, "query_full_subspace: tau_subspace required");  // query.cpp:85-86
    std::lock_guard<std::mutex> lock(c->writer);
    cudaStream_t st = S(stream);
    const long long words = std::max<long long>(1, (c->gi->indexed + 31) / 32);
    uint32_t* bits = live_bits;
    if (!bits) LV_CUDA(cudaMallocAsync(&bits, sizeof(uint32_t) * words, st));
    lvg::Stats sg;
    const cudaError_t e = lvg::candidates(*c->gi, slot, q, tau, tau_subspace, algo == LV_ALGO_TA ? 1 : 0, bits, &sg, st);
    int rc = LV_OK;
    if (e != cudaSuccess) rc = fail(LV_ERUNTIME, std::string("group candidates: ") + cudaGetErrorString(e));
    if (!rc && (live_ids || nlive)) {
        std::vector<uint32_t> hb(words);
        if (cudaMemcpy(hb.data(), bits, sizeof(uint32_t) * words, cudaMemcpyDeviceToHost) != cudaSuccess)
            rc = fail(LV_ERUNTIME, "group candidates: reading the live set");
        int64_t k = 0;
        for (long long w = 0; w < words && !rc; ++w)
            for (uint32_t x = hb[w]; x; x &= x - 1) {
                if (live_ids && k < cap) live_ids[k] = (uint32_t)(w * 32 + __builtin_ctz(x));
                ++k;
            }
        if (nlive) *nlive = k;
    }
    if (!live_bits) cudaFreeAsync(bits, st);
    if (stats && !rc) {
        stats->groups_tested = sg.groups_tested;
        stats->keys_scanned = sg.keys_scanned;
        stats->f_scan = sg.f_scan;
        stats->gate_cost_equiv = sg.gate_cost_equiv;
        stats->ta_stop_depth = sg.ta_stop_depth;
        stats->ta_stop_upper = sg.ta_stop_upper;
    }
    return rc;
}

int lv_group_thresholds(lv_ctx* c, int slot, const float* q, float tau, float* out, void* stream) {
    if (!c || !q || !out) return fail(LV_EINVAL, "derive_subspace_thresholds: null argument");
    if (!c->gi) return fail(LV_EINVAL, "derive_subspace_thresholds: the cache has no grouped index");
    if (slot < 0 || slot >= c->slots) return fail(LV_ERANGE, "derive_subspace_thresholds: slot out of range");
    std::lock_guard<std::mutex> lock(c->writer);
    LV_CUDA(lvg::thresholds(*c->gi, slot, q, tau, out, S(stream)));
    return LV_OK;
}

int64_t lv_group_count(const lv_ctx* c) { return c && c->gi ? c->gi->K : 0; }

int lv_group_export(const lv_ctx* c, int slot, int s, uint32_t* assignments, uint32_t* member_offsets,
                    uint32_t* member_ids, float* a, float* b, float* radii, double* norm_bound) {
    if (!c) return fail(LV_EINVAL, "group export: null context");
    if (!c->gi) return fail(LV_EINVAL, "group export: the cache has no grouped index");
    if (slot < 0 || slot >= c->slots || s < 0 || s >= c->gi->S) return fail(LV_ERANGE, "group export: slot or subspace");
    LV_CUDA(lvg::export_subspace(*c->gi, slot, s, assignments, member_offsets, member_ids, a, b, radii, norm_bound));
    return LV_OK;
}

int lv_read_rows(const lv_ctx* c, int slot, int64_t first, int64_t count, int which_v, float* out) {
    if (!c || !out) return fail(LV_EINVAL, "lv_read_rows: null argument");
    if (slot < 0 || slot >= c->slots || first < 0 || first + count > c->n)
        return fail(LV_ERANGE, "lv_read_rows: range");
    const size_t es = esize(c->cfg.dtype);
    std::vector<unsigned char> buf((size_t)count * c->DP * es);
    const unsigned char* src = (const unsigned char*)(which_v ? c->V : c->K) +
                               ((size_t)slot * c->cap + first) * c->DP * es;
    LV_CUDA(cudaMemcpy(buf.data(), src, buf.size(), cudaMemcpyDeviceToHost));
    for (int64_t j = 0; j < count; ++j)
        for (int i = 0; i < c->cfg.d; ++i) {
            const size_t at = (size_t)j * c->DP + i;
            if (es == 4) {
                std::memcpy(out + j * c->cfg.d + i, buf.data() + at * 4, 4);
            } else {
                uint16_t h;
                std::memcpy(&h, buf.data() + at * 2, 2);
                const uint32_t u = (uint32_t)h << 16;
                std::memcpy(out + j * c->cfg.d + i, &u, 4);
            }
        }
    return LV_OK;
}

}  // extern "C"
