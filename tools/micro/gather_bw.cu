// Microbenchmark: gather bandwidth of 4 KB blocks (16 rows x 256 B, i.e. one
// surviving cell of bf16 keys) from a 2 GiB array at pseudo-random block
// positions, on B200. Variants:
//   ldg<D>   each warp owns blocks; D blocks' LDG.128 loads in flight per warp
//   bulk<S>  one elected lane issues cp.async.bulk of whole 4 KB blocks into an
//            S-deep shared-memory ring per warp (mbarrier completion)
// Prints GB/s for each variant and occupancy.
#include <cstdio>
#include <cstdint>
#include <cuda_runtime.h>

__device__ __forceinline__ uint4 ldg16(const void* p) {
    uint4 r;
    asm volatile("ld.global.nc.L1::no_allocate.v4.u32 {%0,%1,%2,%3}, [%4];" : "=r"(r.x), "=r"(r.y), "=r"(r.z), "=r"(r.w) : "l"(p));
    return r;
}
__device__ __forceinline__ unsigned hashu(unsigned x) { x ^= x >> 16; x *= 0x7feb352d; x ^= x >> 15; x *= 0x846ca68b; x ^= x >> 16; return x; }

template <int D>
__global__ void __launch_bounds__(256) gather_ldg(const uint4* __restrict__ src, long long nblocks, int per_warp, unsigned* sink) {
    const int lane = threadIdx.x & 31;
    const long long warp = (blockIdx.x * (long long)blockDim.x + threadIdx.x) >> 5;
    unsigned acc = 0;
    for (int i = 0; i < per_warp; i += D) {
        uint4 v[D][8];
#pragma unroll
        for (int d = 0; d < D; ++d) {
            const long long b = hashu((unsigned)(warp * per_warp + i + d)) % nblocks;
            const uint4* p = src + b * 256;  // 4 KB = 256 uint4
#pragma unroll
            for (int k = 0; k < 8; ++k) v[d][k] = ldg16(p + k * 32 + lane);
        }
#pragma unroll
        for (int d = 0; d < D; ++d)
#pragma unroll
            for (int k = 0; k < 8; ++k) acc += v[d][k].x ^ v[d][k].w;
    }
    if (acc == 0x12345678) sink[0] = acc;
}

__device__ __forceinline__ unsigned smem_u32(const void* p) { return static_cast<unsigned>(__cvta_generic_to_shared(p)); }

template <int S>
__global__ void __launch_bounds__(128) gather_bulk(const unsigned char* __restrict__ src, long long nblocks, int per_warp, unsigned* sink) {
    extern __shared__ __align__(128) unsigned char sm[];
    const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
    unsigned char* ring = sm + w * S * 4096;
    unsigned long long* bar = reinterpret_cast<unsigned long long*>(sm + 4 * S * 4096) + w * S;
    const long long warp = (blockIdx.x * (long long)blockDim.x + threadIdx.x) >> 5;
    if (lane == 0)
        for (int s = 0; s < S; ++s) asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" :: "r"(smem_u32(bar + s)));
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    __syncwarp();
    auto issue = [&](int i) {
        const int s = i % S;
        const long long b = hashu((unsigned)(warp * per_warp + i)) % nblocks;
        asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], 4096;" :: "r"(smem_u32(bar + s)) : "memory");
        asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], 4096, [%2];"
                     :: "r"(smem_u32(ring + s * 4096)), "l"(src + b * 4096), "r"(smem_u32(bar + s)) : "memory");
    };
    unsigned acc = 0;
    if (lane == 0) for (int i = 0; i < S && i < per_warp; ++i) issue(i);
    for (int i = 0; i < per_warp; ++i) {
        const int s = i % S;
        const unsigned par = (i / S) & 1;
        asm volatile("{ .reg .pred p; W: mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1; @!p bra W; }" :: "r"(smem_u32(bar + s)), "r"(par) : "memory");
        acc += reinterpret_cast<const unsigned*>(ring + s * 4096)[lane * 32];
        __syncwarp();
        if (lane == 0 && i + S < per_warp) {
            asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
            issue(i + S);
        }
    }
    if (acc == 0x12345678) sink[0] = acc;
}

int main() {
    const long long bytes = 2LL << 30;
    const long long nblocks = bytes / 4096;
    unsigned char* src;
    unsigned* sink;
    cudaMalloc(&src, bytes);
    cudaMalloc(&sink, 4);
    cudaMemset(src, 1, bytes);
    cudaEvent_t a, b;
    cudaEventCreate(&a);
    cudaEventCreate(&b);
    const long long total_blocks = 65536;  // 256 MiB gathered per launch
    auto run = [&](const char* name, auto launch) {
        for (int it = 0; it < 3; ++it) launch();
        cudaEventRecord(a);
        for (int it = 0; it < 10; ++it) launch();
        cudaEventRecord(b);
        cudaEventSynchronize(b);
        float ms;
        cudaEventElapsedTime(&ms, a, b);
        printf("%-28s %8.1f GB/s  (%.2f us per 256 MiB)\n", name, total_blocks * 4096.0 * 10 / (ms * 1e-3) / 1e9, ms * 100);
    };
#define LDG(D, WARPS)                                                                           \
    {                                                                                          \
        const int warps = WARPS;                                                               \
        const int per = (int)(total_blocks / warps);                                           \
        char nm[64];                                                                           \
        snprintf(nm, 64, "ldg D=%d warps=%d", D, warps);                                      \
        run(nm, [&] { gather_ldg<D><<<warps / 8, 256>>>((const uint4*)src, nblocks, per, sink); }); \
    }
    LDG(1, 148 * 16) LDG(2, 148 * 16) LDG(4, 148 * 16) LDG(1, 148 * 32) LDG(2, 148 * 32) LDG(1, 148 * 64)
    LDG(4, 148 * 8) LDG(2, 148 * 24)
#define BULK(S, CTAS)                                                                           \
    {                                                                                          \
        const int warps = CTAS * 4;                                                            \
        const int per = (int)(total_blocks / warps);                                           \
        const int smem = 4 * S * 4096 + 4 * S * 8;                                             \
        cudaFuncSetAttribute(gather_bulk<S>, cudaFuncAttributeMaxDynamicSharedMemorySize, smem); \
        char nm[64];                                                                           \
        snprintf(nm, 64, "bulk S=%d ctas=%d", S, CTAS);                                       \
        run(nm, [&] { gather_bulk<S><<<CTAS, 128, smem>>>(src, nblocks, per, sink); });         \
    }
    BULK(2, 148 * 2) BULK(4, 148) BULK(4, 148 * 2) BULK(8, 148) BULK(3, 148 * 4) BULK(12, 148)
    cudaError_t e = cudaDeviceSynchronize();
    printf("status %s\n", cudaGetErrorString(e));
    return 0;
}
