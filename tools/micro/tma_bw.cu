// Microbenchmark: how fast can W warps per SM stream 8 KB tiles (16 rows x 512 B, the
// probe's summary tile) through a D-deep shared-memory ring on B200?
//   tma    4 TMA 2D boxes (64 bf16 x 16 rows, 128-byte swizzle) per tile, mbarrier
//   bulk   one cp.async.bulk of 8 KB per tile, mbarrier
//   cpa    cp.async 16 B per lane (16 per lane per tile), commit/wait_group
// Each warp walks tiles w, w + W*148, ...; reports GB/s for a short burst (32 MB, like one
// layer's summaries) and a long one (256 MB), cold L2 (a 512 MB read in between).
#include <cuda.h>
#include <cudaTypedefs.h>
#include <cuda_runtime.h>
#include <cstdio>

__device__ __forceinline__ unsigned su32(const void* p) { return (unsigned)__cvta_generic_to_shared(p); }
__device__ __forceinline__ void mbar_wait(unsigned bar, unsigned par) {
    asm volatile("{ .reg .pred p; W: mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1; @!p bra W; }" ::"r"(bar), "r"(par) : "memory");
}

template <int MODE, int D>
__global__ void stream_tiles(const __grid_constant__ CUtensorMap map, const unsigned char* src, long long ntiles,
                             unsigned* sink) {
    extern __shared__ __align__(1024) unsigned char sm[];
    const int lane = threadIdx.x & 31, w = threadIdx.x >> 5, W = blockDim.x >> 5;
    const unsigned base = (su32(sm) + 1023) & ~1023u;
    const unsigned ring = base + w * D * 8192;
    const unsigned bar = base + W * D * 8192 + w * D * 8;
    const long long gw = (long long)blockIdx.x * W + w, stride = (long long)gridDim.x * W;
    if (lane == 0)
        for (int s = 0; s < D; ++s) asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(bar + 8 * s));
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    __syncwarp();
    auto issue = [&](long long i) {
        const long long t = gw + i * stride;
        const int s = (int)(i % D);
        if (MODE == 2) {
            if (t < ntiles) {
                const unsigned char* g = src + t * 8192 + lane * 16;
#pragma unroll
                for (int k = 0; k < 16; ++k)
                    asm volatile("cp.async.cg.shared.global [%0], [%1], 16;" ::"r"(ring + s * 8192 + k * 512 + lane * 16), "l"(g + k * 512) : "memory");
            }
            asm volatile("cp.async.commit_group;" ::: "memory");
            return;
        }
        if (t >= ntiles || lane != 0) return;
        asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
        asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], 8192;" ::"r"(bar + 8 * s) : "memory");
        if (MODE == 0) {
            for (int pan = 0; pan < 4; ++pan)
                asm volatile("cp.async.bulk.tensor.2d.shared::cluster.global.tile.mbarrier::complete_tx::bytes [%0], [%1, {%2, %3}], [%4];"
                             ::"r"(ring + s * 8192 + pan * 2048), "l"((unsigned long long)&map), "r"(pan * 64), "r"((int)(t * 16)), "r"(bar + 8 * s) : "memory");
        } else {
            asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], 8192, [%2];"
                         ::"r"(ring + s * 8192), "l"(src + t * 8192), "r"(bar + 8 * s) : "memory");
        }
    };
    unsigned acc = 0;
    for (int i = 0; i < D; ++i) issue(i);
    for (long long i = 0;; ++i) {
        const long long t = gw + i * stride;
        if (t >= ntiles) break;
        const int s = (int)(i % D);
        if (MODE == 2) {
            asm volatile("cp.async.wait_group %0;" ::"n"(D - 1) : "memory");
        } else {
            mbar_wait(bar + 8 * s, (unsigned)((i / D) & 1));
        }
        __syncwarp();
        unsigned v;
        asm volatile("ld.shared.u32 %0, [%1];" : "=r"(v) : "r"(ring + s * 8192 + lane * 256) : "memory");
        acc += v;
        __syncwarp();
        issue(i + D);
    }
    if (MODE == 2) asm volatile("cp.async.wait_group 0;" ::: "memory");
    if (acc == 0x12345678) sink[0] = acc;
}

int main() {
    const long long bytes = 1LL << 30;
    unsigned char *src, *junk;
    unsigned* sink;
    cudaMalloc(&src, bytes);
    cudaMalloc(&junk, 512 << 20);
    cudaMalloc(&sink, 4);
    cudaMemset(src, 1, bytes);
    cudaMemset(junk, 1, 512 << 20);
    cudaDeviceSynchronize();
    PFN_cuTensorMapEncodeTiled_v12000 encode;
    cudaDriverEntryPointQueryResult q;
    cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", (void**)&encode, cudaEnableDefault, &q);
    CUtensorMap map;
    const cuuint64_t dims[2] = {256, (cuuint64_t)(bytes / 512)};
    const cuuint64_t strides[1] = {512};
    const cuuint32_t box[2] = {64, 16}, es[2] = {1, 1};
    encode(&map, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 2, src, dims, strides, box, es, CU_TENSOR_MAP_INTERLEAVE_NONE,
           CU_TENSOR_MAP_SWIZZLE_128B, CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
    cudaEvent_t a, b;
    cudaEventCreate(&a);
    cudaEventCreate(&b);
    auto flush = [&] {  // read 512 MB: clean L2
        cudaMemsetAsync(sink, 0, 4);
        // a read-only pass: reuse stream_tiles in bulk mode over the junk buffer is overkill; memcpy DtoD reads+writes,
        // so read through a trivial kernel instead
    };
    (void)flush;
    const char* names[3] = {"tma4box", "bulk8K", "cpasync"};
    auto run = [&](auto kern, int mode, int W, int D, long long mb) {
        const int smem = W * D * 8192 + W * D * 8 + 1024;
        cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
        const long long ntiles = (mb << 20) / 8192;
        float best = 1e9f;
        for (int it = 0; it < 5; ++it) {
            // cold-ish L2: stream a different 512 MB window of src first
            kern<<<148, W * 32, smem>>>(map, src + (512LL << 20), (256LL << 20) / 8192, sink);
            cudaEventRecord(a);
            kern<<<148, W * 32, smem>>>(map, src, ntiles, sink);
            cudaEventRecord(b);
            cudaEventSynchronize(b);
            float ms;
            cudaEventElapsedTime(&ms, a, b);
            if (ms < best) best = ms;
        }
        printf("%-8s W=%2d D=%d %4lld MB: %7.2f us  %7.1f GB/s\n", names[mode], W, D, mb, best * 1e3,
               (double)(ntiles * 8192) / (best * 1e-3) / 1e9);
    };
    {  // event overhead: an empty launch
        float best = 1e9f;
        for (int it = 0; it < 10; ++it) {
            cudaEventRecord(a);
            stream_tiles<1, 3><<<148, 256, 8 * 3 * 8192 + 1024 + 8 * 3 * 8>>>(map, src, 0, sink);
            cudaEventRecord(b);
            cudaEventSynchronize(b);
            float ms;
            cudaEventElapsedTime(&ms, a, b);
            if (ms < best) best = ms;
        }
        printf("empty launch: %.2f us\n", best * 1e3);
    }
    for (long long mb : {8LL, 16LL, 32LL, 64LL, 128LL, 256LL}) run(stream_tiles<1, 3>, 1, 8, 3, mb);
    for (long long mb : {8LL, 16LL, 32LL, 64LL, 128LL, 256LL}) run(stream_tiles<2, 3>, 2, 8, 3, mb);
    printf("status %s\n", cudaGetErrorString(cudaDeviceSynchronize()));
    return 0;
}
