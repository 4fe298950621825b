// Microbenchmark: per-SM issue rate of 4 KB block copies into shared memory on B200,
// one issuing thread per CTA (the loader-warp pattern), a 32-stage ring, 148 CTAs.
//   box128   2 TMA 2D boxes of 64 bf16 x 16 rows (128-byte rows, 128-byte swizzle)
//   box256   1 TMA 2D box of 128 bf16 x 16 rows (256-byte rows, no swizzle)
//   bulk     1 cp.async.bulk of 4 KB
// Working set: L2-resident (16 MB) and HBM (1 GB). Prints ns per 4 KB block per SM.
#include <cuda.h>
#include <cudaTypedefs.h>
#include <cuda_runtime.h>
#include <cstdio>

__device__ __forceinline__ unsigned su32(const void* p) { return (unsigned)__cvta_generic_to_shared(p); }

template <int MODE>
__global__ void issue_blocks(const __grid_constant__ CUtensorMap m128, const __grid_constant__ CUtensorMap m256,
                             const unsigned char* src, long long nblk_src, int per_cta, unsigned* sink) {
    extern __shared__ __align__(1024) unsigned char sm[];
    constexpr int S = 8;  // stages per issuing warp
    const int w = threadIdx.x >> 5;
    const unsigned base = ((su32(sm) + 1023) & ~1023u) + w * (S * 4096 + 1024);
    const unsigned bar = base + S * 4096;
    if ((threadIdx.x & 31) != 0) return;
    for (int s = 0; s < S; ++s) asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(bar + 8 * s));
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    unsigned h = (blockIdx.x * 64 + w) * 2654435761u;
    for (int i = 0; i < per_cta; ++i) {
        const int s = i % S;
        if (i >= S) {
            const unsigned par = ((i / S) - 1) & 1;
            asm volatile("{ .reg .pred p; W: mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1; @!p bra W; }" ::"r"(bar + 8 * s), "r"(par) : "memory");
        }
        h = h * 1664525u + 1013904223u;
        const long long blk = (long long)(h % (unsigned)nblk_src);
        const unsigned dst = base + s * 4096;
        asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], 4096;" ::"r"(bar + 8 * s) : "memory");
        if (MODE == 0) {
            for (int pan = 0; pan < 2; ++pan)
                asm volatile("cp.async.bulk.tensor.2d.shared::cluster.global.tile.mbarrier::complete_tx::bytes [%0], [%1, {%2, %3}], [%4];"
                             ::"r"(dst + pan * 2048), "l"((unsigned long long)&m128), "r"(pan * 64), "r"((int)(blk * 16)), "r"(bar + 8 * s) : "memory");
        } else if (MODE == 1) {
            asm volatile("cp.async.bulk.tensor.2d.shared::cluster.global.tile.mbarrier::complete_tx::bytes [%0], [%1, {%2, %3}], [%4];"
                         ::"r"(dst), "l"((unsigned long long)&m256), "r"(0), "r"((int)(blk * 16)), "r"(bar + 8 * s) : "memory");
        } else {
            asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], 4096, [%2];"
                         ::"r"(dst), "l"(src + blk * 4096), "r"(bar + 8 * s) : "memory");
        }
    }
    for (int i = per_cta; i < per_cta + S; ++i) {  // drain
        const int s = i % S;
        const unsigned par = ((i / S) - 1) & 1;
        if (i - S >= 0)
            asm volatile("{ .reg .pred p; W: mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1; @!p bra W; }" ::"r"(bar + 8 * s), "r"(par) : "memory");
    }
    if (h == 0x12345u) sink[0] = h;
}

int main() {
    const long long bytes = 1LL << 30;
    unsigned char* src;
    unsigned* sink;
    cudaMalloc(&src, bytes);
    cudaMalloc(&sink, 4);
    cudaMemset(src, 1, bytes);
    PFN_cuTensorMapEncodeTiled_v12000 encode;
    cudaDriverEntryPointQueryResult q;
    cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", (void**)&encode, cudaEnableDefault, &q);
    CUtensorMap m128, m256;
    const cuuint64_t dims[2] = {128, (cuuint64_t)(bytes / 256)};
    const cuuint64_t strides[1] = {256};
    const cuuint32_t b128[2] = {64, 16}, b256[2] = {128, 16}, es[2] = {1, 1};
    encode(&m128, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 2, src, dims, strides, b128, es, CU_TENSOR_MAP_INTERLEAVE_NONE,
           CU_TENSOR_MAP_SWIZZLE_128B, CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
    encode(&m256, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 2, src, dims, strides, b256, es, CU_TENSOR_MAP_INTERLEAVE_NONE,
           CU_TENSOR_MAP_SWIZZLE_NONE, CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
    cudaEvent_t a, b;
    cudaEventCreate(&a);
    cudaEventCreate(&b);
    const char* names[3] = {"box128x2", "box256", "bulk4K"};
    auto run = [&](auto kern, int mode, long long ws, int W) {
        const int smem = W * (8 * 4096 + 1024) + 1024;
        cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
        const int per = 512 / W;
        float best = 1e9f;
        for (int it = 0; it < 5; ++it) {
            cudaEventRecord(a);
            kern<<<148, 32 * W, smem>>>(m128, m256, src, ws / 4096, per, sink);
            cudaEventRecord(b);
            cudaEventSynchronize(b);
            float ms;
            cudaEventElapsedTime(&ms, a, b);
            if (ms < best) best = ms;
        }
        printf("%-9s W=%2d ws %5lld MB: %7.1f us total, %6.1f ns per 4 KB per SM, %6.0f GB/s\n", names[mode], W, ws >> 20,
               best * 1e3, best * 1e6 / (per * W), 148.0 * per * W * 4096 / (best * 1e-3) / 1e9);
    };
    for (long long ws : {16LL << 20, 1LL << 30})
        for (int W : {1, 2, 4, 8, 16}) {
            run(issue_blocks<0>, 0, ws, W);
            run(issue_blocks<2>, 2, ws, W);
        }
    printf("status %s\n", cudaGetErrorString(cudaDeviceSynchronize()));
    return 0;
}
