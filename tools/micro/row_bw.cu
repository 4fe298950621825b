// Microbenchmark: gather bandwidth of random rows of R bytes (256 B = one bf16 V row at
// d = 128; 4096 B = one 16-key block) with cp.async 16 B per lane into a per-warp ring,
// 16 warps per SM x 148 SMs, 256 MB gathered from a 2 GB array. Also a 25/75 mix of
// 256 B rows and 4 KB blocks (the attend phase's V:K byte ratio).
#include <cuda_runtime.h>
#include <cstdio>

__device__ __forceinline__ unsigned hashu(unsigned x) { x ^= x >> 16; x *= 0x7feb352d; x ^= x >> 15; x *= 0x846ca68b; x ^= x >> 16; return x; }

template <int RB, int D>
__global__ void __launch_bounds__(512) gather_rows(const unsigned char* __restrict__ src, long long nrows, long long per_warp, unsigned* sink) {
    extern __shared__ __align__(16) unsigned char sm[];
    const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
    const long long gw = (blockIdx.x * (long long)blockDim.x + threadIdx.x) >> 5;
    constexpr int CH = RB / 16;                  // 16-byte chunks per row
    constexpr int RPI = CH >= 32 ? 1 : 32 / CH;  // rows per warp instruction
    constexpr int IPR = CH >= 32 ? CH / 32 : 1;  // instructions per row
    unsigned char* ring = sm + w * D * RPI * RB;
    for (long long i = 0; i < per_warp; i += RPI) {
        const int s = (int)((i / RPI) % D);
        const long long r = hashu((unsigned)(gw * 7919 + i + lane / (CH >= 32 ? 32 : CH))) % nrows;
#pragma unroll
        for (int k = 0; k < IPR; ++k) {
            const int ch = (k * 32 + lane) % CH;
            const unsigned dst = (unsigned)__cvta_generic_to_shared(ring + s * RPI * RB + (lane / (CH >= 32 ? 32 : CH)) * RB + ch * 16);
            asm volatile("cp.async.cg.shared.global [%0], [%1], 16;" ::"r"(dst), "l"(src + r * RB + ch * 16) : "memory");
        }
        asm volatile("cp.async.commit_group;" ::: "memory");
        asm volatile("cp.async.wait_group %0;" ::"n"(D - 1) : "memory");
    }
    asm volatile("cp.async.wait_group 0;" ::: "memory");
    if (ring[lane] == 123 && lane == 77) sink[0] = 1;
}

int main() {
    const long long bytes = 2LL << 30;
    unsigned char* src;
    unsigned* sink;
    cudaMalloc(&src, bytes);
    cudaMalloc(&sink, 4);
    cudaMemset(src, 1, bytes);
    cudaEvent_t a, b;
    cudaEventCreate(&a);
    cudaEventCreate(&b);
    auto run = [&](const char* nm, auto kern, int rb, int d, int warps_per_sm) {
        const long long total = 256LL << 20;
        const long long warps = 148LL * warps_per_sm;
        const long long per = total / rb / warps;
        const int rpi = rb >= 512 ? 1 : 512 / rb;
        const int smem = warps_per_sm * d * rpi * rb;
        cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
        float best = 1e9f;
        for (int it = 0; it < 4; ++it) {
            cudaEventRecord(a);
            kern<<<148, warps_per_sm * 32, smem>>>(src, bytes / rb, per, sink);
            cudaEventRecord(b);
            cudaEventSynchronize(b);
            float ms;
            cudaEventElapsedTime(&ms, a, b);
            if (ms < best) best = ms;
        }
        printf("%-22s D=%d W=%2d: %7.1f us  %7.1f GB/s\n", nm, d, warps_per_sm, best * 1e3, (double)(per * warps * rb) / (best * 1e-3) / 1e9);
    };
    run("rows 256 B", gather_rows<256, 4>, 256, 4, 16);
    run("rows 256 B", gather_rows<256, 8>, 256, 8, 16);
    run("rows 256 B", gather_rows<256, 16>, 256, 16, 16);
    run("rows 512 B", gather_rows<512, 8>, 512, 8, 16);
    run("blocks 4 KB", gather_rows<4096, 2>, 4096, 2, 16);
    run("blocks 4 KB", gather_rows<4096, 3>, 4096, 3, 16);
    printf("status %s\n", cudaGetErrorString(cudaDeviceSynchronize()));
    return 0;
}
