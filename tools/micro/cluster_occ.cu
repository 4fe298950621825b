// How many thread-block clusters of size C fit at once on this GPU when each CTA needs a
// whole SM (512 threads, ~229 KB dynamic smem, like the fused layer kernel)?
#include <cuda_runtime.h>
#include <cstdio>
__global__ void dummy(int* p) { extern __shared__ int s[]; if (threadIdx.x == 9999) p[0] = s[0]; }
int main() {
    const int smem = 220 * 1024;
    cudaFuncSetAttribute(dummy, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
    cudaFuncSetAttribute(dummy, cudaFuncAttributeNonPortableClusterSizeAllowed, 1);
    int sms; cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
    printf("SMs %d\n", sms);
    for (int c : {1, 2, 3, 4, 6, 8, 9, 12, 16}) {
        cudaLaunchConfig_t cfg{};
        cfg.gridDim = dim3(c * 8, 1);
        cfg.blockDim = dim3(512);
        cfg.dynamicSmemBytes = smem;
        cudaLaunchAttribute at[1];
        at[0].id = cudaLaunchAttributeClusterDimension;
        at[0].val.clusterDim.x = c; at[0].val.clusterDim.y = 1; at[0].val.clusterDim.z = 1;
        cfg.attrs = at; cfg.numAttrs = 1;
        int n = -1;
        cudaError_t e = cudaOccupancyMaxActiveClusters(&n, dummy, &cfg);
        printf("cluster %2d: max active clusters %3d (%3d CTAs)  %s\n", c, n, n * c, cudaGetErrorString(e));
    }
    return 0;
}
