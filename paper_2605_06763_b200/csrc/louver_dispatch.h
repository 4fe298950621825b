// Launch entry points of the templated query kernel; each (dtype, mode)
// instantiation set lives in its own translation unit (inst_*.cu) so the
// 72 specialisations compile in parallel.
#pragma once

#include <cuda_runtime.h>

#include "louver_kernels.cuh"
#include "louver_launch.h"

namespace lvk {

template <typename T, int DP, int G, int MODE>
cudaError_t launch_query_t(const QueryParams& p, dim3 grid, cudaStream_t st);

// Dynamic shared memory of one instantiation (bytes).
int query_smem_bytes(int dtype, int DP, int G);

cudaError_t launch_query(int dtype, int DP, int G, int mode, const QueryParams& p, dim3 grid,
                         cudaStream_t st);

}  // namespace lvk

#define LVK_DEFINE_LAUNCH(T, DP, G, MODE)                                                        \
    template <>                                                                                  \
    cudaError_t launch_query_t<T, DP, G, MODE>(const QueryParams& p, dim3 grid, cudaStream_t st) { \
        constexpr int smem = Geo<T, DP, G>::SMEM;                                                \
        cudaError_t e = lvl::func_smem(                                                          \
            reinterpret_cast<const void*>(louver_query_kernel<T, DP, G, MODE>), smem);           \
        if (e != cudaSuccess) return e;                                                          \
        louver_query_kernel<T, DP, G, MODE><<<grid, kThreads, smem, st>>>(p);                    \
        return cudaGetLastError();                                                               \
    }

#define LVK_DEFINE_LAUNCH_G(T, DP, MODE) \
    LVK_DEFINE_LAUNCH(T, DP, 1, MODE)    \
    LVK_DEFINE_LAUNCH(T, DP, 2, MODE)    \
    LVK_DEFINE_LAUNCH(T, DP, 4, MODE)    \
    LVK_DEFINE_LAUNCH(T, DP, 8, MODE)

#define LVK_DEFINE_LAUNCH_ALL(T, MODE)  \
    LVK_DEFINE_LAUNCH_G(T, 64, MODE)    \
    LVK_DEFINE_LAUNCH_G(T, 128, MODE)   \
    LVK_DEFINE_LAUNCH_G(T, 256, MODE)
