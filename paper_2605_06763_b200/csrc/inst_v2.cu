// v2 (bf16) query-kernel instantiations: DP in {64,128,256} x G in {1,2,4,8}.
#include "louver_v2.cuh"

namespace lvk2 {

template <int DP, int G>
static cudaError_t launch_t(const V2Params& vp, dim3 grid, cudaStream_t st) {
    static bool attr_done = false;
    constexpr int smem = G2<DP, G>::SMEM;
    if (!attr_done) {
        cudaError_t e = cudaFuncSetAttribute(louver_query_v2<DP, G>,
                                             cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
        if (e != cudaSuccess) return e;
        attr_done = true;
    }
    louver_query_v2<DP, G><<<grid, kThreads, smem, st>>>(vp);
    return cudaGetLastError();
}

int query_v2_smem(int DP, int G) {
#define LV2_S(D)                                  \
    switch (G) {                                  \
        case 1: return G2<D, 1>::SMEM;            \
        case 2: return G2<D, 2>::SMEM;            \
        case 4: return G2<D, 4>::SMEM;            \
        case 8: return G2<D, 8>::SMEM;            \
    }                                             \
    break;
    switch (DP) {
        case 64: LV2_S(64)
        case 128: LV2_S(128)
        case 256: LV2_S(256)
    }
#undef LV2_S
    return -1;
}

cudaError_t launch_query_v2(int DP, int G, const V2Params& vp, dim3 grid, cudaStream_t st) {
#define LV2_G(D)                                          \
    switch (G) {                                          \
        case 1: return launch_t<D, 1>(vp, grid, st);      \
        case 2: return launch_t<D, 2>(vp, grid, st);      \
        case 4: return launch_t<D, 4>(vp, grid, st);      \
        case 8: return launch_t<D, 8>(vp, grid, st);      \
    }                                                     \
    break;
    switch (DP) {
        case 64: LV2_G(64)
        case 128: LV2_G(128)
        case 256: LV2_G(256)
    }
#undef LV2_G
    return cudaErrorInvalidValue;
}

}  // namespace lvk2
