// bf16 query path instantiations (probe -> pipelined cell stream): DP in {64,128,256} x G in {1,2,4,8}.
#include "louver_v8.cuh"

namespace lvk8 {

template <int DP, int G>
static cudaError_t launch_t(const V5Params& vp, int slots, cudaStream_t st) {
    static bool attr_done = false;
    static int smem2_set = 0;
    constexpr int smem1 = P5<DP, G>::SMEM;
    const int smem2 = C8<DP, G>::smem(vp.tiles);
    if (!attr_done) {
        cudaError_t e = cudaFuncSetAttribute(louver_probe_v5<DP, G>, cudaFuncAttributeMaxDynamicSharedMemorySize, smem1);
        if (e != cudaSuccess) return e;
        attr_done = true;
    }
    if (smem2 > smem2_set) {
        cudaError_t e = cudaFuncSetAttribute(louver_cells_v8<DP, G>, cudaFuncAttributeMaxDynamicSharedMemorySize, smem2);
        if (e != cudaSuccess) return e;
        smem2_set = smem2;
    }
    louver_probe_v5<DP, G><<<dim3((unsigned)vp.nbp, (unsigned)slots), kT, smem1, st>>>(vp);
    cudaError_t e = cudaGetLastError();
    if (e != cudaSuccess) return e;
    // programmatic dependent launch: the cell stream's setup overlaps the probe's tail
    cudaLaunchConfig_t cfg{};
    cfg.gridDim = dim3((unsigned)vp.nb, (unsigned)slots);
    cfg.blockDim = dim3(kT);
    cfg.dynamicSmemBytes = (size_t)smem2;
    cfg.stream = st;
    cudaLaunchAttribute attr[1];
    attr[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
    attr[0].val.programmaticStreamSerializationAllowed = 1;
    cfg.attrs = attr;
    cfg.numAttrs = 1;
    e = cudaLaunchKernelEx(&cfg, louver_cells_v8<DP, G>, vp);
    if (e != cudaSuccess) return e;
    return cudaGetLastError();
}

cudaError_t launch_query_v8(int DP, int G, const V5Params& vp, int slots, cudaStream_t st) {
#define LV8_G(D)                                          \
    switch (G) {                                          \
        case 1: return launch_t<D, 1>(vp, slots, st);     \
        case 2: return launch_t<D, 2>(vp, slots, st);     \
        case 4: return launch_t<D, 4>(vp, slots, st);     \
        case 8: return launch_t<D, 8>(vp, slots, st);     \
    }                                                     \
    break;
    switch (DP) {
        case 64: LV8_G(64)
        case 128: LV8_G(128)
        case 256: LV8_G(256)
    }
#undef LV8_G
    return cudaErrorInvalidValue;
}

}  // namespace lvk8
