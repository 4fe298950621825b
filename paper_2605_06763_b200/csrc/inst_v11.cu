// bf16 query path, v11 loader-fed layer kernel: DP in {64,128,256} x G in {1,2,4,8}.
#include "louver_v11.cuh"

namespace lvk11 {

template <int DP, int G>
static cudaError_t launch_t(V10Params vp, int sms, cudaStream_t st, int* geo) {
    using Ge = C11<DP, G>;
    static bool smem_set = false;
    if (!smem_set) {
        cudaError_t e =
            cudaFuncSetAttribute(louver_layer_v11<DP, G>, cudaFuncAttributeMaxDynamicSharedMemorySize, Ge::SMEM);
        if (e != cudaSuccess) return e;
        smem_set = true;
    }
    // one CTA per SM (the shared-memory pool decides it); a team of nb CTAs per slot, all
    // resident together (grid <= SMs); the grid loops over slots when slots > SMs
    const int slots = vp.slots;
    int nb = sms / slots;
    if (nb < 1) nb = 1;
    if (nb > vp.nb) nb = vp.nb;  // the partial workspace holds vp.nb partials per slot
    int gy = sms / nb;
    if (gy > slots) gy = slots;
    vp.nb = nb;
    if (geo) {  // team CTAs per slot, threads per CTA, dynamic smem, resident CTAs per SM
        geo[0] = nb;
        geo[1] = Ge::NTHR;
        geo[2] = Ge::SMEM;
        geo[3] = 1;
    }
    cudaLaunchConfig_t cfg{};
    cfg.gridDim = dim3((unsigned)nb, (unsigned)gy);
    cfg.blockDim = dim3(Ge::NTHR);
    cfg.dynamicSmemBytes = (size_t)Ge::SMEM;
    cfg.stream = st;
    cudaLaunchAttribute attr[1];
    attr[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
    attr[0].val.programmaticStreamSerializationAllowed = 1;
    cfg.attrs = attr;
    cfg.numAttrs = 1;
    cudaError_t e = cudaLaunchKernelEx(&cfg, louver_layer_v11<DP, G>, vp);
    if (e != cudaSuccess) return e;
    return cudaGetLastError();
}

cudaError_t launch_layer_v11(int DP, int G, const V10Params& vp, int sms, cudaStream_t st, int* geo) {
#define LV11_G(D)                                        \
    switch (G) {                                         \
        case 1: return launch_t<D, 1>(vp, sms, st, geo); \
        case 2: return launch_t<D, 2>(vp, sms, st, geo); \
        case 4: return launch_t<D, 4>(vp, sms, st, geo); \
        case 8: return launch_t<D, 8>(vp, sms, st, geo); \
    }                                                    \
    break;
    switch (DP) {
        case 64: LV11_G(64)
        case 128: LV11_G(128)
        case 256: LV11_G(256)
    }
#undef LV11_G
    return cudaErrorInvalidValue;
}

}  // namespace lvk11
