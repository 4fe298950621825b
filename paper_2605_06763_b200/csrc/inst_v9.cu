// bf16 query path, fused persistent layer kernel: DP in {64,128,256} x G in {1,2,4,8}.
#include "louver_v9.cuh"

namespace lvk9 {

template <int DP, int G>
static cudaError_t launch_t(V5Params vp, int slots, int sms, cudaStream_t st, int* geo) {
    using Ge = C9<DP, G>;
    static int smem_set = 0;
    static int occ = 0;
    // one wave, CTAs of a slot's team side by side; CTA b lists the survivors of
    // cells b, b + nb, ... so its list holds at most ceil(cap_cells / nb) cells
    const long long cap_cells = vp.p.cap_cells;
    int nb = vp.nb, smem = 0;
    for (int it = 0; it < 8; ++it) {
        smem = Ge::smem((int)((cap_cells + nb - 1) / nb));
        if (smem > smem_set) {
            cudaError_t e =
                cudaFuncSetAttribute(louver_layer_v9<DP, G>, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
            if (e != cudaSuccess) return e;
            e = cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ, louver_layer_v9<DP, G>, Ge::NTHR, smem);
            if (e != cudaSuccess) return e;
            if (occ < 1) return cudaErrorInvalidConfiguration;
            smem_set = smem;
        }
        int nb2 = occ * sms / slots;
        if (nb2 > vp.nb) nb2 = vp.nb;  // workspace holds vp.nb partials per slot
        if (nb2 < 1) nb2 = 1;
        if (nb2 >= nb) break;  // the list capacity for nb CTAs fits the resident wave
        nb = nb2;              // fewer CTAs per slot: longer lists, recheck
    }
    const int cap = occ * sms;
    int gy = cap / nb;
    if (gy > slots) gy = slots;
    vp.nb = nb;
    vp.slots = slots;
    if (geo) {  // team CTAs per slot, threads per CTA, dynamic smem, resident CTAs per SM
        geo[0] = nb;
        geo[1] = Ge::NTHR;
        geo[2] = smem;
        geo[3] = occ;
    }
    cudaLaunchConfig_t cfg{};
    cfg.gridDim = dim3((unsigned)nb, (unsigned)gy);
    cfg.blockDim = dim3(Ge::NTHR);
    cfg.dynamicSmemBytes = (size_t)smem;
    cfg.stream = st;
    cudaLaunchAttribute attr[1];
    attr[0].id = cudaLaunchAttributeCooperative;
    attr[0].val.cooperative = 1;
    cfg.attrs = attr;
    cfg.numAttrs = 1;
    cudaError_t e = cudaLaunchKernelEx(&cfg, louver_layer_v9<DP, G>, vp);
    if (e != cudaSuccess) return e;
    return cudaGetLastError();
}

cudaError_t launch_layer_v9(int DP, int G, V5Params vp, int slots, int sms, cudaStream_t st, int* geo) {
#define LV9_G(D)                                              \
    switch (G) {                                              \
        case 1: return launch_t<D, 1>(vp, slots, sms, st, geo);    \
        case 2: return launch_t<D, 2>(vp, slots, sms, st, geo);    \
        case 4: return launch_t<D, 4>(vp, slots, sms, st, geo);    \
        case 8: return launch_t<D, 8>(vp, slots, sms, st, geo);    \
    }                                                         \
    break;
    switch (DP) {
        case 64: LV9_G(64)
        case 128: LV9_G(128)
        case 256: LV9_G(256)
    }
#undef LV9_G
    return cudaErrorInvalidValue;
}

}  // namespace lvk9
