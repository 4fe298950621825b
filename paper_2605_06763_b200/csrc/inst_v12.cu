// bf16 query path, fused persistent layer kernel: DP in {64,128,256} x G in {1,2,4,8}.
#include "louver_v12.cuh"

namespace lvk12 {

template <int DP, int G>
static cudaError_t launch_t(V5Params vp, int slots, int sms, cudaStream_t st, int* geo) {
    using Ge = C12<DP, G>;
    static int smem_set = 0;
    static int occ = 0;
    // one wave, CTAs of a slot's team side by side; CTA b lists the survivors of
    // cells b, b + nb, ... so its list holds at most ceil(cap_cells / nb) cells
    const long long cap_cells = vp.p.cap_cells;
    // CTA b of a slot's team owns cells b, b + nb, ...: its survivor list holds at most
    // ceil(cap_cells / nb) u16 entries, in smem when that fits, else in global scratch
    constexpr int kSmemMax = 227 * 1024;
    int nb = vp.nb, smem = 0;
    bool glist = false;
    for (int it = 0; it < 8; ++it) {
        const long long lc = (cap_cells + nb - 1) / nb;
        if (lc > 65536) return cudaErrorInvalidValue;  // u16 interleave indices
        glist = Ge::smem((int)lc) > kSmemMax;
        smem = glist ? Ge::DYN : Ge::smem((int)lc);
        if (smem > smem_set) {
            cudaError_t e =
                cudaFuncSetAttribute(louver_layer_v12<DP, G>, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
            if (e != cudaSuccess) return e;
            e = cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ, louver_layer_v12<DP, G>, Ge::NTHR, smem);
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
    vp.list_cap = (int)((cap_cells + nb - 1) / nb);
    if (!glist) vp.glist = nullptr;  // else: the caller's scratch of slots * (cap_cells + nb) entries
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
    // no grid-wide waiting remains (the merge ticket never blocks), so no cooperative
    // launch is needed; the grid is still sized to one resident wave. Programmatic
    // stream serialization lets the CTAs be dispatched while the previous kernel
    // drains; the kernel's first instruction waits for that kernel's completion.
    cudaLaunchAttribute attr[1];
    attr[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
    attr[0].val.programmaticStreamSerializationAllowed = 1;
    cfg.attrs = attr;
    cfg.numAttrs = 1;
    cudaError_t e = cudaLaunchKernelEx(&cfg, louver_layer_v12<DP, G>, vp);
    if (e != cudaSuccess) return e;
    return cudaGetLastError();
}

cudaError_t launch_layer_v12(int DP, int G, V5Params vp, int slots, int sms, cudaStream_t st, int* geo) {
#define LV12_G(D)                                              \
    switch (G) {                                              \
        case 1: return launch_t<D, 1>(vp, slots, sms, st, geo);    \
        case 2: return launch_t<D, 2>(vp, slots, sms, st, geo);    \
        case 4: return launch_t<D, 4>(vp, slots, sms, st, geo);    \
        case 8: return launch_t<D, 8>(vp, slots, sms, st, geo);    \
    }                                                         \
    break;
    switch (DP) {
        case 64: LV12_G(64)
        case 128: LV12_G(128)
        case 256: LV12_G(256)
    }
#undef LV12_G
    return cudaErrorInvalidValue;
}

}  // namespace lvk12
