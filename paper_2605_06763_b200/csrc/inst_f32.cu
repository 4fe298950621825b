// fp32 layer kernel instantiations: DP in {128, 256} x G in {1, 2, 4, 8}.
#include "louver_f32.cuh"
#include "louver_launch.h"

namespace lvkf {

template <int DP, int G>
static cudaError_t launch_t(F32Params fp, int slots, int sms, cudaStream_t st, int* geo) {
    using Ge = CF<DP, G>;
    const void* fn = reinterpret_cast<const void*>(louver_layer_f32<DP, G>);
    const long long cap_cells = fp.p.cap_cells;
    if (fp.p.cap >= (1LL << 31) - 64) return cudaErrorInvalidValue;  // 32-bit key indices
    constexpr int kSmemMax = 227 * 1024;
    int nb = fp.nb, smem = 0, occ = 0;
    bool glist = false;
    for (int it = 0; it < 8; ++it) {
        const long long lc = (cap_cells + nb - 1) / nb;
        if (lc > 65536) return cudaErrorInvalidValue;  // u16 interleave indices
        glist = Ge::smem((int)lc) > kSmemMax;
        smem = glist ? Ge::DYN : Ge::smem((int)lc);
        cudaError_t e = lvl::func_smem(fn, smem, Ge::NTHR, &occ);
        if (e != cudaSuccess) return e;
        if (occ < 1) return cudaErrorInvalidConfiguration;
        int nb2 = occ * sms / slots;
        if (nb2 > fp.nb) nb2 = fp.nb;
        if (nb2 < 1) nb2 = 1;
        if (nb2 >= nb) break;
        nb = nb2;
    }
    fp.list_cap = (int)((cap_cells + nb - 1) / nb);
    if (!glist) fp.glist = nullptr;
    int gy = occ * sms / nb;
    if (gy > slots) gy = slots;
    fp.nb = nb;
    fp.slots = slots;
    if (geo) {
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
    attr[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
    attr[0].val.programmaticStreamSerializationAllowed = 1;
    cfg.attrs = attr;
    cfg.numAttrs = 1;
    cudaError_t e = cudaLaunchKernelEx(&cfg, louver_layer_f32<DP, G>, fp);
    if (e != cudaSuccess) return e;
    return cudaGetLastError();
}

cudaError_t launch_layer_f32(int DP, int G, F32Params fp, int slots, int sms, cudaStream_t st, int* geo) {
#define LVF_G(D)                                                            \
    switch (G) {                                                            \
        case 1: return launch_t<D, 1>(fp, slots, sms, st, geo);             \
        case 2: return launch_t<D, 2>(fp, slots, sms, st, geo);             \
        case 4: return launch_t<D, 4>(fp, slots, sms, st, geo);             \
        case 8: return launch_t<D, 8>(fp, slots, sms, st, geo);             \
    }                                                                       \
    break;
    switch (DP) {
        case 128: LVF_G(128)
        case 256: LVF_G(256)
    }
#undef LVF_G
    return cudaErrorInvalidValue;
}

}  // namespace lvkf
