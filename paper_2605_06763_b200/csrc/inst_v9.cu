// bf16 layer kernel instantiations: DP in {64,128,256} x G in {1,2,4,8} x {query, dense}.
#include "louver_launch.h"
#include "louver_v9.cuh"

namespace lvk9 {

template <int DP, int G, bool DENSE, bool CNT>
static cudaError_t launch_t(LayerParams vp, int slots, int sms, cudaStream_t st, int* geo) {
    using Ge = C9<DP, G>;
    const void* fn = reinterpret_cast<const void*>(louver_layer_v9<DP, G, DENSE, CNT>);
    // One resident wave, a slot's team CTAs side by side. CTA b of a team owns cells b,
    // b + nb, ...: its survivor list holds at most ceil(cap_cells / nb) u16 entries, in
    // shared memory when that fits, else in global scratch (the dense scan keeps no list).
    const long long cap_cells = vp.p.cap_cells;
    if (vp.p.cap >= (1LL << 31) - 64) return cudaErrorInvalidValue;  // 32-bit key indices in the task loop
    constexpr int kSmemMax = 227 * 1024;
    int nb = vp.nb, smem = 0, occ = 0;
    bool glist = false;
    for (int it = 0; it < 8; ++it) {
        const long long lc = (cap_cells + nb - 1) / nb;
        if (!DENSE && lc > 65536) return cudaErrorInvalidValue;  // u16 interleave indices
        glist = !DENSE && Ge::smem((int)lc) > kSmemMax;
        smem = (DENSE || glist) ? Ge::DYN : Ge::smem((int)lc);
        cudaError_t e = lvl::func_smem(fn, smem, Ge::NTHR, &occ);
        if (e != cudaSuccess) return e;
        if (occ < 1) return cudaErrorInvalidConfiguration;
        int nb2 = occ * sms / slots;
        if (nb2 > vp.nb) nb2 = vp.nb;  // the workspace holds vp.nb partials per slot
        if (nb2 < 1) nb2 = 1;
        if (nb2 >= nb) break;  // the list capacity for nb CTAs fits the resident wave
        nb = nb2;              // fewer CTAs per slot: longer lists, recheck
    }
    if (Ge::PERW % 128) vp.ktma = 0;  // TMA destinations need 128-byte aligned stages
    vp.list_cap = (int)((cap_cells + nb - 1) / nb);
    if (!glist) vp.glist = nullptr;  // else: the caller's scratch of slots * (cap_cells + nb) entries
    const int cap = occ * sms;
    int gy = cap / nb;
    if (gy > slots) gy = slots;
    // Every slot resident and SMs left over (148 over 8 slots: 4 idle with teams of 18):
    // the first cap - nb * slots slots get one CTA more (lists sized for the smaller team,
    // partial records for vp.nb per slot; vp.nfull != 0 on entry allows it)
    int nfull = slots;
    if (vp.nfull && !glist && gy == slots && nb >= 2 && nb + 1 <= vp.nb && cap > nb * slots) {
        nfull = cap - nb * slots < slots ? cap - nb * slots : slots;
        ++nb;
    }
    vp.nfull = nfull;
    vp.nb = nb;
    vp.slots = slots;
    if (geo) {  // team CTAs per slot, threads per CTA, dynamic smem, resident CTAs per SM
        geo[0] = nb;
        geo[1] = Ge::NTHR;
        geo[2] = smem;
        geo[3] = occ;
    }
    cudaLaunchConfig_t cfg{};
    // spread: grid (slots, team), so the CTAs dispatched last (onto the SMs the previous
    // layer's merging CTAs free) are one member of each slot. The smaller teams leave
    // placeholder CTAs at the very end of the order, which exit at once; measured, they are
    // better than an exact 1-D grid
    if (gy != slots) vp.spread = 0;
    cfg.gridDim = vp.spread ? dim3((unsigned)gy, (unsigned)nb) : dim3((unsigned)nb, (unsigned)gy);
    cfg.blockDim = dim3(Ge::NTHR);
    cfg.dynamicSmemBytes = (size_t)smem;
    cfg.stream = st;
    // No grid-wide waiting (the merge ticket never blocks), so no cooperative launch; the
    // grid is still one resident wave. Programmatic stream serialisation lets the CTAs be
    // dispatched while the previous kernel drains; the kernel waits for it with
    // griddepcontrol.wait before reading anything mutable.
    cudaLaunchAttribute attr[1];
    attr[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
    attr[0].val.programmaticStreamSerializationAllowed = 1;
    cfg.attrs = attr;
    cfg.numAttrs = 1;
    cudaError_t e;
    if constexpr (!CNT) {
        if (nb == 1) {  // teams of one: the instantiation without the team merge
            const void* fn1 = reinterpret_cast<const void*>(louver_layer_v9<DP, G, DENSE, false, true>);
            if ((e = lvl::func_smem(fn1, smem)) != cudaSuccess) return e;
            e = cudaLaunchKernelEx(&cfg, louver_layer_v9<DP, G, DENSE, false, true>, vp);
            if (e != cudaSuccess) return e;
            return cudaGetLastError();
        }
    }
    e = cudaLaunchKernelEx(&cfg, louver_layer_v9<DP, G, DENSE, CNT>, vp);
    if (e != cudaSuccess) return e;
    return cudaGetLastError();
}

cudaError_t launch_layer_v9(int DP, int G, bool dense, LayerParams vp, int slots, int sms, cudaStream_t st,
                            int* geo) {
    // dense decode never reports counts; a query does when p.counts is set
    const int mode = dense ? 0 : (vp.p.counts ? 2 : 1);
#define LV9_M(D, GG)                                                                                   \
    return mode == 0 ? launch_t<D, GG, true, false>(vp, slots, sms, st, geo)                          \
                     : (mode == 1 ? launch_t<D, GG, false, false>(vp, slots, sms, st, geo)            \
                                  : launch_t<D, GG, false, true>(vp, slots, sms, st, geo));
#define LV9_G(D)          \
    switch (G) {          \
        case 1: LV9_M(D, 1) \
        case 2: LV9_M(D, 2) \
        case 4: LV9_M(D, 4) \
        case 8: LV9_M(D, 8) \
    }                     \
    break;
    switch (DP) {
        case 64: LV9_G(64)
        case 128: LV9_G(128)
        case 256: LV9_G(256)
    }
#undef LV9_G
#undef LV9_M
    return cudaErrorInvalidValue;
}

}  // namespace lvk9
