// Per-device, thread-safe launch attributes (host side).
//
// cudaFuncSetAttribute(MaxDynamicSharedMemorySize) applies to the CURRENT device only,
// and lv_query may be called from several host threads (louver_b200.h threading
// contract), so the raised limit and the occupancy it yields are cached per
// (device, kernel) under one mutex instead of in function-local statics.
#pragma once

#include <cuda_runtime.h>

#include <map>
#include <mutex>
#include <tuple>

namespace lvl {

// Make `fn` launchable with `bytes` of dynamic shared memory on the current device and
// (when occ != nullptr) return its resident CTAs per SM at `threads` x `bytes`.
inline cudaError_t func_smem(const void* fn, int bytes, int threads = 0, int* occ = nullptr) {
    static std::mutex mu;
    static std::map<std::pair<int, const void*>, int> limit;              // raised limit per (device, fn)
    static std::map<std::tuple<int, const void*, int, int>, int> blocks;  // occupancy per (device, fn, threads, bytes)
    int dev = 0;
    cudaError_t e = cudaGetDevice(&dev);
    if (e != cudaSuccess) return e;
    std::lock_guard<std::mutex> lock(mu);
    int& lim = limit[{dev, fn}];
    if (bytes > lim && bytes > 48 * 1024) {
        // only ever raised: a concurrent launch with a larger request stays valid
        e = cudaFuncSetAttribute(fn, cudaFuncAttributeMaxDynamicSharedMemorySize, bytes);
        if (e != cudaSuccess) return e;
        lim = bytes;
    }
    if (occ) {
        const auto key = std::make_tuple(dev, fn, threads, bytes);
        auto it = blocks.find(key);
        if (it == blocks.end()) {
            int o = 0;
            e = cudaOccupancyMaxActiveBlocksPerMultiprocessor(&o, fn, threads, bytes);
            if (e != cudaSuccess) return e;
            it = blocks.emplace(key, o).first;
        }
        *occ = it->second;
    }
    return cudaSuccess;
}

// Multiprocessor count of the current device (cached per device).
inline int device_sms() {
    static std::mutex mu;
    static std::map<int, int> sms;
    int dev = 0;
    if (cudaGetDevice(&dev) != cudaSuccess) return 148;
    std::lock_guard<std::mutex> lock(mu);
    auto it = sms.find(dev);
    if (it == sms.end()) {
        int s = 148;
        cudaDeviceGetAttribute(&s, cudaDevAttrMultiProcessorCount, dev);
        it = sms.emplace(dev, s).first;
    }
    return it->second;
}

}  // namespace lvl
