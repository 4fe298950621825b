// C++ sharded decode layer (include/louver_b200_nccl.hpp): query -> ncclAllGather of the
// (m, l, o) partials -> lv_lse_merge, and tail-shard inserts. One GPU here, so the
// communicator has one rank (ncclCommInitAll over device 0): the output must equal the
// unsharded layer's, and pushes go to the (single, tail) shard. The two-rank logic is
// covered by tests/test_sharding.py (two processes, gloo).
// usage: test_sharded [--compile-only]
#include <cmath>
#include <cstdio>
#include <cstring>
#include <vector>

#include "louver_b200_nccl.hpp"

using namespace louver_b200;

extern "C" int lv_synth_keys(int64_t n, int d, uint64_t seed, float* out);
extern "C" int lv_synth_queries(int64_t nq, int d, uint64_t seed, float* out);

int main(int argc, char** argv) {
    if (argc > 1 && std::strcmp(argv[1], "--compile-only") == 0) {
        std::printf("%s nccl %d\n", lv_build_info(), NCCL_VERSION_CODE);
        return 0;
    }
    const int d = 128, H = 2, G = 4, n = 6000, rows = H * G;
    auto [f0, c0] = shard_range(n, 3, 1);
    if (f0 != 2000 || c0 != 2000 || insert_owner(4) != 3) {
        std::printf("FAIL shard_range\n");
        return 1;
    }
    std::vector<float> K((size_t)H * n * d), V((size_t)H * n * d), Q((size_t)rows * d), tau(rows, 30.0f);
    for (int h = 0; h < H; ++h) {
        lv_synth_keys(n, d, 300 + h, K.data() + (size_t)h * n * d);
        lv_synth_keys(n, d, 400 + h, V.data() + (size_t)h * n * d);
        lv_synth_queries(G, d, 300 + h, Q.data() + (size_t)h * G * d);
    }
    BuildConfig cfg;
    cfg.r = 16;
    LouverLayer a(d, H, G, 1, n + 64, cfg, 32), b(d, H, G, 1, n + 64, cfg, 32);
    a.build(K.data(), V.data(), n, LV_F32, LV_HOST);
    b.build(K.data(), V.data(), n, LV_F32, LV_HOST);
    ncclComm_t comm;
    int dev = 0;
    detail::nccl_check(ncclCommInitAll(&comm, 1, &dev), "ncclCommInitAll");
    ShardedLayer sh(b, comm);
    float *qd, *td, *oa, *ob, *kv;
    cudaMalloc(&qd, sizeof(float) * rows * d);
    cudaMalloc(&td, sizeof(float) * rows);
    cudaMalloc(&oa, sizeof(float) * rows * d);
    cudaMalloc(&ob, sizeof(float) * rows * d);
    cudaMalloc(&kv, sizeof(float) * H * d);
    cudaMemcpy(qd, Q.data(), sizeof(float) * rows * d, cudaMemcpyHostToDevice);
    cudaMemcpy(td, tau.data(), sizeof(float) * rows, cudaMemcpyHostToDevice);
    cudaMemcpy(kv, K.data(), sizeof(float) * H * d, cudaMemcpyHostToDevice);  // a new key per slot
    for (int s = 0; s < 40; ++s) {  // inserts through the sharded layer reach the tail shard
        sh.push_key(kv, kv, LV_F32, LV_DEVICE);
        a.push_key(kv, kv, LV_F32, LV_DEVICE);
    }
    a.query_device(qd, td, oa, nullptr);
    sh.query(qd, td, ob, nullptr);
    cudaDeviceSynchronize();
    std::vector<float> ha(rows * d), hb(rows * d);
    cudaMemcpy(ha.data(), oa, sizeof(float) * rows * d, cudaMemcpyDeviceToHost);
    cudaMemcpy(hb.data(), ob, sizeof(float) * rows * d, cudaMemcpyDeviceToHost);
    double num = 0, den = 0;
    for (int i = 0; i < rows * d; ++i) {
        num += (double(ha[i]) - hb[i]) * (double(ha[i]) - hb[i]);
        den += double(ha[i]) * ha[i];
    }
    const double err = std::sqrt(num / (den > 0 ? den : 1));
    const bool ok = err <= 1e-6 && b.n() == n + 40 && den > 0;
    std::printf("sharded (1 rank) vs unsharded: rel err %.3g, n %lld -> %s\n", err, (long long)b.n(), ok ? "OK" : "FAIL");
    ncclCommDestroy(comm);
    return ok ? 0 : 1;
}
