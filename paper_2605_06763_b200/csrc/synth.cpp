// Synthetic key/value/query streams with the reference's data laws
// (proj/src/io.cpp:89-206), used as measurement input by bench.py and the
// parity tests. Host-only; built into liblouver_synth.so. The generators draw
// from std::mt19937_64 + std::normal_distribution<double>, so with libstdc++
// they reproduce the reference's bytes exactly.
//
// Gaussian law (io.cpp:145-169): key_t = 1.5 * m_t * v + 0.3 * e_t where v is
// a fixed heavy-tailed direction (random signs, exp(2.5 N(0,1)) magnitudes,
// io.cpp:106-115), m_t a unit-variance AR(1) with phi 0.95 and e_t a
// per-coordinate unit-variance AR(1) with phi 0.9.
// Queries (io.cpp:186-202): sign(v) + 0.25 N(0,1), from an independent stream.

#include <cmath>
#include <cstdint>
#include <random>
#include <thread>
#include <vector>

#include "louver_b200.h"

namespace {

constexpr double kMagScale = 1.5, kMagPhi = 0.95;
constexpr double kResScale = 0.3, kResPhi = 0.9;
constexpr double kDirLogStd = 2.5;
constexpr double kQuerySignWeight = 1.0, kQueryNoise = 0.25;
constexpr std::uint64_t kDirSalt = 0x9E3779B97F4A7C15ULL;
constexpr std::uint64_t kQuerySalt = 0xC2B2AE3D27D4EB4FULL;

std::vector<float> direction(int d, std::uint64_t seed) {
    std::mt19937_64 eng(seed ^ kDirSalt);
    std::normal_distribution<double> z(0.0, 1.0);
    std::vector<float> v(d);
    for (int c = 0; c < d; ++c) {
        const double sgn = z(eng) < 0.0 ? -1.0 : 1.0;
        v[c] = static_cast<float>(sgn * std::exp(kDirLogStd * z(eng)));
    }
    return v;
}

void gaussian_stream(std::int64_t n, int d, std::uint64_t seed, float* out) {
    const std::vector<float> v = direction(d, seed);
    std::mt19937_64 eng(seed);
    std::normal_distribution<double> z(0.0, 1.0);
    const double inn_m = std::sqrt(1.0 - kMagPhi * kMagPhi);
    const double inn_r = std::sqrt(1.0 - kResPhi * kResPhi);
    double mag = z(eng);
    std::vector<double> res(d);
    for (int c = 0; c < d; ++c) res[c] = z(eng);
    for (std::int64_t t = 0; t < n; ++t) {
        if (t > 0) mag = kMagPhi * mag + inn_m * z(eng);
        float* row = out + static_cast<std::size_t>(t) * d;
        for (int c = 0; c < d; ++c) {
            if (t > 0) res[c] = kResPhi * res[c] + inn_r * z(eng);
            row[c] = static_cast<float>(kMagScale * mag * double(v[c]) + kResScale * res[c]);
        }
    }
}

void gaussian_queries(std::int64_t nq, int d, std::uint64_t seed, float* out) {
    const std::vector<float> v = direction(d, seed);
    std::mt19937_64 eng(seed ^ kQuerySalt);
    std::normal_distribution<double> z(0.0, 1.0);
    for (std::int64_t i = 0; i < nq; ++i)
        for (int c = 0; c < d; ++c) {
            const double sgn = v[c] < 0.0f ? -1.0 : 1.0;
            out[static_cast<std::size_t>(i) * d + c] =
                static_cast<float>(kQuerySignWeight * sgn + kQueryNoise * z(eng));
        }
}

// Mixture law (io.cpp:117-143, 171-183, 203-205).
std::vector<float> mixture_centers(int k, int d, std::uint64_t seed) {
    std::mt19937_64 eng(seed);
    std::normal_distribution<double> z(0.0, 1.0);
    std::vector<float> c(static_cast<std::size_t>(k) * d);
    for (auto& x : c) x = static_cast<float>(4.0 * z(eng));
    return c;
}

void mixture_points(const std::vector<float>& centers, int k, double spread, std::int64_t n, int d,
                    std::mt19937_64& eng, std::normal_distribution<double>& z, float* out) {
    std::uniform_int_distribution<int> pick(0, k - 1);
    for (std::int64_t i = 0; i < n; ++i) {
        const int which = pick(eng);
        for (int c = 0; c < d; ++c)
            out[static_cast<std::size_t>(i) * d + c] =
                centers[static_cast<std::size_t>(which) * d + c] + static_cast<float>(spread * z(eng));
    }
}

}  // namespace

extern "C" {

int lv_synth_keys(int64_t n, int d, uint64_t seed, float* out) {
    if (n < 1 || d < 1 || !out) return LV_EINVAL;
    gaussian_stream(n, d, seed, out);
    return LV_OK;
}

int lv_synth_queries(int64_t nq, int d, uint64_t seed, float* out) {
    if (nq < 1 || d < 1 || !out) return LV_EINVAL;
    gaussian_queries(nq, d, seed, out);
    return LV_OK;
}

int lv_synth_mixture(int64_t n, int d, int k, double spread, uint64_t seed, int queries,
                     float* out) {
    if (n < 1 || d < 1 || k < 1 || spread < 0.0 || !out) return LV_EINVAL;
    const std::vector<float> centers = mixture_centers(k, d, seed);
    std::normal_distribution<double> z(0.0, 1.0);
    if (queries) {
        std::mt19937_64 eng(seed ^ kQuerySalt);
        mixture_points(centers, k, spread, n, d, eng, z, out);
    } else {
        std::mt19937_64 eng(seed);
        for (int i = 0; i < k * d; ++i) z(eng);  // skip the draws the centers used
        mixture_points(centers, k, spread, n, d, eng, z, out);
    }
    return LV_OK;
}

// Many independent key streams at once (one per (layer, batch, kv head)):
// streams[s] = gen(n, d, seeds[s]) written at out + s*n*d. Threads split the
// streams; each stream is sequential in t, as its AR(1) law requires.
int lv_synth_keys_multi(int64_t n, int d, const uint64_t* seeds, int64_t nstreams, float* out,
                        int threads) {
    if (n < 1 || d < 1 || nstreams < 0 || !out || !seeds) return LV_EINVAL;
    if (threads < 1) threads = static_cast<int>(std::max(1u, std::thread::hardware_concurrency()));
    std::vector<std::thread> pool;
    for (int t = 0; t < threads; ++t)
        pool.emplace_back([=] {
            for (int64_t s = t; s < nstreams; s += threads)
                gaussian_stream(n, d, seeds[s], out + static_cast<std::size_t>(s) * n * d);
        });
    for (auto& th : pool) th.join();
    return LV_OK;
}

}  // extern "C"
