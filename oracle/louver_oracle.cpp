// TEST INFRASTRUCTURE — NOT PRODUCT CODE (see louver_oracle.h).
//
// Plain C++17 restatement of the reference Louver library (CPU, Eigen-free).
// Reference paths below are relative to /root/reference/proj. Build flags
// (oracle/Makefile): -O3 -ffp-contract=off, no -march: the reference's
// Release build on x86-64 emits mulss/addss with no FMA,
// and fp-contract=off keeps that true here whatever the host CPU is.

#include "louver_oracle.h"

#include <algorithm>
#include <cmath>
#include <cstring>
#include <limits>
#include <memory>
#include <numeric>
#include <random>
#include <stdexcept>
#include <string>
#include <vector>

namespace {

thread_local std::string g_error;

using Id = std::uint32_t;
constexpr float kInf = std::numeric_limits<float>::infinity();

// core.hpp:17-21 — strict left-to-right fp32 accumulation, one rounding per
// multiply and per add.
inline float ndot(const float* a, const float* b, std::ptrdiff_t len) {
    float acc = 0.0f;
    for (std::ptrdiff_t i = 0; i < len; ++i) acc += a[i] * b[i];
    return acc;
}

inline float nnorm(const float* a, std::ptrdiff_t len) { return std::sqrt(ndot(a, a, len)); }

// core.hpp:35-54 — S contiguous slices of [0,d), the d%S wider ones first.
struct Slices {
    int d = 0, S = 0;
    std::vector<int> off;
    Slices() = default;
    Slices(int dim, int subspaces) : d(dim), S(subspaces) {
        if (subspaces < 1 || subspaces > dim)
            throw std::invalid_argument("SubspaceLayout: need 1 <= S <= d");
        off.assign(S + 1, 0);
        const int base = d / S, extra = d % S;
        for (int s = 0; s < S; ++s) off[s + 1] = off[s] + base + (s < extra ? 1 : 0);
    }
    int begin(int s) const { return off[s]; }
    int width(int s) const { return off[s + 1] - off[s]; }
};

struct Config {
    int S = 4, r = 4, grouping = 3, enclosure = 0;
    std::uint64_t seed = 0;
    // index.hpp:17-21
    void validate(int d) const {
        if (S < 1) throw std::invalid_argument("BuildConfig: S >= 1 required");
        if (r < 1) throw std::invalid_argument("BuildConfig: r >= 1 required");
        if (S > d) throw std::invalid_argument("BuildConfig: S <= d required");
        if (grouping < 0 || grouping > 3 || enclosure < 0 || enclosure > 2)
            throw std::invalid_argument("BuildConfig: unknown grouping/enclosure");
    }
};

Config to_config(const lvo_build_config* c) {
    Config out;
    if (c) {
        out.S = c->S;
        out.r = c->r;
        out.grouping = c->grouping;
        out.enclosure = c->enclosure;
        out.seed = c->rng_seed;
    }
    return out;
}

// core.hpp:116-169 — append-only fp32 row store (growth is std::vector's).
struct Store {
    int d = 0;
    std::int64_t n = 0;
    std::vector<float> K, V;
    const float* key(Id j) const { return K.data() + static_cast<std::size_t>(j) * d; }
    const float* value(Id j) const { return V.data() + static_cast<std::size_t>(j) * d; }
    void append(const float* k, const float* v) {
        K.insert(K.end(), k, k + d);
        V.insert(V.end(), v, v + d);
        ++n;
    }
};

enum { kBall = 0, kAabb = 1, kSpan = 2 };

// core.hpp:79-93
struct Encl {
    int kind = kBall;
    std::vector<float> center, lo, hi;
    float radius = 0.0f;
};

// index.hpp:24-49, flattened: per-group enclosures plus the packed
// coordinate-major gate arrays and member lists the query path streams.
struct Sub {
    std::vector<std::uint32_t> assign;
    std::vector<Encl> encl;
    std::vector<std::vector<float>> gc, glo, ghi;  // [width][K]
    std::vector<float> grad;                       // [K]
    double norm_bound = 0.0;
    std::vector<std::uint32_t> moff{0};
    std::vector<Id> mids;
    std::size_t groups() const { return encl.size(); }
};

struct Index {
    Slices lay;
    Config cfg;
    std::vector<Sub> subs;
    std::int64_t indexed = 0;
};

// ---------------------------------------------------------------- grouping

// index.cpp:15-56 — median bisection on the max-variance axis. `pts` is the
// local row-major block [m][w]; `ids` the working permutation.
std::uint32_t pca_split(const float* pts, int w, Id* ids, std::size_t lo, std::size_t hi, int r,
                        std::uint32_t offset, std::vector<std::uint32_t>& out) {
    const std::size_t m = hi - lo;
    if (m <= static_cast<std::size_t>(r)) {
        for (std::size_t i = lo; i < hi; ++i) out[ids[i]] = offset;
        return 1;
    }
    int axis = 0;
    double best = -1.0;
    for (int c = 0; c < w; ++c) {
        double mu = 0.0;
        for (std::size_t i = lo; i < hi; ++i) mu += pts[static_cast<std::size_t>(ids[i]) * w + c];
        mu /= static_cast<double>(m);
        double var = 0.0;
        for (std::size_t i = lo; i < hi; ++i) {
            const double dv = pts[static_cast<std::size_t>(ids[i]) * w + c] - mu;
            var += dv * dv;
        }
        if (var > best) {  // strict: the lowest axis wins ties
            best = var;
            axis = c;
        }
    }
    std::sort(ids + lo, ids + hi, [&](Id a, Id b) {
        const float pa = pts[static_cast<std::size_t>(a) * w + axis];
        const float pb = pts[static_cast<std::size_t>(b) * w + axis];
        return pa != pb ? pa < pb : a < b;
    });
    const std::size_t half = m / 2;
    const std::uint32_t left = pca_split(pts, w, ids, lo, lo + half, r, offset, out);
    const std::uint32_t right = pca_split(pts, w, ids, lo + half, hi, r, offset + left, out);
    return left + right;
}

// index.cpp:60-68
std::vector<std::uint32_t> pca_tree(const float* pts, std::size_t m, int w, int r) {
    if (m == 0) throw std::invalid_argument("balanced_pca_tree: empty point set");
    std::vector<Id> ids(m);
    std::iota(ids.begin(), ids.end(), 0u);
    std::vector<std::uint32_t> out(m);
    pca_split(pts, w, ids.data(), 0, m, r, 0, out);
    return out;
}

// index.cpp:70-102
std::vector<std::uint32_t> group_keys(const float* pts, std::size_t m, int w, const Config& cfg,
                                      int subspace, Id base_id) {
    if (m == 0) throw std::invalid_argument("assign_groups: empty point set");
    const std::size_t r = static_cast<std::size_t>(cfg.r);
    std::vector<std::uint32_t> out(m);
    if (cfg.grouping == 0) {
        for (std::size_t j = 0; j < m; ++j) out[j] = static_cast<std::uint32_t>(j / r);
    } else if (cfg.grouping == 1) {
        const std::size_t K = (m + r - 1) / r;
        for (std::size_t j = 0; j < m; ++j) out[j] = static_cast<std::uint32_t>(j % K);
    } else if (cfg.grouping == 2) {
        // Same seed material and engine as the reference, so the permutation
        // (libstdc++ std::shuffle over mt19937_64) is identical.
        std::seed_seq seq{static_cast<std::uint32_t>(cfg.seed),
                          static_cast<std::uint32_t>(cfg.seed >> 32),
                          static_cast<std::uint32_t>(subspace), static_cast<std::uint32_t>(base_id)};
        std::mt19937_64 eng(seq);
        std::vector<std::uint32_t> perm(m);
        std::iota(perm.begin(), perm.end(), 0u);
        std::shuffle(perm.begin(), perm.end(), eng);
        for (std::size_t p = 0; p < m; ++p) out[perm[p]] = static_cast<std::uint32_t>(p / r);
    } else {
        out = pca_tree(pts, m, w, cfg.r);
    }
    return out;
}

// index.cpp:104-137 — `rows` lists the member rows of the local block.
Encl enclose(const float* pts, int w, const std::vector<std::size_t>& rows, int kind) {
    if (rows.empty()) throw std::invalid_argument("enclose_group: empty group");
    Encl e;
    e.kind = kind;
    auto box = [&](std::vector<float>& lo, std::vector<float>& hi) {
        lo.assign(pts + rows[0] * w, pts + rows[0] * w + w);
        hi = lo;
        for (std::size_t i = 1; i < rows.size(); ++i) {
            const float* p = pts + rows[i] * w;
            for (int c = 0; c < w; ++c) {
                lo[c] = std::min(lo[c], p[c]);
                hi[c] = std::max(hi[c], p[c]);
            }
        }
    };
    if (kind == kAabb) {
        box(e.lo, e.hi);
        return e;
    }
    e.center.assign(w, 0.0f);
    if (kind == kBall) {
        std::vector<double> sum(w, 0.0);
        for (std::size_t row : rows)
            for (int c = 0; c < w; ++c) sum[c] += static_cast<double>(pts[row * w + c]);
        for (int c = 0; c < w; ++c)
            e.center[c] = static_cast<float>(sum[c] / static_cast<double>(rows.size()));
    } else {
        std::vector<float> lo, hi;
        box(lo, hi);
        for (int c = 0; c < w; ++c) e.center[c] = 0.5f * (lo[c] + hi[c]);
    }
    float rad = 0.0f;
    std::vector<float> diff(w);
    for (std::size_t row : rows) {
        for (int c = 0; c < w; ++c) diff[c] = pts[row * w + c] - e.center[c];
        rad = std::max(rad, nnorm(diff.data(), w));
    }
    if (rad > 0.0f) rad = std::nextafter(rad, kInf);  // one ulp of containment headroom
    e.radius = rad;
    return e;
}

// index.cpp:139-168
void push_gate(Sub& sub, Encl e, const std::vector<Id>& members) {
    double b = 0.0;
    if (e.kind == kAabb) {
        const std::size_t w = e.lo.size();
        if (sub.glo.empty()) {
            sub.glo.resize(w);
            sub.ghi.resize(w);
        }
        double sq = 0.0;
        for (std::size_t c = 0; c < w; ++c) {
            sub.glo[c].push_back(e.lo[c]);
            sub.ghi[c].push_back(e.hi[c]);
            const double a = std::max(std::abs(double(e.lo[c])), std::abs(double(e.hi[c])));
            sq += a * a;
        }
        b = std::sqrt(sq);
    } else {
        const std::size_t w = e.center.size();
        if (sub.gc.empty()) sub.gc.resize(w);
        for (std::size_t c = 0; c < w; ++c) sub.gc[c].push_back(e.center[c]);
        sub.grad.push_back(e.radius);
        // Eigen's center.norm() in the reference; the sequential fp32 norm here
        // can differ in the last bit, which moves only derive_subspace_thresholds'
        // float-safety slack (candidate sets, never final sets).
        b = double(nnorm(e.center.data(), static_cast<std::ptrdiff_t>(w))) + double(e.radius);
    }
    sub.norm_bound = std::max(sub.norm_bound, b);
    sub.mids.insert(sub.mids.end(), members.begin(), members.end());
    sub.moff.push_back(static_cast<std::uint32_t>(sub.mids.size()));
    sub.encl.push_back(std::move(e));
}

// index.cpp:172-209 — group keys [first, first+count) in every subspace.
void index_range(Index& idx, const Store& st, Id first, std::size_t count) {
    for (int s = 0; s < idx.lay.S; ++s) {
        const int w = idx.lay.width(s), b0 = idx.lay.begin(s);
        std::vector<float> blk(count * static_cast<std::size_t>(w));
        for (std::size_t j = 0; j < count; ++j)
            std::memcpy(&blk[j * w], st.key(first + static_cast<Id>(j)) + b0, sizeof(float) * w);
        const auto local = group_keys(blk.data(), count, w, idx.cfg, s, first);
        Sub& sub = idx.subs[s];
        const std::uint32_t gbase = static_cast<std::uint32_t>(sub.groups());
        std::uint32_t ng = 0;
        for (auto a : local) ng = std::max(ng, a + 1);
        std::vector<std::vector<std::size_t>> rows(ng);
        for (std::size_t j = 0; j < count; ++j) rows[local[j]].push_back(j);
        for (std::size_t j = 0; j < count; ++j) sub.assign.push_back(gbase + local[j]);
        for (std::uint32_t g = 0; g < ng; ++g) {
            std::vector<Id> mem;
            mem.reserve(rows[g].size());
            for (std::size_t j : rows[g]) mem.push_back(first + static_cast<Id>(j));
            push_gate(sub, enclose(blk.data(), w, rows[g], idx.cfg.enclosure), mem);
        }
    }
    idx.indexed = static_cast<std::int64_t>(first + count);
}

// index.cpp:213-222
Index build_index(const Store& st, const Config& cfg) {
    cfg.validate(st.d);
    if (st.n == 0) throw std::invalid_argument("build_index: empty store");
    Index idx;
    idx.lay = Slices(st.d, cfg.S);
    idx.cfg = cfg;
    idx.subs.resize(cfg.S);
    index_range(idx, st, 0, static_cast<std::size_t>(st.n));
    return idx;
}

// index.cpp:224-232
void append_index(Index& idx, const Store& st, Id first, std::size_t count) {
    if (static_cast<std::int64_t>(first) != idx.indexed)
        throw std::invalid_argument("append_to_index: ids must extend the indexed range");
    if (count == 0) return;
    if (static_cast<std::int64_t>(first + count) > st.n)
        throw std::invalid_argument("append_to_index: range exceeds store");
    index_range(idx, st, first, count);
}

// ------------------------------------------------------------------- query

struct Stats {
    std::vector<std::int64_t> per_sub;
    std::int64_t groups = 0, scanned = 0;
    double f_scan = 0.0, gate_cost = 0.0;
    int stop_depth = -1;
    double stop_upper = 0.0;
};

struct Cands {
    std::vector<Id> live;
    Stats st;
};

// query.cpp:11-20
std::vector<Id> brute(const Store& st, const float* q, float tau, std::int64_t limit) {
    if (limit > st.n) throw std::invalid_argument("brute_force_range: limit > n");
    std::vector<Id> out;
    for (std::int64_t j = 0; j < limit; ++j)
        if (ndot(q, st.key(static_cast<Id>(j)), st.d) >= tau) out.push_back(static_cast<Id>(j));
    return out;
}

// query.cpp:22-31
std::vector<Id> exact(const Store& st, const std::vector<Id>& cand, const float* q, float tau) {
    std::vector<Id> out;
    out.reserve(cand.size());
    for (Id j : cand)
        if (ndot(q, st.key(j), st.d) >= tau) out.push_back(j);
    std::sort(out.begin(), out.end());
    return out;
}

std::vector<Id> mask_ids(const std::vector<std::uint8_t>& m) {  // query.cpp:35-40
    std::vector<Id> out;
    for (std::size_t j = 0; j < m.size(); ++j)
        if (m[j]) out.push_back(static_cast<Id>(j));
    return out;
}

// query.cpp:47-68 — same per-group float op order as the single-enclosure
// bound (core.hpp:95-105): 0 + term_0 + term_1 + ..., radius term last.
void bounds_of(const Sub& sub, const float* qs, int w, int kind, float* out) {
    const std::size_t K = sub.groups();
    std::fill(out, out + K, 0.0f);
    if (kind == kAabb) {
        for (int c = 0; c < w; ++c) {
            const float qc = qs[c];
            const float* lo = sub.glo[c].data();
            const float* hi = sub.ghi[c].data();
            for (std::size_t i = 0; i < K; ++i) out[i] += std::max(qc * lo[i], qc * hi[i]);
        }
        return;
    }
    for (int c = 0; c < w; ++c) {
        const float qc = qs[c];
        const float* ctr = sub.gc[c].data();
        for (std::size_t i = 0; i < K; ++i) out[i] += qc * ctr[i];
    }
    const float qn = nnorm(qs, w);
    for (std::size_t i = 0; i < K; ++i) out[i] += sub.grad[i] * qn;
}

// query.cpp:70-78
void finalize(Stats& st, const Index& idx) {
    st.groups = 0;
    for (auto g : st.per_sub) st.groups += g;
    st.f_scan = idx.indexed ? double(st.scanned) / double(idx.indexed) : 0.0;
    const int gate = idx.cfg.enclosure == kAabb ? 2 : 1;
    st.gate_cost = double(gate) * double(st.groups) / idx.cfg.r;
}

// query.cpp:82-117 — Query 1: AND across subspaces of per-subspace passes.
Cands full_subspace(const Index& idx, const float* q, const std::vector<float>& tau_s) {
    if (static_cast<int>(tau_s.size()) != idx.lay.S)
        throw std::invalid_argument("query_full_subspace: tau_subspace length != S");
    const std::size_t n = static_cast<std::size_t>(idx.indexed);
    std::vector<std::uint8_t> live(n, 1), pass(n);
    Cands res;
    res.st.per_sub.assign(idx.lay.S, 0);
    std::vector<float> b;
    for (int s = 0; s < idx.lay.S; ++s) {
        const Sub& sub = idx.subs[s];
        std::fill(pass.begin(), pass.end(), 0);
        res.st.per_sub[s] = static_cast<std::int64_t>(sub.groups());
        b.resize(sub.groups());
        bounds_of(sub, q + idx.lay.begin(s), idx.lay.width(s), idx.cfg.enclosure, b.data());
        for (std::size_t g = 0; g < b.size(); ++g) {
            if (b[g] < tau_s[s]) continue;  // ties intersect
            for (std::uint32_t t = sub.moff[g]; t < sub.moff[g + 1]; ++t) pass[sub.mids[t]] = 1;
        }
        for (std::size_t j = 0; j < n; ++j) live[j] &= pass[j];
    }
    res.live = mask_ids(live);
    res.st.scanned = static_cast<std::int64_t>(res.live.size());
    finalize(res.st, idx);
    return res;
}

// query.cpp:123-132 — monotone float <-> uint32 map (ascending floats give
// ascending keys).
inline std::uint32_t order_key(float x) {
    std::uint32_t u;
    std::memcpy(&u, &x, 4);
    return (u & 0x80000000u) ? ~u : (u | 0x80000000u);
}
inline float order_key_inv(std::uint32_t t) {
    const std::uint32_t u = (t & 0x80000000u) ? (t ^ 0x80000000u) : ~t;
    float x;
    std::memcpy(&x, &u, 4);
    return x;
}

// query.cpp:134-146 — descending sort of the uint32 keys (byte-radix here;
// only the resulting order matters).
void sort_desc(std::vector<std::uint32_t>& v, std::vector<std::uint32_t>& tmp) {
    tmp.resize(v.size());
    for (int shift = 0; shift < 32; shift += 8) {
        std::size_t cnt[257] = {};
        for (std::uint32_t t : v) ++cnt[((t >> shift) & 0xFFu) + 1];
        for (int i = 1; i <= 256; ++i) cnt[i] += cnt[i - 1];
        for (std::uint32_t t : v) tmp[cnt[(t >> shift) & 0xFFu]++] = t;
        v.swap(tmp);
    }
    std::reverse(v.begin(), v.end());
}

// query.cpp:160-200 — lazily materialized descending bound ranking: a stride
// sample of <= 256 bounds sets a cutoff, one ascending-id gather keeps every
// group at or above it, and only the gathered values are sorted.
struct Ranking {
    std::vector<float> bound, sample;
    std::vector<std::uint32_t> ids, keys, sorted;
    std::size_t filled = 0;

    void prepare() {
        const std::size_t stride = std::max<std::size_t>(1, bound.size() / 256);
        sample.clear();
        for (std::size_t i = 0; i < bound.size(); i += stride) sample.push_back(bound[i]);
        std::sort(sample.begin(), sample.end(), std::greater<float>());
    }

    void grow(std::size_t want, std::vector<std::uint32_t>& tmp) {
        const std::size_t K = bound.size();
        want = std::min(want, K);
        if (filled >= want) return;
        std::size_t pos = want * sample.size() / K;
        pos += pos / 2 + 8;
        while (true) {
            const bool all = pos >= sample.size();
            const float cut = all ? -kInf : sample[pos];
            ids.clear();
            keys.clear();
            for (std::uint32_t g = 0; g < K; ++g)
                if (bound[g] >= cut) {
                    ids.push_back(g);
                    keys.push_back(order_key(bound[g]));
                }
            if (ids.size() >= want || all) break;
            pos = pos * 2 + 8;
        }
        sorted = keys;
        sort_desc(sorted, tmp);
        filled = sorted.size();
    }
};

// query.cpp:204-303 — Query 2, the threshold-algorithm scan. U(d) sums the
// d-th ranked bound of every subspace in double; the scan halts at the first
// d with U(d) < tau and the live set is the union of each subspace's top-d
// prefix (bound descending, group id ascending on ties).
Cands ta_scan(const Index& idx, const float* q, float tau) {
    const int S = idx.lay.S;
    const std::size_t n = static_cast<std::size_t>(idx.indexed);
    Cands res;
    res.st.per_sub.assign(S, 0);
    std::vector<Ranking> rk(S);
    std::size_t maxg = 0;
    for (int s = 0; s < S; ++s) {
        const Sub& sub = idx.subs[s];
        rk[s].bound.resize(sub.groups());
        bounds_of(sub, q + idx.lay.begin(s), idx.lay.width(s), idx.cfg.enclosure,
                  rk[s].bound.data());
        rk[s].prepare();
        res.st.per_sub[s] = static_cast<std::int64_t>(sub.groups());
        maxg = std::max(maxg, sub.groups());
    }
    std::vector<std::uint32_t> tmp;
    std::size_t prefix = std::min<std::size_t>(1024, maxg);
    for (auto& r : rk) r.grow(prefix, tmp);

    std::size_t halt = 0;
    double halt_upper = 0.0;
    for (std::size_t dd = 1; dd <= maxg; ++dd) {
        if (dd > prefix) {
            prefix = std::min(prefix * 2, maxg);
            for (auto& r : rk) r.grow(prefix, tmp);
        }
        double u = 0.0;
        for (int s = 0; s < S; ++s)
            if (dd <= rk[s].filled) u += static_cast<double>(order_key_inv(rk[s].sorted[dd - 1]));
        if (u < static_cast<double>(tau)) {
            halt = dd;
            halt_upper = u;
            break;
        }
    }

    std::vector<std::uint8_t> live(n, 0);
    std::size_t nlive = 0;
    for (int s = 0; s < S; ++s) {
        const Sub& sub = idx.subs[s];
        auto mark = [&](std::uint32_t g) {
            for (std::uint32_t t = sub.moff[g]; t < sub.moff[g + 1]; ++t) {
                const Id j = sub.mids[t];
                if (!live[j]) {
                    live[j] = 1;
                    ++nlive;
                }
            }
        };
        const std::size_t K = sub.groups();
        const std::size_t depth = halt == 0 ? K : std::min(halt, K);
        if (depth == K) {
            for (std::uint32_t g = 0; g < K; ++g) mark(g);
            continue;
        }
        const Ranking& r = rk[s];
        const std::uint32_t edge = r.sorted[depth - 1];
        std::size_t above = 0;
        while (above < depth && r.sorted[above] > edge) ++above;
        std::size_t ties = depth - above;
        for (std::size_t i = 0; i < r.ids.size(); ++i) {
            if (r.keys[i] > edge) {
                mark(r.ids[i]);
            } else if (r.keys[i] == edge && ties > 0) {
                mark(r.ids[i]);
                --ties;
            }
        }
    }
    if (halt > 0) {
        res.st.stop_depth = static_cast<int>(halt);
        res.st.stop_upper = halt_upper;
    }
    res.live = mask_ids(live);
    res.st.scanned = static_cast<std::int64_t>(nlive);
    finalize(res.st, idx);
    return res;
}

// query.cpp:305-336
std::vector<float> subspace_taus(const Index& idx, const float* q, float tau) {
    const int S = idx.lay.S;
    std::vector<double> peak(S, 0.0);
    double nb2 = 0.0;
    std::vector<float> b;
    for (int s = 0; s < S; ++s) {
        const Sub& sub = idx.subs[s];
        b.resize(sub.groups());
        bounds_of(sub, q + idx.lay.begin(s), idx.lay.width(s), idx.cfg.enclosure, b.data());
        double m = -std::numeric_limits<double>::infinity();
        for (float f : b) m = std::max(m, static_cast<double>(f));
        peak[s] = m;
        nb2 += sub.norm_bound * sub.norm_bound;
    }
    const double eps = std::numeric_limits<float>::epsilon();
    // Reference uses Eigen q.norm(); see push_gate on last-bit differences.
    const double slack =
        S == 1 ? 0.0 : 4.0 * idx.lay.d * eps * double(nnorm(q, idx.lay.d)) * std::sqrt(nb2);
    double total = 0.0;
    for (int s = 0; s < S; ++s) total += peak[s];
    std::vector<float> out(S);
    for (int s = 0; s < S; ++s) out[s] = static_cast<float>(double(tau) - (total - peak[s]) - slack);
    return out;
}

struct Attn {
    std::vector<Id> ids;
    std::vector<float> w;
    std::vector<float> out;
};

// query.cpp:338-371 — three passes in ascending token order: scores + max,
// exp + denominator, normalize + axpy.
bool attend(const Store& st, const Id* buf, std::size_t nbuf, const Id* sel, std::size_t nsel,
            const float* q, float scale, Attn& res) {
    std::vector<Id> tok(sel, sel + nsel);
    tok.insert(tok.end(), buf, buf + nbuf);
    std::sort(tok.begin(), tok.end());
    tok.erase(std::unique(tok.begin(), tok.end()), tok.end());
    if (tok.empty()) return false;
    for (Id j : tok)
        if (static_cast<std::int64_t>(j) >= st.n)
            throw std::out_of_range("sparse_attention: id out of range");
    const int d = st.d;
    std::vector<float> sc(tok.size());
    float mx = -kInf;
    for (std::size_t i = 0; i < tok.size(); ++i) {
        sc[i] = scale * ndot(q, st.key(tok[i]), d);
        mx = std::max(mx, sc[i]);
    }
    res.w.resize(tok.size());
    float den = 0.0f;
    for (std::size_t i = 0; i < tok.size(); ++i) {
        res.w[i] = std::exp(sc[i] - mx);
        den += res.w[i];
    }
    res.out.assign(d, 0.0f);
    for (std::size_t i = 0; i < tok.size(); ++i) {
        res.w[i] /= den;
        const float* v = st.value(tok[i]);
        for (int c = 0; c < d; ++c) res.out[c] += res.w[i] * v[c];
    }
    res.ids = std::move(tok);
    return true;
}

}  // namespace

// ------------------------------------------------------------- LouverCache

struct lvo_cache {
    Store store;
    Config cfg;
    std::int64_t B = 128;
    Index idx;
    bool has_index = false;
    std::int64_t flushes = 0;

    std::int64_t pending() const { return store.n - (has_index ? idx.indexed : 0); }

    // cache.cpp:12-22
    bool flush() {
        const std::int64_t p = pending();
        if (p == 0) return false;
        if (!has_index) {
            idx = build_index(store, cfg);
            has_index = true;
        } else {
            append_index(idx, store, static_cast<Id>(idx.indexed), static_cast<std::size_t>(p));
        }
        ++flushes;
        return true;
    }

    // cache.cpp:7-10
    void push(const float* k, const float* v) {
        store.append(k, v);
        if (pending() >= B) flush();
    }
};

namespace {

template <typename F>
int guarded(F&& f) {
    try {
        return f();
    } catch (const std::invalid_argument& e) {
        g_error = e.what();
        return LVO_EINVAL;
    } catch (const std::out_of_range& e) {
        g_error = e.what();
        return LVO_ERANGE;
    } catch (const std::exception& e) {
        g_error = e.what();
        return LVO_EINVAL;
    }
}

Store view_store(const float* keys, const float* values, std::int64_t n, int d) {
    if (d < 1) throw std::invalid_argument("KeyStore: d >= 1 required");
    Store st;
    st.d = d;
    st.n = n;
    st.K.assign(keys, keys + static_cast<std::size_t>(n) * d);
    if (values) st.V.assign(values, values + static_cast<std::size_t>(n) * d);
    return st;
}

void copy_ids(const std::vector<Id>& v, std::uint32_t* out, std::int64_t cap, std::int64_t* count) {
    if (count) *count = static_cast<std::int64_t>(v.size());
    if (out) std::memcpy(out, v.data(), sizeof(Id) * std::min<std::int64_t>(cap, v.size()));
}

}  // namespace

extern "C" {

const char* lvo_last_error(void) { return g_error.c_str(); }

float lvo_dot(const float* a, const float* b, int64_t len) { return ndot(a, b, len); }

int lvo_brute_force_range(const float* keys, int64_t n, int d, const float* q, float tau,
                          int64_t limit, uint32_t* out_ids, int64_t cap, int64_t* count) {
    return guarded([&] {
        if (limit > n) throw std::invalid_argument("brute_force_range: limit > n");
        std::vector<Id> out;
        for (int64_t j = 0; j < limit; ++j)
            if (ndot(q, keys + static_cast<std::size_t>(j) * d, d) >= tau)
                out.push_back(static_cast<Id>(j));
        copy_ids(out, out_ids, cap, count);
        return LVO_OK;
    });
}

int lvo_exact_check(const float* keys, int64_t n, int d, const uint32_t* cand, int64_t ncand,
                    const float* q, float tau, uint32_t* out_ids, int64_t* count) {
    return guarded([&] {
        Store st;
        st.d = d;
        st.n = n;
        st.K.assign(keys, keys + static_cast<std::size_t>(n) * d);
        std::vector<Id> c(cand, cand + ncand);
        for (Id j : c)
            if (static_cast<int64_t>(j) >= n) throw std::out_of_range("exact_check: id out of range");
        const auto out = exact(st, c, q, tau);
        copy_ids(out, out_ids, ncand, count);
        return LVO_OK;
    });
}

int lvo_layout(int d, int S, int* offsets) {
    return guarded([&] {
        const Slices L(d, S);
        for (int s = 0; s <= S; ++s) offsets[s] = L.off[s];
        return LVO_OK;
    });
}

int lvo_scores(const float* keys, int64_t n, int d, const float* q, float* out) {
    for (int64_t j = 0; j < n; ++j) out[j] = ndot(q, keys + static_cast<std::size_t>(j) * d, d);
    return LVO_OK;
}

float lvo_kth_score(const float* keys, int64_t n, int d, const float* q, int64_t k) {
    std::vector<float> s(static_cast<std::size_t>(n));
    lvo_scores(keys, n, d, q, s.data());
    std::nth_element(s.begin(), s.begin() + (k - 1), s.end(), std::greater<float>());
    return s[static_cast<std::size_t>(k - 1)];
}

// threshold.hpp:29-50 — Algorithm R with the reference's engine and distribution
struct lvo_reservoir {
    std::size_t capacity;
    std::vector<uint32_t> ids;
    std::size_t seen = 0;
    std::mt19937_64 rng;
};

lvo_reservoir* lvo_reservoir_create(int64_t capacity, uint64_t seed) {
    if (capacity < 1) return nullptr;  // threshold.hpp:33
    auto* r = new lvo_reservoir{static_cast<std::size_t>(capacity), {}, 0, std::mt19937_64(seed)};
    return r;
}

void lvo_reservoir_destroy(lvo_reservoir* r) { delete r; }

// threshold.cpp:40-55
int64_t lvo_reservoir_update(lvo_reservoir* r, uint32_t id) {
    ++r->seen;
    if (r->ids.size() < r->capacity) {
        r->ids.push_back(id);
        return static_cast<int64_t>(r->ids.size() - 1);
    }
    std::uniform_int_distribution<std::size_t> pick(0, r->seen - 1);
    const std::size_t slot = pick(r->rng);
    if (slot < r->capacity) {
        r->ids[slot] = id;
        return static_cast<int64_t>(slot);
    }
    return -1;
}

int64_t lvo_reservoir_size(const lvo_reservoir* r) { return static_cast<int64_t>(r->ids.size()); }
int64_t lvo_reservoir_seen(const lvo_reservoir* r) { return static_cast<int64_t>(r->seen); }
void lvo_reservoir_ids(const lvo_reservoir* r, uint32_t* out) {
    if (!r->ids.empty()) std::memcpy(out, r->ids.data(), sizeof(uint32_t) * r->ids.size());
}

// threshold.cpp:63-103 (OracleConfig::validate: threshold.hpp:17-22)
int lvo_estimate_tau(const float* keys, int64_t n_, int d, const float* q, int variant, int m,
                     double alpha, float* tau) {
    return guarded([&] {
        if (variant == 1 && m < 1) throw std::invalid_argument("OracleConfig: m >= 1 required");
        if (variant == 4 && !(alpha > 0.0 && alpha < 1.0))
            throw std::invalid_argument("OracleConfig: 0 < alpha < 1 required");
        if (variant < 0 || variant > 4) throw std::invalid_argument("unknown oracle variant");
        const std::size_t n = static_cast<std::size_t>(n_);
        if (n == 0) throw std::invalid_argument("estimate_tau: empty reservoir");
        std::vector<float> scores(n);
        lvo_scores(keys, n_, d, q, scores.data());
        std::sort(scores.begin(), scores.end(), std::greater<>());
        float r = 0.0f;
        switch (variant) {
            case 0:
                r = scores[0];
                break;
            case 1:
                if (n < static_cast<std::size_t>(m))
                    throw std::invalid_argument("estimate_tau: sample smaller than topk rank");
                r = scores[static_cast<std::size_t>(m - 1)];
                break;
            case 2: {
                if (n < 2) throw std::invalid_argument("estimate_tau: gap needs >= 2 samples");
                std::size_t best = 0;
                float best_gap = scores[0] - scores[1];
                for (std::size_t i = 1; i + 1 < n; ++i) {
                    const float gap = scores[i] - scores[i + 1];
                    if (gap > best_gap) {
                        best_gap = gap;
                        best = i;
                    }
                }
                r = scores[best];
                break;
            }
            case 3: {
                double mean = 0.0;
                for (float s : scores) mean += s;
                mean /= static_cast<double>(n);
                r = static_cast<float>((double(scores[0]) + mean) / 2.0);
                break;
            }
            case 4: {
                const auto idx = static_cast<std::size_t>(std::min<double>(
                    std::ceil((1.0 - alpha) * static_cast<double>(n)), static_cast<double>(n - 1)));
                r = scores[n - 1 - idx];
                break;
            }
        }
        *tau = r;
        return LVO_OK;
    });
}

int lvo_sparse_attention(const float* keys, const float* values, int64_t n, int d,
                         const uint32_t* buffer_ids, int64_t nbuf, const uint32_t* sel_ids,
                         int64_t nsel, const float* q, float scale, float* out, float* weights,
                         int64_t* ntok) {
    return guarded([&] {
        const Store st = view_store(keys, values, n, d);
        Attn a;
        if (!attend(st, buffer_ids, static_cast<std::size_t>(nbuf), sel_ids,
                    static_cast<std::size_t>(nsel), q, scale, a)) {
            if (ntok) *ntok = 0;
            return LVO_EMPTY;
        }
        std::memcpy(out, a.out.data(), sizeof(float) * d);
        if (weights) std::memcpy(weights, a.w.data(), sizeof(float) * a.w.size());
        if (ntok) *ntok = static_cast<int64_t>(a.ids.size());
        return LVO_OK;
    });
}

int lvo_cache_create(int d, const lvo_build_config* cfg, int64_t buffer_capacity,
                     lvo_cache** out) {
    return guarded([&] {
        const Config c = to_config(cfg);
        if (d < 1) throw std::invalid_argument("KeyStore: d >= 1 required");
        c.validate(d);  // cache.hpp:26
        if (buffer_capacity < 1)
            throw std::invalid_argument("LouverCache: buffer capacity >= 1 required");
        auto cache = std::make_unique<lvo_cache>();
        cache->store.d = d;
        cache->cfg = c;
        cache->B = buffer_capacity;
        *out = cache.release();
        return LVO_OK;
    });
}

int lvo_cache_adopt(const float* keys, const float* values, int64_t n, int d,
                    const lvo_build_config* cfg, int64_t buffer_capacity, lvo_cache** out) {
    return guarded([&] {
        if (buffer_capacity < 1)
            throw std::invalid_argument("LouverCache: buffer capacity >= 1 required");
        auto cache = std::make_unique<lvo_cache>();
        cache->store = view_store(keys, values, n, d);
        cache->cfg = to_config(cfg);
        cache->B = buffer_capacity;
        if (n > 0) {  // cache.hpp:35
            cache->idx = build_index(cache->store, cache->cfg);
            cache->has_index = true;
        }
        *out = cache.release();
        return LVO_OK;
    });
}

void lvo_cache_destroy(lvo_cache* c) { delete c; }

int lvo_cache_push_key(lvo_cache* c, const float* k, const float* v) {
    return guarded([&] {
        c->push(k, v);
        return LVO_OK;
    });
}

int lvo_cache_flush(lvo_cache* c) {
    return guarded([&] { return c->flush() ? LVO_OK : LVO_EMPTY; });
}

int64_t lvo_cache_n(const lvo_cache* c) { return c->store.n; }
int64_t lvo_cache_indexed_count(const lvo_cache* c) { return c->has_index ? c->idx.indexed : 0; }
int64_t lvo_cache_flush_count(const lvo_cache* c) { return c->flushes; }

int64_t lvo_cache_groups(const lvo_cache* c, int s) {
    if (!c->has_index || s < 0 || s >= static_cast<int>(c->idx.subs.size())) return 0;
    return static_cast<int64_t>(c->idx.subs[s].groups());
}

int64_t lvo_cache_group_members(const lvo_cache* c, int s, int64_t g, uint32_t* out, int64_t cap) {
    if (!c->has_index) return 0;
    const Sub& sub = c->idx.subs[s];
    const int64_t cnt = sub.moff[g + 1] - sub.moff[g];
    for (int64_t i = 0; i < std::min(cnt, cap); ++i) out[i] = sub.mids[sub.moff[g] + i];
    return cnt;
}

int lvo_cache_candidates(const lvo_cache* c, const float* q, float tau, const float* tau_s, int algo,
                         uint32_t* ids, int64_t cap, int64_t* n, lvo_stats* stats) {
    return guarded([&] {
        if (!c->has_index) throw std::invalid_argument("candidates: no index");
        Cands cand;
        if (algo == 0) {
            if (!tau_s) throw std::invalid_argument("query_full_subspace: tau_subspace required");
            cand = full_subspace(c->idx, q, std::vector<float>(tau_s, tau_s + c->idx.subs.size()));
        } else {
            cand = ta_scan(c->idx, q, tau);
        }
        copy_ids(cand.live, ids, cap, n);
        if (stats) {
            stats->groups_tested = cand.st.groups;
            stats->keys_scanned = cand.st.scanned;
            stats->f_scan = cand.st.f_scan;
            stats->gate_cost_equiv = cand.st.gate_cost;
            stats->ta_stop_depth = cand.st.stop_depth;
            stats->ta_stop_upper = cand.st.stop_upper;
        }
        return LVO_OK;
    });
}

int lvo_cache_thresholds(const lvo_cache* c, const float* q, float tau, float* out) {
    return guarded([&] {
        if (!c->has_index) throw std::invalid_argument("thresholds: no index");
        const auto t = subspace_taus(c->idx, q, tau);
        std::memcpy(out, t.data(), sizeof(float) * t.size());
        return LVO_OK;
    });
}

int lvo_cache_subspace(const lvo_cache* c, int s, uint32_t* assign, uint32_t* moff, uint32_t* mids, float* a,
                       float* b, float* radii, double* norm_bound) {
    return guarded([&] {
        if (!c->has_index || s < 0 || s >= (int)c->idx.subs.size()) throw std::out_of_range("subspace");
        const Sub& sb = c->idx.subs[s];
        const std::size_t K = sb.groups();
        if (assign) std::memcpy(assign, sb.assign.data(), sizeof(uint32_t) * sb.assign.size());
        if (moff) std::memcpy(moff, sb.moff.data(), sizeof(uint32_t) * sb.moff.size());
        if (mids) std::memcpy(mids, sb.mids.data(), sizeof(uint32_t) * sb.mids.size());
        const bool box = c->cfg.enclosure == kAabb;
        const auto& A = box ? sb.glo : sb.gc;
        for (std::size_t i = 0; a && i < A.size(); ++i) std::memcpy(a + i * K, A[i].data(), sizeof(float) * K);
        for (std::size_t i = 0; b && box && i < sb.ghi.size(); ++i) std::memcpy(b + i * K, sb.ghi[i].data(), sizeof(float) * K);
        if (radii && !box) std::memcpy(radii, sb.grad.data(), sizeof(float) * K);
        if (norm_bound) *norm_bound = sb.norm_bound;
        return LVO_OK;
    });
}

// cache.cpp:30-70
int lvo_cache_query(const lvo_cache* c, const float* q, float tau, float scale, int algo,
                    int strict, uint32_t* selected, int64_t* nsel, uint32_t* retrieved,
                    int64_t* nret, int64_t cap, float* attn_out, int* has_attn,
                    lvo_stats* stats) {
    return guarded([&] {
        const Store& st = c->store;
        const int d = st.d;
        // query.hpp:17-19
        const float eff_scale = scale != 0.0f ? scale : float(1.0 / std::sqrt(double(d)));
        std::vector<Id> sel;
        Stats s;
        const std::int64_t indexed = c->has_index ? c->idx.indexed : 0;
        if (indexed > 0) {
            Cands cand = algo == 0 ? full_subspace(c->idx, q, subspace_taus(c->idx, q, tau))
                                   : ta_scan(c->idx, q, tau);
            s = cand.st;
            sel = exact(st, cand.live, q, tau);
        }
        std::vector<Id> ret = sel;
        for (std::int64_t j = indexed; j < st.n; ++j) {  // dense buffer scan
            ret.push_back(static_cast<Id>(j));
            if (ndot(q, st.key(static_cast<Id>(j)), d) >= tau) sel.push_back(static_cast<Id>(j));
        }
        if (st.n > 0) {
            s.scanned += st.n - indexed;
            s.f_scan = double(s.scanned) / double(st.n);
        } else {
            s.f_scan = 1.0;
        }
        const std::vector<Id>& att = strict ? sel : ret;
        Attn a;
        const bool ok = attend(st, nullptr, 0, att.data(), att.size(), q, eff_scale, a);
        if (has_attn) *has_attn = ok ? 1 : 0;
        if (ok && attn_out) std::memcpy(attn_out, a.out.data(), sizeof(float) * d);
        copy_ids(sel, selected, cap, nsel);
        copy_ids(ret, retrieved, cap, nret);
        if (stats) {
            stats->groups_tested = s.groups;
            stats->keys_scanned = s.scanned;
            stats->f_scan = s.f_scan;
            stats->gate_cost_equiv = s.gate_cost;
            stats->ta_stop_depth = s.stop_depth;
            stats->ta_stop_upper = s.stop_upper;
        }
        return LVO_OK;
    });
}

int lvo_balanced_pca_tree(const float* points, int64_t m, int w, int r, uint32_t* out) {
    return guarded([&] {
        const auto a = pca_tree(points, static_cast<std::size_t>(m), w, r);
        std::memcpy(out, a.data(), sizeof(uint32_t) * a.size());
        return LVO_OK;
    });
}

int lvo_assign_groups(const float* points, int64_t m, int w, const lvo_build_config* cfg,
                      int subspace, uint32_t base_id, uint32_t* out) {
    return guarded([&] {
        const auto a = group_keys(points, static_cast<std::size_t>(m), w, to_config(cfg),
                                  subspace, base_id);
        std::memcpy(out, a.data(), sizeof(uint32_t) * a.size());
        return LVO_OK;
    });
}

int lvo_enclose_group(const float* points, int64_t m, int w, int kind, float* center,
                      float* radius, float* lo, float* hi) {
    return guarded([&] {
        std::vector<std::size_t> rows(static_cast<std::size_t>(m));
        std::iota(rows.begin(), rows.end(), std::size_t{0});
        const Encl e = enclose(points, w, rows, kind);
        if (kind == kAabb) {
            std::memcpy(lo, e.lo.data(), sizeof(float) * w);
            std::memcpy(hi, e.hi.data(), sizeof(float) * w);
        } else {
            std::memcpy(center, e.center.data(), sizeof(float) * w);
            *radius = e.radius;
        }
        return LVO_OK;
    });
}

}  // extern "C"
