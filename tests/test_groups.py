"""Grouped index on the device (lv_config.group_index, csrc/louver_groups.cu) against the
reference's own index.cpp / query.cpp: the reference library compiled here (oracle/_ref,
its unmodified sources) when present, else the oracle restatement.

Every BuildConfig axis is covered — GroupingStrategy (contiguous, interleaved, random,
PCA tree), EnclosureKind (ball, AABB, span ball), S with uneven subspace widths — on the
reference's decode-trace key law and on i.i.d. keys, for a prefill build and for a cache
filled through pushes (append_to_index per flush). Bit-exact: assignments, member lists,
packed gate arrays, radii, norm bounds, the candidate sets and statistics of query_ta and
query_full_subspace, derive_subspace_thresholds, and the LVIX snapshot bytes
(test_index.cpp:59-134, test_query.cpp:74-160, test_cache.cpp:102-121, test_io.cpp:74-123).
"""
import os
import tempfile

import numpy as np
import pytest

from oracle import pyoracle as rest
from paper_2605_06763_b200 import (BuildConfig, FilterAlgo, LouverCache, QueryRequest, derive_subspace_thresholds,
                                   query_full_subspace, query_ta, synth)

pytestmark = pytest.mark.gpu

REF = rest.reference_module() or rest

CONFIGS = [
    (4, 4, "pca_tree", "ball", 0),       # the reference default (index.hpp:10-15)
    (4, 4, "pca_tree", "aabb", 0),
    (2, 8, "pca_tree", "span_ball", 0),
    (3, 5, "pca_tree", "ball", 0),       # uneven widths (core.hpp:41-50)
    (1, 16, "contiguous", "aabb", 0),
    (4, 4, "interleaved", "ball", 0),
    (4, 6, "random", "ball", 12345),
    (8, 3, "random", "aabb", 7),
]


def keys_of(law, n, d, seed):
    if law == "trace":
        return synth.keys(n, d, seed), synth.keys(n, d, seed + 1)
    rng = np.random.default_rng(seed)
    return rng.standard_normal((n, d)).astype(np.float32), rng.standard_normal((n, d)).astype(np.float32)


def widths(d, S):
    return [d // S + (1 if s < d % S else 0) for s in range(S)]


def same_f32(a, b):
    return np.array_equal(np.asarray(a, np.float32).view(np.uint32), np.asarray(b, np.float32).view(np.uint32))


def check_index(dev, ref, d, S, enclosure):
    for s, w in enumerate(widths(d, S)):
        got = dev.index_subspace(s)
        asg, off, mem, a, b, rad, nb = ref.subspace(s, w, enclosure)
        assert np.array_equal(got.assignments, asg), f"assignments, subspace {s}"
        assert np.array_equal(got.member_offsets, off), f"member offsets, subspace {s}"
        assert np.array_equal(got.member_ids, mem), f"member ids, subspace {s}"
        if enclosure == "aabb":
            assert same_f32(got.gate_lo, a) and same_f32(got.gate_hi, b), f"gate lo/hi, subspace {s}"
        else:
            assert same_f32(got.gate_centers, a), f"gate centers, subspace {s}"
            assert same_f32(got.gate_radii, rad), f"gate radii, subspace {s}"
        assert got.norm_bound == nb, f"norm bound, subspace {s}: {got.norm_bound} vs {nb}"


def check_queries(dev, ref, K, d, S, seed):
    qs = [synth.queries(1, d, seed)[0], np.random.default_rng(seed).standard_normal(d).astype(np.float32)]
    for q in qs:
        for frac in (0.01, 0.05, 0.3):
            tau = rest.kth_score(K[: dev.indexed_count()], q, max(1, int(frac * dev.indexed_count())))
            req = QueryRequest(q=q, tau=float(tau))
            got = query_ta(dev, req)
            ids, st = ref.candidates(q, tau, 1)
            assert np.array_equal(got.live_ids, ids), ("ta live ids", frac)
            assert got.stats.keys_scanned == st["keys_scanned"] and got.stats.groups_tested == st["groups_tested"]
            assert (got.stats.ta_stop_depth or -1) == st["ta_stop_depth"], ("ta stop depth", frac)
            if st["ta_stop_depth"] >= 0:
                assert got.stats.ta_stop_upper == st["ta_stop_upper"]
            assert got.stats.gate_cost_equiv == st["gate_cost_equiv"] and got.stats.f_scan == st["f_scan"]
            ts = derive_subspace_thresholds(dev, q, tau)
            assert same_f32(ts, ref.thresholds(q, tau, S)), ("thresholds", frac)
            got = query_full_subspace(dev, QueryRequest(q=q, tau=float(tau), tau_subspace=list(ts)))
            ids, st = ref.candidates(q, tau, 0, ts)
            assert np.array_equal(got.live_ids, ids), ("full-subspace live ids", frac)
            assert got.stats.keys_scanned == st["keys_scanned"]


@pytest.mark.parametrize("S,r,grouping,enclosure,seed", CONFIGS)
@pytest.mark.parametrize("law", ["trace", "iid"])
def test_prefill_index_matches_reference(S, r, grouping, enclosure, seed, law):
    d, n = 64, 3001
    K, V = keys_of(law, n, d, 17)
    cfg = BuildConfig(S=S, r=r, grouping=grouping, enclosing=enclosure, rng_seed=seed)
    dev = LouverCache.adopt(K, V, cfg, 128)
    ref = REF.Cache(d, REF.cfg(S, r, grouping, enclosure, seed), 128, K, V)
    assert dev.indexed_count() == ref.indexed_count() == n
    check_index(dev, ref, d, S, enclosure)
    check_queries(dev, ref, K, d, S, 5)


@pytest.mark.parametrize("S,r,grouping,enclosure,seed", [CONFIGS[0], CONFIGS[2], CONFIGS[6]])
def test_appended_index_matches_reference(S, r, grouping, enclosure, seed):
    """A cache filled through push_key: build at the first flush, append_to_index at every
    later one (cache.cpp:12-22), random seeds keyed by each block's first id."""
    d, n, B = 32, 700, 96
    K, V = keys_of("trace", n, d, 3)
    cfg = BuildConfig(S=S, r=r, grouping=grouping, enclosing=enclosure, rng_seed=seed)
    dev = LouverCache(d, cfg, B, capacity=64)  # grows through lv_reserve
    ref = REF.Cache(d, REF.cfg(S, r, grouping, enclosure, seed), B)
    for j in range(n):
        dev.push_key(K[j], V[j])
        ref.push_key(K[j], V[j])
        if (j + 1) % B == 0 or j == n - 1:
            assert dev.indexed_count() == ref.indexed_count() and dev.flush_count() == ref.flush_count()
            if dev.indexed_count():
                check_index(dev, ref, d, S, enclosure)
    assert dev.flush_buffer() == ref.flush_buffer()
    check_index(dev, ref, d, S, enclosure)
    check_queries(dev, ref, K, d, S, 9)


@pytest.mark.parametrize("algo", [FilterAlgo.Ta, FilterAlgo.FullSubspace])
def test_cache_query_stats_match_reference(algo):
    """LouverCache.query's QueryStats come from the grouped index: keys_scanned (buffer
    included), f_scan, groups_tested, gate_cost_equiv and the TA stop depth equal the
    reference cache's (cache.cpp:30-70); the selected set is the fused kernel's."""
    d, n, B = 64, 2500, 200
    K, V = keys_of("trace", n, d, 21)
    cfg = BuildConfig()  # S=4, r=4, PCA tree, ball
    dev = LouverCache.adopt(K[:2000], V[:2000], cfg, B)
    ref = REF.Cache(d, REF.cfg(), B, K[:2000], V[:2000])
    for j in range(2000, n):
        dev.push_key(K[j], V[j])
        ref.push_key(K[j], V[j])
    for i in range(3):
        q = synth.queries(3, d, 40)[i]
        tau = rest.kth_score(K, q, 120)
        got = dev.query(QueryRequest(q=q, tau=float(tau)), algo)
        want = ref.query(q, tau, int(algo))
        assert np.array_equal(got.selected, want["selected"])
        st = want["stats"]
        assert got.stats.keys_scanned == st["keys_scanned"] and got.stats.f_scan == st["f_scan"]
        assert got.stats.groups_tested == st["groups_tested"] and got.stats.gate_cost_equiv == st["gate_cost_equiv"]
        want_depth = st["ta_stop_depth"] if st["ta_stop_depth"] is not None and st["ta_stop_depth"] >= 0 else None
        assert got.stats.ta_stop_depth == want_depth


@pytest.mark.skipif(not getattr(REF, "IS_REFERENCE", False), reason="reference build oracle/_ref absent")
@pytest.mark.parametrize("S,r,grouping,enclosure,seed", [CONFIGS[0], CONFIGS[1], CONFIGS[6]])
def test_snapshot_bytes_equal_reference_and_load(S, r, grouping, enclosure, seed):
    """lv_save_index of the grouped index writes the reference's save_index bytes
    (io.cpp:236-268); a reference snapshot loaded into an empty-index cache restores the
    same index (io.cpp:270-317) and the same candidate sets."""
    import ctypes as C

    from paper_2605_06763_b200.snapshot import load_index, save_index

    d, n, B = 32, 900, 128
    K, V = keys_of("trace", n, d, 8)
    cfg = BuildConfig(S=S, r=r, grouping=grouping, enclosing=enclosure, rng_seed=seed)
    dev = LouverCache(d, cfg, B)
    ref = REF.Cache(d, REF.cfg(S, r, grouping, enclosure, seed), B)
    for j in range(n):
        dev.push_key(K[j], V[j])
        ref.push_key(K[j], V[j])
    lib = REF.lib()
    lib.lvr_cache_save_index.argtypes = [C.c_void_p, C.c_char_p]
    with tempfile.TemporaryDirectory() as tmp:
        pd, pr = os.path.join(tmp, "dev.lvix"), os.path.join(tmp, "ref.lvix")
        save_index(dev, pd)
        assert lib.lvr_cache_save_index(ref.h, pr.encode()) == 0
        assert open(pd, "rb").read() == open(pr, "rb").read()
        # load the reference's snapshot into a cache holding the same keys but no index yet
        dev2 = LouverCache(d, cfg, 10**6, capacity=1024)
        for j in range(n):
            dev2.push_key(K[j], V[j])
        assert dev2.indexed_count() == 0
        assert load_index(dev2, pr) == ref.indexed_count()
        check_index(dev2, ref, d, S, enclosure)
        check_queries(dev2, ref, K, d, S, 2)


@pytest.mark.parametrize("S,r,grouping,enclosure,n,d", [
    (1, 1, "pca_tree", "ball", 37, 8),        # every key its own group
    (8, 2, "pca_tree", "span_ball", 19, 8),   # S = d: one coordinate per subspace
    (3, 64, "pca_tree", "aabb", 50, 10),      # one group holds every key (m < r)
    (2, 5, "interleaved", "aabb", 23, 7),
    (5, 3, "random", "span_ball", 41, 13),
])
def test_grouped_index_edge_shapes(S, r, grouping, enclosure, n, d):
    """Degenerate shapes of index.cpp: r = 1, r > m, S = d, odd widths; the prefill build and
    one appended block (push_key up to a flush) equal the reference's."""
    K, V = keys_of("iid", n + 9, d, 31)
    cfg = BuildConfig(S=S, r=r, grouping=grouping, enclosing=enclosure, rng_seed=11)
    dev = LouverCache.adopt(K[:n], V[:n], cfg, 9)
    ref = REF.Cache(d, REF.cfg(S, r, grouping, enclosure, 11), 9, K[:n], V[:n])
    check_index(dev, ref, d, S, enclosure)
    for j in range(n, n + 9):
        dev.push_key(K[j], V[j])
        ref.push_key(K[j], V[j])
    assert dev.indexed_count() == ref.indexed_count() == n + 9
    check_index(dev, ref, d, S, enclosure)
    check_queries(dev, ref, K, d, S, 4)


def test_grouped_index_errors():
    """The reference's argument errors (query.cpp:84-87) and the API's own."""
    d = 16
    K, V = keys_of("iid", 64, d, 2)
    dev = LouverCache.adopt(K, V, BuildConfig(S=4, r=4), 16)
    q = K[0]
    with pytest.raises(ValueError, match="tau_subspace required"):
        query_full_subspace(dev, QueryRequest(q=q, tau=0.0))
    with pytest.raises(ValueError, match="length != S"):
        query_full_subspace(dev, QueryRequest(q=q, tau=0.0, tau_subspace=[0.0, 0.0]))
    with pytest.raises(ValueError):
        query_ta(dev, QueryRequest(q=q[:8], tau=0.0))
    plain = LouverCache.adopt(K, V, BuildConfig(S=4, r=4), 16, group_index=False)
    with pytest.raises(ValueError, match="grouped index"):
        query_ta(plain, QueryRequest(q=q, tau=0.0))
