"""The oracle restatement (oracle/louver_oracle.cpp) against the reference library itself.

oracle/_ref/liblouver_ref.so is the reference's own sources (/root/reference/proj/src/*.cpp,
unmodified) compiled against the Eigen shim in oracle/ref (``make -C oracle ref``; built by
__graft_entry__.build() wherever /root/reference exists). Both expose the same C ABI
(oracle/louver_oracle.h), so every call below runs twice on the same bytes and the results
must agree: selected / retrieved sets, attention outputs and weights bit for bit, index
groupings and enclosures, TA statistics, threshold estimates, reservoir contents, and the
synthetic key / query streams the tests and the bench generate (io.cpp:145-206).
"""
import ctypes as C
import itertools

import numpy as np
import pytest

from oracle import pyoracle as rest
from paper_2605_06763_b200 import synth

ref = rest.reference_module()
pytestmark = pytest.mark.skipif(ref is None, reason="reference build oracle/_ref absent (needs /root/reference)")


def same_f32(a, b):
    return np.array_equal(np.asarray(a, np.float32).view(np.uint32), np.asarray(b, np.float32).view(np.uint32))


def test_synthetic_streams_are_the_reference_generators():
    """synth.keys / synth.queries (liblouver_synth.so) reproduce gen_synthetic /
    gen_synthetic_queries (io.cpp:145-206) bit for bit."""
    lib = ref.lib()
    lib.lvr_gen_synthetic.argtypes = [C.c_int64, C.c_int, C.c_uint64, C.c_int, C.c_void_p]
    for n, d, seed in ((1000, 128, 7), (300, 33, 12345), (17, 64, 0)):
        for queries in (0, 1):
            out = np.empty((n, d), np.float32)
            assert lib.lvr_gen_synthetic(n, d, seed, queries, out.ctypes.data) == 0
            mine = synth.queries(n, d, seed) if queries else synth.keys(n, d, seed)
            assert same_f32(out, mine), (n, d, seed, queries)


def test_groupings_and_enclosures():
    pts = synth.keys(513, 16, 3)
    for r in (1, 2, 4, 7, 16):
        assert np.array_equal(rest.balanced_pca_tree(pts, r), ref.balanced_pca_tree(pts, r)), r
    for g, e in itertools.product(range(4), range(3)):
        cfg = rest.cfg(4, 4, g, e, seed=99)
        for s, base in ((0, 0), (3, 4096)):
            assert np.array_equal(rest.assign_groups(pts, cfg, s, base), ref.assign_groups(pts, ref.cfg(4, 4, g, e, 99), s, base))
    for kind in ("ball", "aabb", "span_ball"):
        for m in (1, 3, 16):
            a, b = rest.enclose_group(pts[:m], kind), ref.enclose_group(pts[:m], kind)
            assert all(same_f32(x, y) for x, y in zip(a, b)), (kind, m)


def test_brute_force_exact_check_attention():
    k, v = synth.keys(2000, 64, 21), synth.keys(2000, 64, 22)
    for i, q in enumerate(np.concatenate([synth.queries(3, 64, 21), synth.iid_normal(3, 64, 5)])):
        sc = rest.scores(k, q)
        assert same_f32(sc, ref.scores(k, q))
        for tau in (np.sort(sc)[::-1][99], sc[13], np.float32(-np.inf)):
            a = rest.brute_force_range(k, q, tau)
            assert np.array_equal(a, ref.brute_force_range(k, q, tau))
            cand = np.arange(0, 2000, 3, dtype=np.uint32)[::-1].copy()
            assert np.array_equal(rest.exact_check(k, cand, q, tau), ref.exact_check(k, cand, q, tau))
            buf = np.arange(1990, 2000)
            ra, rb = rest.sparse_attention(k, v, buf, a, q, 0.125), ref.sparse_attention(k, v, buf, a, q, 0.125)
            assert np.array_equal(ra[0], rb[0]) and same_f32(ra[1], rb[1]) and same_f32(ra[2], rb[2]), (i, tau)


@pytest.mark.parametrize("S,r", list(itertools.product((1, 2, 4, 8, 16), (2, 4, 8))))  # acceptance.cpp:79-181 grid
def test_cache_queries_all_build_configs(S, r):
    """LouverCache::query (cache.cpp:30-70) under every grouping x enclosure, both filters,
    strict and not: sets, attention output and the filter statistics agree."""
    n, d = 1024, 32
    k, v = synth.keys(n, d, 100 + S), synth.keys(n, d, 101 + S)
    qs = np.concatenate([synth.queries(2, d, 100 + S), synth.iid_normal(1, d, S)])
    for g, e in itertools.product(range(4), range(3)):
        a = rest.Cache(d, rest.cfg(S, r, g, e, seed=5), 64, keys=k[:900], values=v[:900])
        b = ref.Cache(d, ref.cfg(S, r, g, e, seed=5), 64, keys=k[:900], values=v[:900])
        for t in range(900, n):  # pushes across a flush at B = 64
            a.push_key(k[t], v[t])
            b.push_key(k[t], v[t])
        assert (a.indexed_count(), a.flush_count()) == (b.indexed_count(), b.flush_count())
        for q in qs:
            tau = np.sort(rest.scores(k, q))[::-1][int(0.05 * n)]
            for algo, strict in itertools.product((0, 1), (False, True)):
                x, y = a.query(q, tau, algo, strict), b.query(q, tau, algo, strict)
                assert np.array_equal(x["selected"], y["selected"])
                assert np.array_equal(x["retrieved"], y["retrieved"])
                assert (x["output"] is None) == (y["output"] is None)
                if x["output"] is not None:
                    assert same_f32(x["output"], y["output"]), (S, r, g, e, algo, strict)
                sx, sy = x["stats"], y["stats"]
                assert sx["groups_tested"] == sy["groups_tested"]
                assert sx["keys_scanned"] == sy["keys_scanned"], (S, r, g, e, algo)
                assert sx["f_scan"] == sy["f_scan"] and sx["gate_cost_equiv"] == sy["gate_cost_equiv"]
                assert sx["ta_stop_depth"] == sy["ta_stop_depth"]
                assert sx["ta_stop_upper"] == sy["ta_stop_upper"]


def test_threshold_oracle_and_reservoir():
    keys = synth.keys(300, 64, 8)
    q = synth.queries(1, 64, 8)[0]
    for variant, m, alpha in ((0, 2, 0.1), (1, 5, 0.1), (2, 2, 0.1), (3, 2, 0.1), (4, 2, 0.05), (4, 2, 0.5)):
        assert same_f32([rest.estimate_tau(keys, q, variant, m, alpha)], [ref.estimate_tau(keys, q, variant, m, alpha)])
    for cap, seed in ((1, 3), (16, 0), (256, 42)):
        a, b = rest.Reservoir(cap, seed), ref.Reservoir(cap, seed)
        for t in range(2000):
            assert a.update(t) == b.update(t)
        assert np.array_equal(a.ids(), b.ids()) and a.seen() == b.seen()
