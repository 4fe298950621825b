"""Pin the CPU oracle against the reference's own known-answer and oracle-equality
tests (paths relative to /root/reference/proj/tests). CPU only."""
import math

import numpy as np
import pytest

from paper_2605_06763_b200 import synth

NEG_INF = np.float32(-np.inf)


def random_matrix(n, d, seed):  # test_util.hpp:10-12
    return synth.keys(n, d, seed)


def random_store(n, d, seed):  # test_util.hpp:14-16
    return random_matrix(n, d, seed), random_matrix(n, d, seed + 1)


def random_query(d, seed):  # test_util.hpp:18-24 (iid N(0,1); numpy RNG, not bit-identical)
    return synth.iid_normal(1, d, seed)[0]


def tiny_store():  # test_query.cpp:15-19
    k = np.array([[1, 0], [0, 1], [-1, 0], [0, -1], [2, 2], [0.5, 0.5]], np.float32)
    return k, k.copy()


# ---------------------------------------------------------------- test_core.cpp


def test_subspace_layout_widths(oracle):  # test_core.cpp:11-26
    assert list(np.diff(oracle.layout(4, 2))) == [2, 2]
    assert list(np.diff(oracle.layout(1, 1))) == [1]
    assert list(np.diff(oracle.layout(5, 2))) == [3, 2]
    with pytest.raises(ValueError):
        oracle.layout(4, 5)
    with pytest.raises(ValueError):
        oracle.layout(4, 0)


def test_dot_basics(oracle):  # test_core.cpp:60-65
    assert oracle.dot([1, 1], [2, 2]) == 4.0
    assert oracle.dot([1, 0], [0, 1]) == 0.0
    with pytest.raises(ValueError):
        oracle.dot([1], [1, 2])


def test_dot_matches_scalar_loop_bit_for_bit(oracle):  # test_core.cpp:67-73
    a, b = random_query(64, 1), random_query(64, 2)
    ref = np.float32(0)
    for i in range(64):
        ref = np.float32(ref + np.float32(a[i] * b[i]))
    assert oracle.dot(a, b) == ref
    assert oracle.dot(a, b) == oracle.dot(a, b)


def test_enclosure_bounds_known_answers(oracle):  # test_core.cpp:75-98 via enclose_group
    # ball around {(1.5,0),(2.5,0)}: center (2,0), radius 0.5 (+1 ulp): bound for q=(1,0) = 2.5(+)
    c, r = oracle.enclose_group(np.array([[1.5, 0], [2.5, 0]]), "ball")
    assert list(c) == [2.0, 0.0]
    assert r == np.nextafter(np.float32(0.5), np.float32(np.inf))
    lo, hi = oracle.enclose_group(np.array([[0, 0], [1, 1]]), "aabb")
    q = np.array([1, -1], np.float32)
    assert np.float32(sum(max(q[i] * lo[i], q[i] * hi[i]) for i in range(2))) == 1.0


# --------------------------------------------------------------- test_index.cpp


def test_pca_tree_simple(oracle):  # test_index.cpp:59-70
    assert list(oracle.balanced_pca_tree(np.array([[0], [1], [2], [3]]), 2)) == [0, 0, 1, 1]
    assert list(oracle.balanced_pca_tree(np.array([[0, 0], [1, 1], [2, 2]]), 4)) == [0, 0, 0]
    with pytest.raises(ValueError):
        oracle.balanced_pca_tree(np.zeros((0, 1)), 2)


def test_pca_tree_m10_r4_sizes(oracle):  # test_index.cpp:72-81
    a = oracle.balanced_pca_tree(random_matrix(10, 3, 5), 4)
    sizes = np.bincount(a)
    assert list(sizes) == [2, 3, 2, 3]


def test_assign_groups_strategies(oracle):  # test_index.cpp:83-107
    pts8 = random_matrix(8, 2, 1)
    c = oracle.cfg(r=4, grouping="contiguous")
    assert list(oracle.assign_groups(pts8, c)) == [0, 0, 0, 0, 1, 1, 1, 1]
    c = oracle.cfg(r=4, grouping="interleaved")
    assert list(oracle.assign_groups(pts8, c)) == [0, 1, 0, 1, 0, 1, 0, 1]
    pts9 = random_matrix(9, 2, 2)
    sizes = np.bincount(oracle.assign_groups(pts9, oracle.cfg(r=4, grouping="contiguous")))
    assert list(sizes) == [4, 4, 1]
    c = oracle.cfg(r=4, grouping="random", seed=7)
    a1, a2 = oracle.assign_groups(pts9, c), oracle.assign_groups(pts9, c)
    assert list(a1) == list(a2)
    assert np.bincount(a1).max() <= 4


def test_enclose_group_known_answers(oracle):  # test_index.cpp:109-134
    c, r = oracle.enclose_group(np.array([[0, 0], [2, 0]]), "ball")
    assert list(c) == [1.0, 0.0]
    assert r == pytest.approx(1.0, rel=1e-6)
    for kind in ("ball", "span_ball"):
        c, r = oracle.enclose_group(np.array([[3, -4]]), kind)
        assert list(c) == [3.0, -4.0] and r == 0.0
    lo, hi = oracle.enclose_group(np.array([[3, -4]]), "aabb")
    assert list(lo) == [3.0, -4.0] and list(hi) == [3.0, -4.0]
    lo, hi = oracle.enclose_group(np.array([[0, 0], [1, 2], [2, 1]]), "aabb")
    assert list(lo) == [0.0, 0.0] and list(hi) == [2.0, 2.0]
    with pytest.raises(ValueError):
        oracle.enclose_group(np.zeros((0, 2)), "ball")


def test_pca_tree_balance_bounds(oracle):  # test_index.cpp:160-177
    rng = np.random.default_rng(17)
    for trial in range(50):
        n = 16 + int(rng.integers(0, 700))
        r = 2 + int(rng.integers(0, 7))
        sizes = np.bincount(oracle.balanced_pca_tree(random_matrix(n, 4, trial), r))
        K = sizes.size
        assert K >= (n + r - 1) // r
        assert K <= (2 * n + r) // (r + 1)
        assert sizes.min() >= (r + 1) // 2 and sizes.max() <= r


def test_build_partition_invariant(oracle):  # test_index.cpp:136-158 (partition part)
    k, v = random_store(4096, 64, 11)
    cache = oracle.Cache(64, oracle.cfg(4, 4), 128, keys=k, values=v)
    for s in range(4):
        seen = np.zeros(4096, np.int32)
        for g in range(cache.groups(s)):
            m = cache.group_members(s, g)
            assert 1 <= m.size <= 4
            seen[m] += 1
        assert (seen == 1).all()


# --------------------------------------------------------------- test_query.cpp


def test_brute_force_hand_checked(oracle):  # test_query.cpp:25-33
    k, _ = tiny_store()
    q = np.array([1, 1], np.float32)
    assert list(oracle.brute_force_range(k, q, 1.0)) == [0, 1, 4, 5]
    assert list(oracle.brute_force_range(k, q, NEG_INF)) == [0, 1, 2, 3, 4, 5]
    assert list(oracle.brute_force_range(k, q, 100.0)) == []
    assert list(oracle.brute_force_range(k, q, 1.0, 2)) == [0, 1]
    with pytest.raises(ValueError):
        oracle.brute_force_range(k, q, 1.0, 7)


def test_exact_check_basics(oracle):  # test_query.cpp:35-43
    k, _ = tiny_store()
    q = np.array([1, 1], np.float32)
    allids = [0, 1, 2, 3, 4, 5]
    assert list(oracle.exact_check(k, allids, q, 1.0)) == list(oracle.brute_force_range(k, q, 1.0))
    assert list(oracle.exact_check(k, [], q, 1.0)) == []
    once = oracle.exact_check(k, allids, q, 1.0)
    assert list(oracle.exact_check(k, once, q, 1.0)) == list(once)


@pytest.mark.parametrize("algo", [0, 1])
def test_degenerate_groups_equal_oracle(oracle, algo):  # test_query.cpp:45-56
    k, v = random_store(64, 8, 5)
    cache = oracle.Cache(8, oracle.cfg(1, 1, "contiguous", "ball"), 128, keys=k, values=v)
    q = random_query(8, 6)
    res = cache.query(q, 0.5, algo=algo)
    assert list(res["selected"]) == list(oracle.brute_force_range(k, q, 0.5))


def test_minus_inf_scans_everything(oracle):  # test_query.cpp:58-72, 106-117
    k, v = random_store(100, 16, 7)
    cache = oracle.Cache(16, oracle.cfg(4, 4), 128, keys=k, values=v)
    q = random_query(16, 8)
    for algo in (0, 1):
        res = cache.query(q, NEG_INF, algo=algo)
        assert res["stats"]["keys_scanned"] == 100
        assert res["stats"]["f_scan"] == 1.0
        assert res["selected"].size == 100
    assert cache.query(q, NEG_INF, algo=1)["stats"]["ta_stop_depth"] is None


def test_derived_thresholds_zero_fn(oracle):  # test_query.cpp:74-89
    k, v = random_store(512, 16, 9)
    cache = oracle.Cache(16, oracle.cfg(4, 4), 1024, keys=k, values=v)
    for trial in range(50):
        q = random_query(16, 100 + trial)
        tau = np.float32(trial % 11) - np.float32(3.0)
        res = cache.query(q, tau, algo=0)
        assert list(res["selected"]) == list(oracle.brute_force_range(k, q, tau))


def test_ta_exact_equals_oracle(oracle):  # test_query.cpp:148-160
    k, v = random_store(4096, 64, 17)
    cache = oracle.Cache(64, oracle.cfg(4, 4), 8192, keys=k, values=v)
    halted = 0
    for trial in range(20):
        q = synth.queries(1, 64, 200 + trial)[0]
        scores = oracle.scores(k, q)
        tau = np.float32(np.sort(scores)[::-1][int(0.05 * 4096)])  # ~5% selectivity
        res = cache.query(q, tau, algo=1)
        assert list(res["selected"]) == list(oracle.brute_force_range(k, q, tau))
        halted += res["stats"]["ta_stop_depth"] is not None
    assert halted > 0


def test_lowering_tau_never_shrinks(oracle):  # test_query.cpp:162-176
    k, v = random_store(512, 16, 19)
    cache = oracle.Cache(16, oracle.cfg(4, 4), 1024, keys=k, values=v)
    q = random_query(16, 20)
    prev = 0
    for tau in (8.0, 4.0, 2.0, 0.0, -4.0):
        live = cache.query(q, tau, algo=1)["stats"]["keys_scanned"]
        assert live >= prev
        prev = live


def test_sparse_attention_basics(oracle):  # test_query.cpp:178-196
    k, v = tiny_store()
    q = np.array([1, 1], np.float32)
    tok, w, out = oracle.sparse_attention(k, v, [], [4], q, 1.0)
    assert list(w) == [1.0] and list(out) == [2.0, 2.0]
    tok, w, out = oracle.sparse_attention(k, v, [], [0, 1], q, 1.0)
    assert w[0] == pytest.approx(0.5, rel=1e-6) and w[1] == pytest.approx(0.5, rel=1e-6)
    assert oracle.sparse_attention(k, v, [], [], q, 1.0) is None


def test_softmax_weights_sum_and_shift(oracle):  # test_query.cpp:198-223
    k, v = random_store(64, 16, 21)
    q = random_query(16, 22)
    allids = np.arange(64)
    _, w, _ = oracle.sparse_attention(k, v, [], allids, q, 0.25)
    assert (w >= 0).all() and float(np.sum(w.astype(np.float64))) == pytest.approx(1.0, rel=1e-6)
    shift = random_query(16, 23)
    _, w2, _ = oracle.sparse_attention(k + shift, v, [], allids, q, 0.25)
    np.testing.assert_allclose(w2, w, rtol=1e-4)


def test_stats_self_consistent(oracle):  # test_query.cpp:235-248
    k, v = random_store(256, 16, 25)
    cache = oracle.Cache(16, oracle.cfg(4, 4, "pca_tree", "aabb"), 1024, keys=k, values=v)
    res = cache.query(random_query(16, 26), 2.0, algo=1)
    st = res["stats"]
    assert st["f_scan"] == st["keys_scanned"] / 256
    assert st["gate_cost_equiv"] == 2.0 * st["groups_tested"] / 4


# --------------------------------------------------------------- test_cache.cpp


def test_push_key_buffer_semantics(oracle):  # test_cache.cpp:33-54
    c = oracle.Cache(8, oracle.cfg(2, 4), 128)
    keys = random_matrix(128, 8, 1)
    c.push_key(keys[0], keys[0])
    assert (c.pending_count(), c.indexed_count(), c.flush_count()) == (1, 0, 0)
    for t in range(1, 127):
        c.push_key(keys[t], keys[t])
    assert c.pending_count() == 127
    c.push_key(keys[127], keys[127])
    assert (c.pending_count(), c.indexed_count(), c.flush_count()) == (0, 128, 1)


def test_4096_pushes_flush_32_times(oracle):  # test_cache.cpp:56-64
    c = oracle.Cache(16, oracle.cfg(4, 4), 128)
    keys = random_matrix(4096, 16, 2)
    for t in range(4096):
        c.push_key(keys[t], keys[t])
    assert c.flush_count() == 32 and c.pending_count() == 0


def test_flush_b8_r4_two_groups(oracle):  # test_cache.cpp:66-78
    c = oracle.Cache(8, oracle.cfg(2, 4), 16)
    keys = random_matrix(8, 8, 3)
    for t in range(8):
        c.push_key(keys[t], keys[t])
    assert c.pending_count() == 8
    assert c.flush_buffer()
    assert c.groups(0) == 2 and c.groups(1) == 2
    assert not c.flush_buffer()
    assert c.flush_count() == 1


def test_interleaved_pushes_and_queries(oracle):  # test_cache.cpp:102-121
    c = oracle.Cache(16, oracle.cfg(4, 4), 32)
    keys, values = random_matrix(512, 16, 5), random_matrix(512, 16, 6)
    for t in range(512):
        c.push_key(keys[t], values[t])
        if t % 16 != 15:
            continue
        q = random_query(16, 1000 + t)
        want = oracle.brute_force_range(keys[: t + 1], q, 2.0)
        for algo in (1, 0):
            assert list(c.query(q, 2.0, algo=algo)["selected"]) == list(want)


def test_strict_toggle(oracle):  # test_cache.cpp:123-144
    c = oracle.Cache(4, oracle.cfg(2, 2), 64)
    keys = np.array([[1, 1, 1, 1], [-1, -1, -1, -1], [2, 2, 2, 2]], np.float32)
    for t in range(3):
        c.push_key(keys[t], keys[t])
    q = np.ones(4, np.float32)
    dense = c.query(q, 0.0, algo=1, strict=False)
    assert dense["output"] is not None
    assert list(dense["selected"]) == [0, 2] and dense["retrieved"].size == 3
    strict = c.query(q, 0.0, algo=1, strict=True)
    # attended set {0, 2}: output = softmax over scores (4, 8) * scale 1/2 of the values
    s = np.array([4.0, 8.0], np.float32) * np.float32(0.5)
    w = np.exp(s - s.max())
    w = w / w.sum()
    np.testing.assert_allclose(strict["output"], w[0] * keys[0] + w[1] * keys[2], rtol=1e-6)


def test_partial_final_flush(oracle):  # test_cache.cpp:146-158
    c = oracle.Cache(8, oracle.cfg(2, 4, "contiguous", "ball"), 64)
    keys = random_matrix(6, 8, 7)
    for t in range(6):
        c.push_key(keys[t], keys[t])
    assert c.flush_buffer()
    for s in range(2):
        assert c.groups(s) == 2
        assert c.group_members(s, 0).size == 4 and c.group_members(s, 1).size == 2


# ---------------------------------------------------------------- acceptance.cpp


def test_dense_equivalence_vs_double(oracle):  # acceptance.cpp:291-336 (criterion 6)
    rng = np.random.default_rng(9000)
    worst = 0.0
    for _ in range(25):
        k = rng.standard_normal((1024, 64)).astype(np.float32)
        v = rng.standard_normal((1024, 64)).astype(np.float32)
        q = rng.standard_normal(64).astype(np.float32)
        scale = np.float32(1.0 / math.sqrt(64.0))
        _, _, out = oracle.sparse_attention(k, v, [], np.arange(1024), q, scale)
        s = np.float64(scale) * oracle.scores(k, q).astype(np.float64)
        w = np.exp(s - s.max())
        dense = (w / w.sum()) @ v.astype(np.float64)
        worst = max(worst, np.linalg.norm(out - dense) / np.linalg.norm(dense))
    assert worst <= 1e-5


def test_recall_at_k(oracle):  # acceptance.cpp:342-374 (criterion 7)
    for inst in range(10):
        k = random_matrix(1024, 64, 11000 + inst)
        cache = oracle.Cache(64, oracle.cfg(8, 4), 4096, keys=k, values=k)
        q = random_query(64, 11100 + inst)
        sc = oracle.scores(k, q)
        for kk in (10, 100):
            top = np.argsort(-sc, kind="stable")[:kk]
            tau = np.nextafter(np.sort(sc)[::-1][kk - 1], np.float32(-np.inf))
            got = set(cache.query(q, tau, algo=1)["selected"].tolist())
            assert set(top.tolist()) <= got
