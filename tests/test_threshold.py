"""Threshold oracle: the reference's threshold tests
(proj/tests/test_threshold.cpp, acceptance.cpp:446-474) against the CPU oracle and
the product's reservoir sampler (host code in liblouver_b200.so, no device needed);
the device estimate_tau against the oracle is in the GPU section (bit-exact τ)."""
import numpy as np
import pytest

from paper_2605_06763_b200 import (BuildConfig, LouverCache, LouverLayer, OracleConfig, OracleVariant,
                                   Reservoir, estimate_tau, estimate_tau_layer, parse_oracle)
from paper_2605_06763_b200.threshold import to_string

V = OracleVariant
ALL = [V.SampleMax, V.SampleTopK, V.SampleGap, V.SampleMeanMax, V.Budget]


def col(xs):
    return np.array(xs, np.float32).reshape(-1, 1)


# ------------------------------------------------------------------ oracle KATs (CPU)


def test_oracle_variants_hand_enumerated(oracle):  # test_threshold.cpp:63-84
    k, q = col([10, 7, 6, 2, 1]), np.array([1], np.float32)
    assert oracle.estimate_tau(k, q, V.SampleMax) == 10.0
    assert oracle.estimate_tau(k, q, V.SampleTopK, m=2) == 7.0
    with pytest.raises(ValueError):
        oracle.estimate_tau(k, q, V.SampleTopK, m=6)
    assert oracle.estimate_tau(k, q, V.SampleGap) == 6.0
    assert oracle.estimate_tau(k, q, V.SampleMeanMax) == pytest.approx((10.0 + 26.0 / 5.0) / 2.0)


def test_oracle_budget_nearest_rank(oracle):  # test_threshold.cpp:86-98
    k, q = col(np.arange(1, 101)), np.array([1], np.float32)
    assert oracle.estimate_tau(k, q, V.Budget, alpha=0.10) == 91.0
    assert oracle.estimate_tau(k, q, V.Budget, alpha=0.999) <= 2.0
    assert oracle.estimate_tau(k, q, V.Budget, alpha=0.001) == 100.0
    with pytest.raises(ValueError):
        oracle.estimate_tau(k, q, V.Budget, alpha=1.5)
    with pytest.raises(ValueError):
        oracle.estimate_tau(np.zeros((0, 1), np.float32), q, V.SampleMax)


def test_oracle_variant_ordering_and_scale(oracle):  # test_threshold.cpp:100-130
    for trial in range(100):
        rng = np.random.default_rng(trial)
        keys = rng.standard_normal((32, 8)).astype(np.float32)
        q = rng.standard_normal(8).astype(np.float32)
        t = lambda v, m=2, qq=q: oracle.estimate_tau(keys, qq, v, m=m)  # noqa: E731
        assert t(V.SampleMax) >= t(V.SampleTopK, 2) >= t(V.SampleTopK, 5) >= t(V.SampleTopK, 10)
        assert t(V.SampleMax) >= t(V.SampleGap)
        for v in ALL:
            assert t(v, qq=2.0 * q) == pytest.approx(2.0 * t(v), rel=1e-4)


# ------------------------------------------------------- reservoir sampler (product host code)


def test_reservoir_admits_until_capacity():  # test_threshold.cpp:23-33
    r = Reservoir(4, 1)
    for t in range(4):
        assert r.update(t) == t
        assert r.size() == t + 1 and r.ids()[t] == t
    r.update(4)
    assert r.size() == 4 and r.seen() == 5 and r.capacity() == 4
    with pytest.raises(ValueError):
        Reservoir(0, 0)


def test_reservoir_matches_oracle_draws(oracle):  # test_threshold.cpp:35-42, same engine + distribution
    for cap, seed in [(8, 77), (256, 0), (32, 17000), (1, 5), (64, 2**63 + 11)]:
        a, b = Reservoir(cap, seed), oracle.Reservoir(cap, seed)
        for t in range(2000):
            assert a.update(t) == b.update(t)
        assert np.array_equal(a.ids(), b.ids())
        assert a.seen() == b.seen() == 2000


def test_capacity_one_reservoir_is_uniform():  # test_threshold.cpp:44-61
    counts = np.zeros(8, int)
    for trial in range(50000):
        r = Reservoir(1, trial)
        for t in range(8):
            r.update(t)
        counts[r.ids()[0]] += 1
    exp = 50000 / 8
    assert float(((counts - exp) ** 2 / exp).sum()) < 24.32


def test_parse_oracle_round_trip():  # test_threshold.cpp:132-140
    assert parse_oracle("max").variant == V.SampleMax
    assert parse_oracle("topk:5").m == 5
    assert parse_oracle("budget:0.05").alpha == pytest.approx(0.05)
    assert parse_oracle("gap").variant == V.SampleGap
    assert parse_oracle("meanmax").variant == V.SampleMeanMax
    with pytest.raises(ValueError):
        parse_oracle("bogus")
    with pytest.raises(ValueError):
        parse_oracle("budget:1.5")
    assert to_string(parse_oracle("topk:3")) == "topk:3"
    assert to_string(parse_oracle("budget:0.05")) == "budget:0.050000"


# ------------------------------------------------------------------------ device (GPU)


@pytest.fixture(scope="module")
def torch():
    import torch

    assert torch.cuda.is_available(), "GPU tests need a CUDA device"
    return torch


@pytest.mark.gpu
def test_device_estimate_hand_enumerated(torch):  # test_threshold.cpp:63-98 on the device
    k = col([10, 7, 6, 2, 1])
    c = LouverCache.adopt(k, k.copy(), BuildConfig(S=1, r=2), 128)
    r = Reservoir(64, 0, cache=c)
    for t in range(5):
        r.update(t, k[t])
    q = np.array([1], np.float32)
    assert estimate_tau(r, q, OracleConfig(V.SampleMax)) == 10.0
    assert estimate_tau(r, q, OracleConfig(V.SampleTopK, 2)) == 7.0
    with pytest.raises(ValueError):
        estimate_tau(r, q, OracleConfig(V.SampleTopK, 6))
    assert estimate_tau(r, q, OracleConfig(V.SampleGap)) == 6.0
    assert estimate_tau(r, q, OracleConfig(V.SampleMeanMax)) == pytest.approx((10.0 + 26.0 / 5.0) / 2.0)
    k2 = col(np.arange(1, 101))
    c2 = LouverCache.adopt(k2, k2.copy(), BuildConfig(S=1, r=2), 128)
    r2 = Reservoir(128, 0, cache=c2)
    for t in range(100):
        r2.update(t)
    assert estimate_tau(r2, q, OracleConfig(V.Budget, alpha=0.10)) == 91.0
    assert estimate_tau(r2, q, OracleConfig(V.Budget, alpha=0.999)) <= 2.0
    assert estimate_tau(r2, q, OracleConfig(V.Budget, alpha=0.001)) == 100.0
    with pytest.raises(ValueError):
        estimate_tau(Reservoir(4, 0, cache=c2), q, OracleConfig())  # empty reservoir


@pytest.mark.gpu
@pytest.mark.parametrize("cap,d", [(32, 8), (256, 128), (1000, 64), (4096, 128)])
def test_device_estimate_matches_oracle_f32(torch, oracle, cap, d):
    rng = np.random.default_rng(cap + d)
    n = 3 * cap + 7
    keys = rng.standard_normal((n, d)).astype(np.float32)
    c = LouverCache.adopt(keys, keys.copy(), BuildConfig(S=1, r=16), 128)
    r = Reservoir(cap, 1234 + cap, cache=c)
    for t in range(n):
        r.update(t)
    sample = keys[r.ids()]
    for trial in range(4):
        q = rng.standard_normal(d).astype(np.float32)
        for cfg in [OracleConfig(V.SampleMax), OracleConfig(V.SampleTopK, 5), OracleConfig(V.SampleGap),
                    OracleConfig(V.SampleMeanMax), OracleConfig(V.Budget, alpha=0.05),
                    OracleConfig(V.Budget, alpha=0.5)]:
            want = oracle.estimate_tau(sample, q, int(cfg.variant), m=cfg.m, alpha=cfg.alpha)
            assert np.float32(estimate_tau(r, q, cfg)) == want, (cfg, trial)


@pytest.mark.gpu
def test_device_estimate_layer_bf16_every_head(torch, oracle):
    """C2-shaped GQA layer (bf16 arena): every q head's τ from its kv slot's reservoir,
    device tensors in and out (enqueue-only path), against the oracle on the stored keys."""
    d, H, G, B, n, cap = 128, 4, 4, 2, 6000, 256
    rng = np.random.default_rng(7)
    K = rng.standard_normal((B, H, n, d)).astype(np.float32)
    layer = LouverLayer(d, H, G, B, n + 64)
    layer.build(K, K)
    slots = B * H
    ids = np.zeros((slots, cap), np.uint32)
    for s in range(slots):
        r = Reservoir(cap, 1000 * s + 3)
        for t in range(n):
            r.update(t)
        ids[s] = r.ids()
    q = rng.standard_normal((B, H * G, d)).astype(np.float32)
    for cfg in [OracleConfig(V.SampleMax), OracleConfig(V.SampleTopK, 3), OracleConfig(V.SampleGap),
                OracleConfig(V.SampleMeanMax), OracleConfig(V.Budget, alpha=0.05)]:
        tau_d = estimate_tau_layer(layer, torch.from_numpy(ids).cuda(), cap, torch.from_numpy(q).cuda(), cfg)
        tau_h = estimate_tau_layer(layer, ids, cap, q, cfg)
        torch.cuda.synchronize()
        tau_d = tau_d.cpu().numpy()
        for s in range(slots):
            sample = layer.read_rows(s, 0, n)[ids[s]]
            for g in range(G):
                row = (s // H, (s % H) * G + g)
                want = oracle.estimate_tau(sample, q[row], int(cfg.variant), m=cfg.m, alpha=cfg.alpha)
                assert tau_d[row] == want and tau_h[row] == want, (cfg, s, g)
