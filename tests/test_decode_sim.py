"""Decode-loop driver: run_decode_sim (bench.cpp:54-136) on the
device. Ports test_bench.cpp:19-60 and checks every per-step quantity the final sets
determine (selected, retrieved, τ, flushes) against the oracle's own decode loop —
LouverCache::query + Reservoir + estimate_tau restated on the CPU — on the same rows."""
import math

import numpy as np
import pytest

from paper_2605_06763_b200 import BuildConfig, FilterAlgo, OracleConfig, OracleVariant
from paper_2605_06763_b200.decode_sim import (DecodeSimConfig, ThresholdSource, run_decode_sim,
                                              speedup_estimate)


def rmat(n, d, seed):
    return np.random.default_rng(seed).standard_normal((n, d)).astype(np.float32)


def test_speedup_estimate():  # bench.cpp:12-19
    assert speedup_estimate(2, 4, 0.5) == pytest.approx(1.0)
    with pytest.raises(ValueError):
        speedup_estimate(1, 0.5, 0.1)
    with pytest.raises(ValueError):
        speedup_estimate(1, 4, 1.5)
    with pytest.raises(ArithmeticError):
        speedup_estimate(0, 4, 0.0)


def test_config_errors():
    with pytest.raises(ValueError):
        run_decode_sim(rmat(4, 8, 1), rmat(4, 8, 2), rmat(3, 8, 3), DecodeSimConfig(threshold=ThresholdSource(0.0)))
    with pytest.raises(ValueError):
        run_decode_sim(rmat(4, 8, 1), rmat(4, 8, 2), rmat(4, 8, 3), DecodeSimConfig())


@pytest.fixture(scope="module")
def torch():
    import torch

    assert torch.cuda.is_available(), "GPU tests need a CUDA device"
    return torch


@pytest.mark.gpu
def test_neg_inf_threshold_scans_everything(torch):  # test_bench.cpp:19-38
    steps = 512
    cfg = DecodeSimConfig(build=BuildConfig(4, 4, "pca_tree", "ball", 0), buffer_capacity=64,
                          threshold=ThresholdSource(fixed_tau=-math.inf), verify=True, recall_ks=[8])
    rep = run_decode_sim(rmat(steps, 16, 41), rmat(steps, 16, 42), rmat(steps, 16, 43), cfg)
    assert rep.steps == steps
    assert rep.flushes == steps // 64
    assert rep.violations == 0
    assert rep.mean_f_scan == pytest.approx(1.0, abs=1e-12)
    assert rep.recall[8] == pytest.approx(1.0, abs=1e-12)


@pytest.mark.gpu
@pytest.mark.parametrize("algo", [FilterAlgo.FullSubspace, FilterAlgo.Ta])
def test_oracle_threshold_zero_false_negative(torch, algo):  # test_bench.cpp:40-60
    steps = 384
    cfg = DecodeSimConfig(build=BuildConfig(4, 4, "pca_tree", "ball", 0), buffer_capacity=32, algo=algo,
                          threshold=ThresholdSource(oracle=OracleConfig(OracleVariant.Budget, 0, 0.25)),
                          verify=True)
    rep = run_decode_sim(rmat(steps, 32, 51), rmat(steps, 32, 52), rmat(steps, 32, 53), cfg)
    assert rep.steps == steps and rep.violations == 0
    assert 0.0 < rep.mean_f_scan <= 1.0


def oracle_decode(oracle, keys, values, queries, B, oc, cap, seed, strict):
    """bench.cpp:71-120 with the CPU oracle (test-only): per-step selected, retrieved, τ."""
    steps, d = keys.shape
    cache = oracle.Cache(d, oracle.cfg(1, 16, "contiguous", "aabb"), B)
    res = oracle.Reservoir(cap, seed)
    sel, ret, taus = [], [], []
    need = oc.m if oc is not None and oc.variant == OracleVariant.SampleTopK else 1
    for t in range(steps):
        if oc is None:
            tau = np.float32(0.5)
        elif res.size() >= 2 and res.size() >= need:
            tau = oracle.estimate_tau(keys[res.ids()], queries[t], int(oc.variant), m=oc.m, alpha=oc.alpha)
        else:
            tau = np.float32(-np.inf)
        r = cache.query(queries[t], float(tau), algo=1, strict=strict)
        sel.append(r["selected"].size)
        ret.append(r["retrieved"].size)
        taus.append(float(tau) if math.isfinite(tau) else 0.0)
        cache.push_key(keys[t], values[t])
        res.update(t)
    return np.mean(sel), np.mean(ret), np.mean(taus), cache.flush_count()


@pytest.mark.gpu
@pytest.mark.parametrize("oc,strict", [
    (OracleConfig(OracleVariant.Budget, 0, 0.1), False),
    (OracleConfig(OracleVariant.SampleTopK, 5, 0.1), False),
    (OracleConfig(OracleVariant.SampleGap), True),
    (OracleConfig(OracleVariant.SampleMeanMax), False),
    (None, True),
])
def test_decode_matches_oracle_loop(torch, oracle, oc, strict):
    steps, d, B, cap, seed = 600, 32, 48, 64, 9
    keys, values, queries = rmat(steps, d, 61), rmat(steps, d, 62), rmat(steps, d, 63)
    src = ThresholdSource(oracle=oc) if oc is not None else ThresholdSource(fixed_tau=0.5)
    cfg = DecodeSimConfig(build=BuildConfig(1, 16, "contiguous", "aabb", 0), buffer_capacity=B, threshold=src,
                          reservoir_capacity=cap, seed=seed, verify=True, strict_threshold=strict)
    rep = run_decode_sim(keys, values, queries, cfg)
    m_sel, m_ret, m_tau, flushes = oracle_decode(oracle, keys, values, queries, B, oc, cap, seed, strict)
    assert rep.violations == 0
    assert rep.flushes == flushes == steps // B
    assert rep.mean_selected == pytest.approx(m_sel, rel=0, abs=1e-9)
    assert rep.mean_retrieved == pytest.approx(m_ret, rel=0, abs=1e-9)
    assert rep.mean_tau == pytest.approx(m_tau, rel=1e-12, abs=1e-12)
    assert rep.median_query_us > 0.0


# ---------------------------------------------------------------------------------------------
# run_decode_graph: the whole decode loop of a GQA layer captured as CUDA graphs (SURVEY §8(f)
# row 2 at the C2 head shape). Checked step by step against the oracle: every step's τ is the
# oracle's estimate_tau over the reservoir the reference would hold, and every step's selected
# count is the oracle's brute_force_range over the keys stored before the step.


def _graph_case(H_kv, G, d, prefill, steps, seed):
    from paper_2605_06763_b200 import synth

    rows = prefill + steps
    K = np.stack([synth.keys(rows, d, seed + 7 * h) for h in range(H_kv)], axis=1)       # [rows][H][d]
    V = np.stack([synth.keys(rows, d, seed + 7 * h + 1) for h in range(H_kv)], axis=1)
    Q = np.stack([synth.queries(rows * G, d, seed + 7 * h).reshape(rows, G, d) for h in range(H_kv)],
                 axis=1).reshape(rows, H_kv * G, d)
    return K.astype(np.float32), V.astype(np.float32), Q.astype(np.float32)


@pytest.mark.gpu
@pytest.mark.parametrize("dtype", ["bf16", "f32"])
def test_graph_decode_matches_oracle(torch, dtype):
    from oracle import pyoracle
    from paper_2605_06763_b200 import Reservoir
    from paper_2605_06763_b200.decode_sim import run_decode_graph

    H_kv, G, d, prefill, steps, B, cap = 2, 4, 128, 512, 192, 32, 64
    K, V, Q = _graph_case(H_kv, G, d, prefill, steps, 5)
    if dtype == "bf16":  # the oracle sees the stored (bf16) keys
        K = torch.from_numpy(K).to(torch.bfloat16).float().numpy()
        V = torch.from_numpy(V).to(torch.bfloat16).float().numpy()
    cfg = DecodeSimConfig(build=BuildConfig(1, 16, "contiguous", "aabb", 0), buffer_capacity=B,
                          threshold=ThresholdSource(oracle=OracleConfig(OracleVariant.Budget, 0, 0.05)),
                          reservoir_capacity=cap, seed=3)
    rep = run_decode_graph(K, V, Q, H_kv, G, cfg, prefill, dtype=dtype, steps_per_graph=8, verify=True)
    assert rep.steps == steps and rep.n_final == prefill + steps
    assert rep.flushes == steps // B  # the prompt is indexed at build, not flushed
    assert rep.violations == 0
    res = Reservoir(cap, 3)
    for t in range(prefill):
        res.update(t)
    for i, t in enumerate(range(prefill, prefill + steps)):
        ids = res.ids()
        for hq in range(H_kv * G):
            h = hq // G
            want_tau = pyoracle.estimate_tau(K[ids, h], Q[t, hq], 4, alpha=0.05)
            assert rep.taus[i, hq] == want_tau, (t, hq)
            want = pyoracle.brute_force_range(K[:t, h], Q[t, hq], want_tau)
            assert rep.selected[i, hq] == want.size, (t, hq)
        res.update(t)
