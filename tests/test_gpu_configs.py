"""GPU parity at the BASELINE.json configuration shapes, on the bench's own inputs.

C2 and C3 use bench.py's generators (gen_layer: the reference key law io.cpp:145-169 with
sign-aligned queries io.cpp:186-202) and its tau rule (the ceil(0.05 n)-th largest score),
so the launch geometry under test is the one bench.py times: C2 = 8 slots with a team of
CTAs per slot and the team merge, C3 = 128 slots, one CTA per slot. C1 is the single-head
fp32 cache at 32K keys; C4 is the decode loop (query, then push_key, bench.cpp:91-118) at
the C2 head shape with an 8K prompt, across two flushes at B = 128.

Selected ids are compared with the oracle's brute_force_range bit for bit on every q head;
attention outputs within REL_TOL of the oracle's sparse_attention (anchored to float64
attention where the reference's own fp32 result drifts, as in test_gpu_parity)."""
import concurrent.futures as cf
import math
import os

import numpy as np
import pytest

import bench
from paper_2605_06763_b200 import (BuildConfig, FilterAlgo, LouverCache, LouverLayer, QueryRequest, synth)

pytestmark = pytest.mark.gpu

REL_TOL = 1e-4
THREADS = max(1, os.cpu_count() or 1)


@pytest.fixture(scope="module")
def torch():
    import torch

    assert torch.cuda.is_available(), "GPU tests need a CUDA device"
    return torch


def rel_err(a, b):
    return float(np.linalg.norm(np.asarray(a, np.float64) - b) / max(np.linalg.norm(b), 1e-30))


def exact_attention(kh, vh, q, att):
    s = (kh[att].astype(np.float64) @ q.astype(np.float64)) / math.sqrt(q.size)
    w = np.exp(s - s.max())
    return (w[:, None] * vh[att].astype(np.float64)).sum(0) / w.sum()


def bf16(torch, a):
    return torch.from_numpy(np.ascontiguousarray(a, np.float32)).to(torch.bfloat16).float().numpy()


def run_layer(torch, layer, Q, tau, strict=False):
    B, H_q, d = Q.shape
    qd, td = torch.from_numpy(np.ascontiguousarray(Q)).cuda(), torch.from_numpy(tau).cuda()
    out = torch.zeros((B, H_q, d), dtype=torch.float32, device="cuda")
    bits = torch.zeros((B * H_q, layer.bitmap_words), dtype=torch.int32, device="cuda")
    counts = torch.zeros((B, H_q, 4), dtype=torch.int32, device="cuda")
    layer.query_device(qd, td, out, strict=strict, sel_bits=bits, counts=counts)
    torch.cuda.synchronize()
    return layer.ids_from_bits(bits), out.cpu().numpy(), counts.cpu().numpy()


def check_heads(oracle, K, V, Q, tau, G, ids, outs, cnt, heads, *, n, indexed, strict=False, outputs=None):
    """Every (b, hq) in `heads`: ids == oracle brute force; for (b, hq) in `outputs` (default:
    all of `heads`) the attention output against the oracle, anchored to float64."""
    B, H_q, d = Q.shape
    outputs = set(heads if outputs is None else outputs)
    scale = np.float32(1 / math.sqrt(d))

    def one(bh):
        b, hq = bh
        kh, vh = K[b, hq // G, :n], V[b, hq // G, :n]
        want = oracle.brute_force_range(kh, Q[b, hq], tau[b, hq])
        row = b * H_q + hq
        errs = []
        if not np.array_equal(ids[row], want):
            errs.append(f"ids (b={b}, hq={hq}): got {ids[row].size}, want {want.size}")
        if cnt[b, hq, 0] != want.size:
            errs.append(f"count (b={b}, hq={hq})")
        if bh in outputs:
            att = want if strict else np.union1d(want[want < indexed], np.arange(indexed, n))
            ow = oracle.sparse_attention(kh, vh, [], att, Q[b, hq], scale)
            if ow is None:
                if cnt[b, hq, 3] != 0 or outs[b, hq].any():
                    errs.append(f"empty set (b={b}, hq={hq})")
            else:
                e = rel_err(outs[b, hq], ow[2])
                if e > REL_TOL:
                    ex = exact_attention(kh, vh, Q[b, hq], att)
                    if rel_err(outs[b, hq], ex) > max(REL_TOL, 2 * rel_err(ow[2], ex)):
                        errs.append(f"output (b={b}, hq={hq}): rel {e:.2e}")
        return errs

    with cf.ThreadPoolExecutor(THREADS) as ex:
        errs = [e for r in ex.map(one, heads) for e in r]
    assert not errs, errs[:10]


def bench_layer(torch, name):
    cfg = dict(bench.CONFIGS[name])
    K, V, Q = bench.gen_layer(cfg, 0, 0, THREADS)
    B, H, n, d = K.shape
    dt = cfg["dtype"]
    if dt == "bf16":
        K, V = bf16(torch, K), bf16(torch, V)
    tau = bench.taus_device(torch, K, Q, cfg["G"], bench.SELECTIVITY)
    layer = LouverLayer(d, H, cfg["G"], B, n, BuildConfig(S=1, r=bench.CELL, grouping="contiguous",
                                                         enclosing="aabb"), buffer_capacity=128, dtype=dt)
    layer.build(K, V)
    return cfg, layer, K, V, Q, tau


def test_c2_bench_inputs_all_heads(torch, oracle):
    """C2 exactly as bench.py builds layer 0: 8 slots x 131072 keys, 32 q heads, team merge."""
    cfg, layer, K, V, Q, tau = bench_layer(torch, "c2")
    ids, outs, cnt = run_layer(torch, layer, Q, tau)
    geo = layer.geometry()
    assert geo["team_ctas_per_slot"] > 1  # the team/merge geometry the bench times
    heads = [(0, hq) for hq in range(32)]
    check_heads(oracle, K, V, Q, tau, 4, ids, outs, cnt, heads, n=layer.n, indexed=layer.indexed_count)
    # strict on a quarter of the heads (attends selected only)
    ids_s, outs_s, cnt_s = run_layer(torch, layer, Q, tau, strict=True)
    check_heads(oracle, K, V, Q, tau, 4, ids_s, outs_s, cnt_s, heads[::4], n=layer.n,
                indexed=layer.indexed_count, strict=True)


def test_c3_batch16_one_cta_per_slot(torch, oracle):
    """C3 exactly as bench.py builds it: batch 16 x 8 kv heads x 32768 keys = 128 slots, which the
    launch serves with one CTA per slot (no team merge)."""
    cfg, layer, K, V, Q, tau = bench_layer(torch, "c3")
    ids, outs, cnt = run_layer(torch, layer, Q, tau)
    assert layer.geometry()["team_ctas_per_slot"] == 1
    heads = [(b, hq) for b in range(16) for hq in range(32)]
    check_heads(oracle, K, V, Q, tau, 4, ids, outs, cnt, heads, n=layer.n, indexed=layer.indexed_count)


def test_c1_fp32_single_head_32k(torch, oracle):
    """C1: one head, 32768 fp32 keys, d = 128, fixed tau — through LouverCache (the reference's
    single-head API) and through the bench's LouverLayer(f32) form."""
    n, d = 32768, 128
    k, v = synth.keys(n, d, 1234), synth.keys(n, d, 1235)
    qs = synth.queries(3, d, 1234)
    c = LouverCache.adopt(k, v, BuildConfig(S=4, r=4), 128)
    scale = np.float32(1 / math.sqrt(d))
    for i, q in enumerate(qs):
        sc = oracle.scores(k, q)
        for frac in (0.01, 0.05, 0.10):
            tau = np.sort(sc)[::-1][int(math.ceil(frac * n)) - 1]
            res = c.query(QueryRequest(q=q, tau=float(tau)), FilterAlgo.Ta)
            want = oracle.brute_force_range(k, q, tau)
            assert np.array_equal(res.selected, want), (i, frac)
            ow = oracle.sparse_attention(k, v, [], want, q, scale)
            assert rel_err(res.attention.output, ow[2]) <= REL_TOL, (i, frac)
    cfg, layer, K, V, Q, tau = bench_layer(torch, "c1")
    ids, outs, cnt = run_layer(torch, layer, Q, tau)
    check_heads(oracle, K, V, Q, tau, 1, ids, outs, cnt, [(0, 0)], n=layer.n, indexed=layer.indexed_count)


def test_c4_decode_loop_at_c2_shape(torch, oracle):
    """C4 semantics at the C2 head shape (8 kv / 32 q heads, bf16, d = 128): an 8192-key prompt,
    then query-then-insert steps (bench.cpp:91-118) across two flushes at B = 128; at each checked
    step the selected ids of every q head equal the oracle's, and the outputs (buffer attended
    densely until each flush, cache.cpp:48-68) match."""
    H, G, d, n0, steps, B = 8, 4, 128, 8192, 300, 128
    seeds = np.array([bench.layer_seeds(3, 0, 0, h, H) for h in range(H)], np.uint64)
    Kf = bf16(torch, synth.keys_multi(n0 + steps, d, seeds, THREADS))[None]
    Vf = bf16(torch, synth.keys_multi(n0 + steps, d, seeds + np.uint64(1), THREADS))[None]
    Q = np.stack([synth.queries(G, d, int(s)) for s in seeds]).reshape(1, H * G, d)
    layer = LouverLayer(d, H, G, 1, n0 + steps, BuildConfig(S=1, r=16, grouping="contiguous", enclosing="aabb"),
                        buffer_capacity=B, dtype="bf16")
    layer.build(Kf[:, :, :n0], Vf[:, :, :n0])
    checked = {0, 1, 63, 127, 128, 129, 200, 255, 256, 299}
    heads = [(0, hq) for hq in range(H * G)]
    for t in range(steps):
        n = n0 + t
        if t in checked:
            tau = np.zeros((1, H * G), np.float32)
            for hq in range(H * G):
                tau[0, hq] = oracle.kth_score(Kf[0, hq // G, :n], Q[0, hq], int(math.ceil(0.05 * n)))
            ids, outs, cnt = run_layer(torch, layer, Q, tau)
            check_heads(oracle, Kf, Vf, Q, tau, G, ids, outs, cnt, heads, n=n, indexed=layer.indexed_count,
                        outputs=heads[::3])
        kt = torch.from_numpy(np.ascontiguousarray(Kf[0, :, n])).cuda()
        vt = torch.from_numpy(np.ascontiguousarray(Vf[0, :, n])).cuda()
        layer.push_key(kt, vt)
    torch.cuda.synchronize()
    assert layer.flush_count == steps // B
    assert layer.n == n0 + steps and layer.indexed_count == n0 + (steps // B) * B
