#!/usr/bin/env python
"""Louver decode hot path on B200: µs per decode step per layer at 128K context.

    python bench.py [--gpus N --steps K --warmup W] [--config c2] [--impl reference]

Workload (default, BASELINE.json configs[1], "C2"): a Llama-3-8B-shaped decode
layer — 32 q heads / 8 kv heads (G=4), d=128, 131072 cached keys, batch 1,
bf16 K/V — with the reference's synthetic decode-trace key law (io.cpp:145-169)
and sign-aligned queries (io.cpp:186-202); tau per q head = the ceil(0.05 n)-th
largest score (fixed tau). A "step" is one decode query through every one of
L=8 independent layers (distinct synthetic data, 4 GiB of KV in total), so the
bytes a step touches (~0.7 GB) exceed the 126 MB L2 and no flush is needed
between iterations; value = step time / L.

N>1 (torchrun): the KV cache is sequence-sharded, 131072 keys per GPU per layer
(weak scaling; at N=8 the context is 2^20, config C5); each rank runs the same
fused kernel on its shard and emits (m, l, o) partials, which are all-gathered
over NCCL and merged with a log-sum-exp combine kernel.

--impl reference: the reference library's own CPU path — its unmodified sources
compiled here into oracle/_ref (the build travels with the repo) or, where that
build is absent, the oracle restatement — LouverCache::query with the reference
defaults S=4, r=4, PCA tree, ball, FilterAlgo::Ta, on the same data, all host
threads, rank 0 only.
"""
from __future__ import annotations

import argparse
import json
import math
import os
import statistics
import sys
import threading
import time

import numpy as np

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

METRIC = "decode attention µs/step/layer at 128K ctx, recall=1; HBM GB/s vs roofline"
UNIT = "us/step/layer"

CONFIGS = {
    # name: (batch, H_kv, G, d, n per GPU, dtype, layers)
    "c1": dict(batch=1, H_kv=1, G=1, d=128, n=32768, dtype="f32", layers=8,
               workload="C1 single-head decode, d=128, 32K keys, fixed tau, fp32"),
    "c2": dict(batch=1, H_kv=8, G=4, d=128, n=131072, dtype="bf16", layers=8,
               workload="C2 Llama-3-8B-shaped decode layer (32 q / 8 kv heads, d=128), 128K ctx, batch 1, bf16 KV"),
    "c3": dict(batch=16, H_kv=8, G=4, d=128, n=32768, dtype="bf16", layers=2,
               workload="C3 same shape, batch 16 at 32K ctx, GQA-grouped probing"),
    # C5's 1M-token context on ONE GPU (the unsharded point of the 2/4/8-GPU curve: with
    # --gpus P under torchrun each rank holds n / P of it)
    "c5": dict(batch=1, H_kv=8, G=4, d=128, n=1048576, dtype="bf16", layers=2,
               workload="C5 1M-token context, C2 head shape, one GPU (unsharded)"),
}
SELECTIVITY = 0.05
CELL = 16


def log(*a):
    print(*a, file=sys.stderr, flush=True)


# ----------------------------------------------------------------------------- data


def layer_seeds(layer: int, rank: int, b: int, h: int, H_kv: int) -> int:
    return 1_000_003 * (layer + 1) + 10_007 * rank + 1000 * (b * H_kv + h) + 17


def gen_layer(cfg, layer, rank, threads, qsteps=1):
    """K, V [batch][H_kv][n][d] fp32 (reference key law), Q [batch][H_q][d]; with qsteps > 1,
    Q is [qsteps][batch][H_q][d]: consecutive decode queries of the same stream
    (gen_synthetic_queries rows, io.cpp:186-202; step 0 = the single-query rows)."""
    from paper_2605_06763_b200 import synth

    B, H, G, d, n = cfg["batch"], cfg["H_kv"], cfg["G"], cfg["d"], cfg["n"]
    seeds = np.array([layer_seeds(layer, rank, b, h, H) for b in range(B) for h in range(H)], np.uint64)
    K = synth.keys_multi(n, d, seeds, threads).reshape(B, H, n, d)
    V = synth.keys_multi(n, d, seeds + np.uint64(1), threads).reshape(B, H, n, d)
    # queries follow the layer's key stream direction (independent of the rank's shard)
    R = max(1, qsteps)
    Q = np.stack([np.stack([synth.queries(G * R, d, int(layer_seeds(layer, 0, b, h, H))).reshape(R, G, d)
                            for h in range(H)], axis=1) for b in range(B)], axis=1)  # [R][B][H][G][d]
    Q = Q.reshape(R, B, H * G, d)
    return (K, V, Q[0]) if qsteps <= 1 else (K, V, Q)


def top_scores(torch, K, Q, G, k):
    """[B][H*G][k] descending: the k largest q.k per q head (bf16-rounded K as stored, fp64)."""
    B, H, n, d = K.shape
    k = min(k, n)
    out = torch.empty((B, H * G, k), dtype=torch.float64, device="cuda")
    for b in range(B):
        for h in range(H):
            kh = torch.from_numpy(K[b, h]).cuda().to(torch.bfloat16).double()
            qh = torch.from_numpy(Q[b, h * G:(h + 1) * G]).cuda().double()
            s = kh @ qh.T  # [n][G]
            out[b, h * G:(h + 1) * G] = torch.topk(s, k, dim=0).values.T
    return out


def taus_device(torch, K, Q, G, frac, world=1, dist=None):
    """tau[b][hq] = the ceil(frac * n_total)-th largest q.k over the whole (possibly
    sequence-sharded) context: each rank's top-k candidates are all-gathered and the k-th
    of their union is taken, so every rank uses the global threshold."""
    n_total = K.shape[2] * world
    k = max(1, int(math.ceil(frac * n_total)))
    top = top_scores(torch, K, Q, G, k)
    if world > 1:
        pad = torch.full((top.shape[0], top.shape[1], k), -float("inf"), dtype=torch.float64, device="cuda")
        pad[..., :top.shape[2]] = top
        allt = [torch.empty_like(pad) for _ in range(world)]
        dist.all_gather(allt, pad)
        top = torch.topk(torch.cat(allt, dim=2), k, dim=2).values
    return top[..., k - 1].float().cpu().numpy()


def graph_time(torch, fn, reps, per):
    """Median over `reps` replays of a CUDA graph of fn() (after warm-up), divided by `per`."""
    s = torch.cuda.Stream()
    s.wait_stream(torch.cuda.current_stream())
    with torch.cuda.stream(s):
        for _ in range(2):
            fn()
    torch.cuda.current_stream().wait_stream(s)
    torch.cuda.synchronize()
    g = torch.cuda.CUDAGraph()
    with torch.cuda.graph(g):
        fn()
    for _ in range(5):
        g.replay()
    torch.cuda.synchronize()
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    ts = []
    for _ in range(reps):
        a.record()
        g.replay()
        b.record()
        b.synchronize()
        ts.append(a.elapsed_time(b) * 1e3 / per)
    del g
    return statistics.median(ts)


# ---------------------------------------------------------------------------- clocks


class ClockSampler:
    """NVML sampler of SM clock and throttle reasons while the timed region runs."""

    REASONS = {
        0x1: "gpu_idle", 0x2: "applications_clocks_setting", 0x4: "sw_power_cap", 0x8: "hw_slowdown",
        0x10: "sync_boost", 0x20: "sw_thermal_slowdown", 0x40: "hw_thermal_slowdown",
        0x80: "hw_power_brake_slowdown", 0x100: "display_clock_setting",
    }

    def __init__(self, index: int):
        self.samples, self.reasons, self._stop = [], set(), threading.Event()
        self.max_mhz = None
        try:
            import pynvml

            pynvml.nvmlInit()
            self.nv = pynvml
            self.h = pynvml.nvmlDeviceGetHandleByIndex(index)
            self.max_mhz = pynvml.nvmlDeviceGetMaxClockInfo(self.h, pynvml.NVML_CLOCK_SM)
        except Exception as e:  # pragma: no cover
            log("nvml unavailable:", e)
            self.nv = None

    def _run(self):
        while not self._stop.is_set():
            try:
                self.samples.append(self.nv.nvmlDeviceGetClockInfo(self.h, self.nv.NVML_CLOCK_SM))
                mask = self.nv.nvmlDeviceGetCurrentClocksEventReasons(self.h)
                for bit, name in self.REASONS.items():
                    if mask & bit and name != "gpu_idle":
                        self.reasons.add(name)
            except Exception:
                pass
            time.sleep(0.01)

    def __enter__(self):
        if self.nv:
            self.t = threading.Thread(target=self._run, daemon=True)
            self.t.start()
        return self

    def __exit__(self, *a):
        self._stop.set()
        if self.nv:
            self.t.join()

    def summary(self):
        med = statistics.median(self.samples) if self.samples else None
        return {"sm_mhz": med, "sm_max_mhz": self.max_mhz, "reasons": sorted(self.reasons),
                "samples": len(self.samples)}


# --------------------------------------------------------------------- CPU baseline


def cpu_reference():
    """The reference library's CPU path: oracle/_ref (the reference's own sources compiled
    here, travels with the repo; kind "reference") when present, else the oracle restatement
    (kind "port")."""
    from oracle import pyoracle

    ref = pyoracle.reference_module()
    return (ref, "reference") if ref is not None else (pyoracle, "port")


def oracle_cache_for(K_head, V_head, mod=None):
    if mod is None:
        mod = cpu_reference()[0]
    return mod.Cache(K_head.shape[1], mod.cfg(4, 4, "pca_tree", "ball"), 128, keys=K_head, values=V_head)


def cpu_baseline_sample(K, V, Q, tau, G, budget_s=20.0):
    """Reference CPU path (oracle port, reference defaults, FilterAlgo::Ta, one
    thread as in the reference) on kv head 0 of layer 0: time its G q-head
    queries, scale to all q heads of the layer."""
    import torch

    Kh = torch.from_numpy(K[0, 0]).to(torch.bfloat16).float().numpy()
    Vh = torch.from_numpy(V[0, 0]).to(torch.bfloat16).float().numpy()
    mod, kind = cpu_reference()
    t0 = time.perf_counter()
    cache = oracle_cache_for(Kh, Vh, mod)
    build_s = time.perf_counter() - t0
    times = []
    t_end = time.perf_counter() + budget_s
    reps = 0
    while time.perf_counter() < t_end and reps < 5:
        for g in range(G):
            t1 = time.perf_counter()
            cache.query(Q[0, g], float(tau[0, g]), algo=1)
            times.append(time.perf_counter() - t1)
        reps += 1
    per_head = statistics.median(times)
    H_q = Q.shape[0] * Q.shape[1]
    return {
        "value": per_head * H_q * 1e6,
        "unit": UNIT,
        "cores": 1,
        "kind": kind,
        "sample": f"{'reference build (oracle/_ref)' if kind == 'reference' else 'oracle port'} "
                  f"LouverCache::query (S=4,r=4,pca_tree,ball,Ta) on kv head 0 of layer 0 "
                  f"({Kh.shape[0]} keys): median of {len(times)} single-thread q-head queries x {H_q} q heads; "
                  f"index build {build_s:.1f}s excluded",
    }


# --------------------------------------------------------------------- reference arm


def run_reference(args, cfg):
    import concurrent.futures as cf

    import torch

    threads = os.cpu_count() or 1
    K, V, Q = gen_layer(cfg, 0, 0, threads)
    B, H, n, d = K.shape
    G = cfg["G"]
    K = torch.from_numpy(K).to(torch.bfloat16).float().numpy() if cfg["dtype"] == "bf16" else K
    V = torch.from_numpy(V).to(torch.bfloat16).float().numpy() if cfg["dtype"] == "bf16" else V
    tau = np.zeros((B, H * G), np.float32)
    from oracle import pyoracle

    kk = max(1, int(math.ceil(SELECTIVITY * n)))
    with cf.ThreadPoolExecutor(threads) as ex:
        jobs = {(b, hq): ex.submit(pyoracle.kth_score, K[b, hq // G], Q[b, hq], kk)
                for b in range(B) for hq in range(H * G)}
        for (b, hq), f in jobs.items():
            tau[b, hq] = f.result()
        mod, kind = cpu_reference()
        t0 = time.perf_counter()
        caches = {(b, h): ex.submit(oracle_cache_for, K[b, h], V[b, h], mod) for b in range(B) for h in range(H)}
        caches = {k: f.result() for k, f in caches.items()}
    build_s = time.perf_counter() - t0
    heads = [(b, hq) for b in range(B) for hq in range(H * G)]
    per_step = min(len(heads), threads)  # bounded sample: one q head per host thread per step

    def one(i):
        b, hq = heads[i % len(heads)]
        caches[(b, hq // G)].query(Q[b, hq], float(tau[b, hq]), algo=1)

    times = []
    cursor = 0
    with cf.ThreadPoolExecutor(threads) as ex:
        for step in range(args.warmup + args.steps):
            t1 = time.perf_counter()
            list(ex.map(one, range(cursor, cursor + per_step)))
            dt = time.perf_counter() - t1
            cursor += per_step
            if step >= args.warmup:
                times.append(dt * len(heads) / per_step)
    value = statistics.mean(times) * 1e6
    line = {
        "impl": "reference", "metric": METRIC, "value": value, "unit": UNIT, "n_gpus": args.gpus,
        "steps": args.steps, "warmup": args.warmup, "ms_per_step": value / 1e3, "higher_is_better": False,
        "scaling": "weak", "vs_baseline": None, "dtype": "f32", "data": "synthetic",
        "config": {"workload": cfg["workload"] + " (one layer)", "n": n, "H_q": H * G, "H_kv": H, "d": d,
                   "batch": B, "selectivity": SELECTIVITY, "tau": "fixed, ceil(0.05 n)-th largest score",
                   "build": "reference defaults S=4 r=4 pca_tree ball, FilterAlgo::Ta"},
        "cpu_baseline": {"value": value, "unit": UNIT, "cores": threads, "kind": kind,
                         "sample": f"each step: {per_step} of {len(heads)} q-head queries in parallel on "
                                   f"{threads} threads, scaled to all q heads; index build {build_s:.1f}s excluded"},
        "e2e": {"value": value, "unit": UNIT, "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
    }
    print(json.dumps(line), flush=True)


# ------------------------------------------------------------------------- GPU arm


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=500)
    ap.add_argument("--warmup", type=int, default=5)
    ap.add_argument("--config", default="c2", choices=sorted(CONFIGS))
    ap.add_argument("--layers", type=int, default=0)
    ap.add_argument("--impl", default="louver", choices=["louver", "reference"])
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--no-graph", action="store_true")
    ap.add_argument("--no-dense-lib", action="store_true", help="skip the library (torch SDPA) dense decode")
    ap.add_argument("--qsteps", type=int, default=4,
                    help="distinct consecutive decode queries per layer, cycled through the timed steps")
    args = ap.parse_args()
    args.warmup = max(3, args.warmup)

    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    cfg = dict(CONFIGS[args.config])
    if args.layers:
        cfg["layers"] = args.layers

    if args.impl == "reference":
        if rank == 0:
            run_reference(args, cfg)
        return

    import torch
    import torch.distributed as dist

    torch.cuda.set_device(local)
    if world > 1:
        dist.init_process_group("nccl", device_id=torch.device("cuda", local))
    from paper_2605_06763_b200 import BuildConfig, LouverLayer, lse_merge

    threads = max(1, (os.cpu_count() or 1) // max(1, world))
    B, H, G, d, n, L = cfg["batch"], cfg["H_kv"], cfg["G"], cfg["d"], cfg["n"], cfg["layers"]
    H_q = H * G
    rows = B * H_q
    e = 2 if cfg["dtype"] == "bf16" else 4
    build_cfg = BuildConfig(S=1, r=CELL, grouping="contiguous", enclosing="aabb")

    layers, qs, taus, outs, kts, vts = [], [], [], [], [], []
    qsets, tsets = [], []  # [L][R]: the decode stream's consecutive queries and their tau
    R = max(1, args.qsteps)
    first = None
    t0 = time.perf_counter()
    for l in range(L):
        K, V, QR = gen_layer(cfg, l, rank, threads, qsteps=R if R > 1 else 1)
        QR = QR if R > 1 else QR[None]
        Q = QR[0]
        layer = LouverLayer(d, H, G, B, n, build_cfg, buffer_capacity=128, dtype=cfg["dtype"])
        layer.build(K, V)
        tr = [taus_device(torch, K, QR[i], G, SELECTIVITY, world, dist if world > 1 else None) for i in range(R)]
        tau = tr[0]
        qsets.append([torch.from_numpy(QR[i]).cuda() for i in range(R)])
        tsets.append([torch.from_numpy(tr[i]).cuda() for i in range(R)])
        layers.append(layer)
        if not args.no_dense_lib:  # [B][H][n][d] copies (config dtype) for the library dense decode (SDPA)
            tdt = torch.bfloat16 if cfg["dtype"] == "bf16" else torch.float32
            kts.append(torch.from_numpy(K).to("cuda", tdt))
            vts.append(torch.from_numpy(V).to("cuda", tdt))
        qs.append(qsets[-1][0])
        taus.append(tsets[-1][0])
        outs.append(torch.zeros((B, H_q, d), dtype=torch.float32, device="cuda"))
        if l == 0:
            first = (K, V, Q, tau)
        del K, V
    setup_s = time.perf_counter() - t0
    log(f"[rank {rank}] setup {setup_s:.1f}s: {L} layers x {B}x{H} slots x {n} keys ({cfg['dtype']})")

    # ---- per-layer work accounting (outside the timed region), averaged over the R queries
    totals = torch.zeros((R, L, 4), dtype=torch.int64, device="cuda")
    counts = torch.zeros((R, L, B, H_q, 4), dtype=torch.int32, device="cuda")
    for i in range(R):
        for l in range(L):
            layers[l].query_device(qsets[l][i], tsets[l][i], outs[l], totals=totals[i, l], counts=counts[i, l])
    torch.cuda.synchronize()
    tot = totals.cpu().numpy().astype(np.float64).reshape(R * L, 4)
    cnt = counts.cpu().numpy().astype(np.float64)
    # partials: [slots][splits][G][d+2] fp32 written by every CTA, read by the merge
    slots = B * H
    b_sum = tot[:, 0] * 2 * d * e
    b_key = tot[:, 2] * d * e
    b_val = tot[:, 3] * d * e
    b_qo = rows * (d * 4 * 2 + 4)
    geo = layers[0].geometry()
    team = geo.get("team_ctas_per_slot") or geo["splits"]  # bf16: fused kernel team; fp32: splits
    ctas = slots * team
    if geo.get("ctas_per_sm"):  # bf16 teams of nb and nb - 1 CTAs fill the resident wave exactly
        ctas = min(ctas, geo["ctas_per_sm"] * torch.cuda.get_device_properties(0).multi_processor_count)
    geo["layer_ctas"] = int(ctas)
    b_part = ctas * G * (d + 2) * 4 * 2
    alg_bytes = float(np.mean(b_sum + b_key + b_val)) + b_qo + b_part
    dense_bytes = float(slots * n * d * e * 2 + b_qo)
    keys_scanned = float(np.mean(cnt[..., 2]))
    keys_selected = float(np.mean(cnt[..., 0]))
    keys_attended = float(np.mean(cnt[..., 1]))

    # ---- one step = L layers (sharded: + all-gather + LSE merge per layer)
    if world > 1:
        parts = [torch.zeros((B, H_q, d + 2), dtype=torch.float32, device="cuda") for _ in range(L)]
        gathered = [torch.zeros((world, B * H_q, d + 2), dtype=torch.float32, device="cuda") for _ in range(L)]

    def step(i=0):  # decode step i of the stream: query i % R of every layer
        for l in range(L):
            q, t = qsets[l][i % R], tsets[l][i % R]
            if world > 1:
                layers[l].query_device(q, t, None, partial=parts[l])
                dist.all_gather_into_tensor(gathered[l], parts[l].view(B * H_q, d + 2))
                lse_merge(gathered[l], outs[l].view(B * H_q, d))
            else:
                layers[l].query_device(q, t, outs[l])

    def steps_block():  # R consecutive decode steps
        for i in range(R):
            step(i)

    graph = None
    if world == 1 and not args.no_graph:
        s = torch.cuda.Stream()
        s.wait_stream(torch.cuda.current_stream())
        with torch.cuda.stream(s):
            steps_block()  # warm the lazy attribute setup outside capture
        torch.cuda.current_stream().wait_stream(s)
        torch.cuda.synchronize()
        graph = torch.cuda.CUDAGraph()
        with torch.cuda.graph(graph):
            steps_block()
    # one run = R decode steps; the timed region is ceil(steps / R) runs
    run = graph.replay if graph is not None else steps_block
    args.steps = -(-args.steps // R) * R

    for _ in range(-(-args.warmup // R)):
        run()
    torch.cuda.synchronize()
    if world > 1:
        dist.barrier()
    torch.cuda.synchronize()
    ev0, ev1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    with ClockSampler(local) as clocks:
        ev0.record()
        for _ in range(args.steps // R):
            run()
        ev1.record()
        torch.cuda.synchronize()
    ms_total = ev0.elapsed_time(ev1)
    if world > 1:
        t = torch.tensor([ms_total], device="cuda")
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        ms_total = float(t.item())
        dist.barrier()
    ms_step = ms_total / args.steps
    us_layer = ms_step * 1e3 / L

    # ---- dominant kernel: one fused kernel per layer, so the timed step is L back-to-back
    # launches of it (graph replay, no host work between them): its average launch
    # duration is the step time / L. A single launch bracketed by events is also
    # reported; it includes the host->GPU launch latency.
    reps = max(20, min(200, args.steps))
    kern_ms = []
    ka, kb = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    for i in range(reps):
        l = i % L
        ka.record()
        layers[l].query_device(qs[l], taus[l], outs[l])
        kb.record()
        kb.synchronize()
        kern_ms.append(ka.elapsed_time(kb))
    single_us = statistics.mean(kern_ms) * 1e3
    kern_us = us_layer if (graph is not None and world == 1) else single_us

    # ---- dense full-scan baselines on the same L layers, timed like the metric: a CUDA graph
    # of L launches, median replay time / L after warm-up
    def dense_all():
        for l in range(L):
            layers[l].dense_decode(qs[l], outs[l])

    dense_us = graph_time(torch, dense_all, 50, L)

    # ---- the threshold oracle on the device: estimate_tau for every
    # q head of a layer from a 256-id reservoir per kv slot (budget:0.05), one launch
    tau_oracle = None
    try:
        from paper_2605_06763_b200 import OracleConfig, OracleVariant, Reservoir, estimate_tau_layer

        res_cap = 256
        rids = np.zeros((layers[0].batch * layers[0].H_kv, res_cap), np.uint32)
        n0 = layers[0].n
        for s_ in range(rids.shape[0]):
            rv = Reservoir(res_cap, 1000 * s_ + 1)
            for t_ in range(0, n0, max(1, n0 // 4096)):
                rv.update(t_)
            rids[s_] = rv.ids()
        rids_d = torch.from_numpy(rids).cuda()
        tcfg = OracleConfig(OracleVariant.Budget, alpha=SELECTIVITY)
        tau_bufs = [torch.empty_like(taus[0]) for _ in range(L)]
        side = torch.cuda.Stream()
        side.wait_stream(torch.cuda.current_stream())
        with torch.cuda.stream(side):
            for l in range(L):
                estimate_tau_layer(layers[l], rids_d, res_cap, qs[l], tcfg, tau_bufs[l])
        torch.cuda.current_stream().wait_stream(side)
        torch.cuda.synchronize()
        tg = torch.cuda.CUDAGraph()
        with torch.cuda.graph(tg):
            for l in range(L):
                estimate_tau_layer(layers[l], rids_d, res_cap, qs[l], tcfg, tau_bufs[l])
        tg.replay()
        torch.cuda.synchronize()
        tm = []
        for _ in range(20):
            ka.record()
            tg.replay()
            kb.record()
            kb.synchronize()
            tm.append(ka.elapsed_time(kb) / L)
        tau_oracle = {"us_per_layer": statistics.median(tm) * 1e3, "reservoir": res_cap,
                      "oracle": f"budget:{SELECTIVITY}", "q_heads": int(qs[0].numel() // d),
                      "how": "estimate_tau for all q heads of a layer, one launch; CUDA graph of L launches, "
                             "replay time / L, median of 20"}
    except Exception as ex:  # pragma: no cover
        log(f"threshold oracle timing unavailable: {ex}")

    # ---- library dense decode: torch SDPA (its flash / cuDNN kernel; the fastest dense decode
    # in this image at C2, tools/dense_compare.py) over the same L layers, timed the same way
    sdpa_us = None
    if kts:
        try:
            import torch.nn.functional as F

            qb = [q.to(kts[0].dtype).view(B, H_q, 1, d) for q in qs]

            def sdpa_all():
                for l in range(L):
                    F.scaled_dot_product_attention(qb[l], kts[l], vts[l], enable_gqa=True)

            sdpa_us = graph_time(torch, sdpa_all, 50, L)
        except Exception as ex:  # pragma: no cover - library path unavailable
            log(f"sdpa baseline unavailable: {ex}")
        del kts[:], vts[:]

    # ---- end to end through the public API with host buffers (pinned), one decode step at a
    # time: the step's q and tau go host->device in one copy each, the L layer queries run
    # back to back on the stream (lv_query), the L outputs come back in one copy, then the
    # host waits for the stream. Also reported: one synchronous lv_query(LV_HOST) per layer.
    q_all_h = torch.stack([q.cpu() for q in qs]).pin_memory()      # [L][B][H_q][d]
    t_all_h = torch.stack([t.cpu() for t in taus]).pin_memory()    # [L][B][H_q]
    o_all_h = torch.empty((L, B, H_q, d), dtype=torch.float32).pin_memory()

    from paper_2605_06763_b200 import LayersStep

    q_np, t_np, o_np = q_all_h.numpy(), t_all_h.numpy(), o_all_h.numpy()
    e2e_stream = torch.cuda.Stream()  # a non-default stream: lv_query_layers replays its cached graph
    e2e_stream.wait_stream(torch.cuda.current_stream())
    torch.cuda.synchronize()
    host_step = LayersStep(layers, q_np, t_np, o_np, stream=e2e_stream.cuda_stream) if world == 1 else None

    def e2e_step():
        if world > 1:  # the sharded step: per-layer inputs, shard queries + all-gather + LSE merge
            for l in range(L):
                qs[l].copy_(q_all_h[l], non_blocking=True)
                taus[l].copy_(t_all_h[l], non_blocking=True)
            step()
            for l in range(L):
                o_all_h[l].copy_(outs[l], non_blocking=True)
            torch.cuda.current_stream().synchronize()
        else:  # the C ABI's host-buffer decode step (lv_query_layers): one copy in, L queries, one out
            host_step()

    e2e_steps = max(5, min(50, args.steps))
    for _ in range(3):
        e2e_step()
    t1 = time.perf_counter()
    for _ in range(e2e_steps):
        e2e_step()
    e2e_us = (time.perf_counter() - t1) * 1e6 / (e2e_steps * L)
    # one synchronous host-buffer call per layer (lv_query with LV_HOST)
    qn = [q_all_h[l].numpy() for l in range(L)]
    tn = [t_all_h[l].numpy() for l in range(L)]
    on = [o_all_h[l].numpy() for l in range(L)]
    for l in range(L):
        layers[l].query_host(qn[l], tn[l], out=on[l])
    t2 = time.perf_counter()
    for _ in range(e2e_steps):
        for l in range(L):
            layers[l].query_host(qn[l], tn[l], out=on[l])
    e2e_sync_us = (time.perf_counter() - t2) * 1e6 / (e2e_steps * L)
    if world > 1:
        t = torch.tensor([e2e_us], device="cuda")
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        e2e_us = float(t.item())

    if rank != 0:
        if world > 1:
            dist.barrier()
            dist.destroy_process_group()
        return

    import json as _json

    peaks = {}
    try:
        peaks = _json.load(open(os.path.join(ROOT, "MEASURED_PEAKS.json")))
    except Exception:
        pass
    peak = float(peaks.get("hbm_gbs", 6650.0))
    achieved = alg_bytes / (kern_us * 1e-6) / 1e9
    kname = (f"louver_layer_v9<{geo['dp']},{G}>" if cfg["dtype"] == "bf16"
             else f"louver_layer_f32<{geo['dp']},{G}>" if geo["dp"] >= 128
             else f"louver_query_kernel<f32,{geo['dp']},{G},kQuery>")
    traffic = None  # dram__bytes_read.sum + dram__bytes_write.sum per launch, from a committed ncu capture
    try:
        tr = _json.load(open(os.path.join(ROOT, "profiles", "traffic.json")))
        if tr.get("kernel") == kname and tr.get("config") == args.config:
            traffic = float(tr["dram_bytes_per_launch"])
    except Exception:
        pass
    cpu = None
    if not args.no_cpu_baseline and world == 1:
        K0, V0, Q0, tau0 = first
        try:
            cpu = cpu_baseline_sample(K0, V0, Q0, tau0, G)
        except Exception as ex:  # pragma: no cover
            cpu = {"value": None, "error": str(ex)}
    line = {
        "metric": METRIC,
        "value": us_layer,
        "unit": UNIT,
        "n_gpus": world,
        "steps": args.steps,
        "warmup": args.warmup,
        "ms_per_step": ms_step,
        "higher_is_better": False,
        "scaling": "weak",
        "vs_baseline": None,
        "dtype": cfg["dtype"],
        "data": "synthetic (reference decode-trace key law io.cpp:145-169, sign-aligned queries io.cpp:186-202)",
        "config": {
            "workload": cfg["workload"] + (f"; sequence-sharded {n} keys/GPU, context {n * world}" if world > 1 else ""),
            "batch": B, "H_q": H_q, "H_kv": H, "d": d, "n_per_gpu": n, "context": n * world, "layers": L,
            "cell_keys": CELL, "selectivity": SELECTIVITY, "tau": "fixed, ceil(0.05 n)-th largest score",
            "queries": (f"{R} consecutive decode queries per layer (rows of the stream's "
                        f"gen_synthetic_queries), step i uses query i % {R}, each with its own tau"),
            "l2": f"inputs larger than L2: {L} layers x {slots * n * d * e * 2 / 2**20:.0f} MiB KV; "
                  f"{alg_bytes * L / 1e6:.0f} MB touched per step",
            "parallelism": f"seq-shard{world}" if world > 1 else "single GPU",
            "graph": graph is not None, "geometry": geo,
        },
        "gpu_launches": args.steps * L * (2 if world > 1 else 1),
        "roofline": {
            "bound": "hbm", "achieved": achieved, "peak": peak, "unit": "GB/s", "frac": achieved / peak,
            "traffic": traffic, "kernel": kname,
            "kernel_us": kern_us, "single_launch_us": single_us,
            "kernel_us_how": ("graph-timed step / layers (1 kernel per layer)" if kern_us == us_layer
                              else "per-launch CUDA events"),
            "algorithmic_bytes": alg_bytes,
            "bytes": {"summaries": float(np.mean(b_sum)), "keys": float(np.mean(b_key)),
                      "values": float(np.mean(b_val)), "partials": float(b_part), "q_o_tau": float(b_qo)},
            "frac_of_8000": achieved / 8000.0, "peak_source": "MEASURED_PEAKS.json hbm_gbs",
        },
        "keys": {"n": n, "scanned_per_q_head": keys_scanned, "selected_per_q_head": keys_selected,
                 "attended_per_q_head": keys_attended, "loaded_union_per_layer": float(np.mean(tot[:, 2])),
                 "f_scan": keys_scanned / n},
        "threshold_oracle": tau_oracle,
        "dense": {"us_per_layer": dense_us, "bytes": dense_bytes,
                  "achieved_gbs": dense_bytes / (dense_us * 1e-6) / 1e9,
                  "speedup_vs_dense": dense_us / kern_us,
                  "how": "CUDA graph of L layer launches, median of 50 replays / L (same as the metric)",
                  "torch_sdpa_us_per_layer": sdpa_us,
                  "speedup_vs_torch_sdpa": (sdpa_us / kern_us) if sdpa_us else None,
                  "best_dense_us_per_layer": min(x for x in (dense_us, sdpa_us) if x),
                  "speedup_vs_best_dense": min(x for x in (dense_us, sdpa_us) if x) / kern_us},
        "e2e": {"value": e2e_us, "unit": UNIT, "h2d_bytes_per_step": L * rows * (d + 1) * 4,
                "d2h_bytes_per_step": L * rows * d * 4,
                "how": ("host wall clock per decode step / L through the C ABI with HOST buffers: "
                        "lv_query_layers(pinned q, tau, out) called through a prepared LayersStep (one C call per "
                        "step): a cached CUDA graph in which one kernel stages every layer's q and tau from the "
                        "mapped pinned host buffers, the L fused layer queries write their outputs straight into "
                        "the pinned host buffer, then one stream sync"
                        if world == 1 else
                        "host wall clock per sharded decode step / L: pinned q, tau -> device, L x (lv_query partial, "
                        "NCCL all-gather, lv_lse_merge), outputs -> pinned host, stream sync"),
                "per_layer_sync_us": e2e_sync_us,
                "per_layer_sync_how": "one synchronous lv_query(LV_HOST) per layer: pinned q/tau H2D, kernel, pinned out D2H, sync"},
        "clocks": clocks.summary(),
    }
    if cpu is not None:
        line["cpu_baseline"] = cpu
    print(json.dumps(line), flush=True)
    if world > 1:
        dist.barrier()
        dist.destroy_process_group()


if __name__ == "__main__":
    main()
