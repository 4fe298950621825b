"""Decode-loop driver: ``run_decode_sim`` of proj/include/louver/bench.hpp:16-58 and
proj/src/bench.cpp:12-136, device-resident.

Per step t (bench.cpp:71-120): τ from the fixed source, or from the threshold
oracle once the reservoir holds enough samples (else -inf, the warm-up); the
cache query; optional verification against the brute-force range; optional
recall@k against the exact top-k; then push_key of row t and the reservoir
update. Here every per-step operation is enqueued on one CUDA stream with no
host synchronisation: τ is estimated on the device from a device copy of the
reservoir's ids (``lv_estimate_tau``), the query writes its counts into a
per-step slot of a device array, verification compares the query's selected
bitmap with ``lv_brute_force_range``'s on the device (``lv_bits_diff`` adds to a
device violation counter), and the key/value of the step are appended on the
device (flush-at-B inside ``lv_push_key``). The host only draws the reservoir's
random numbers (the reference's mt19937_64, in the C library). Statistics are
read back once at the end.

Differences a caller sees: ``median_query_us`` is the median DEVICE time of the
query launch (CUDA events around it, the launch queued behind a short device
sleep so that host launch latency is not counted), not host wall time; recall@k (requested
through ``recall_ks``) synchronises each step, since the exact top-k of every
step is ranked on the host with the normative score order (a measurement, as in
the reference, not part of the decode path).
"""
from __future__ import annotations

import dataclasses
import math
import statistics
from typing import Dict, List, Optional

import numpy as np

from . import _capi
from ._capi import check
from .louver import BuildConfig, FilterAlgo, LouverLayer
from .threshold import OracleConfig, OracleVariant, Reservoir, estimate_tau_layer


_SLEEP_CYCLES = 100_000  # ~50 us at the B200's boost clock


def speedup_estimate(g: float, r: float, f_scan: float) -> float:
    """bench.cpp:12-19: 1 / (g / r + f_scan)."""
    if r < 1.0:
        raise ValueError("speedup_estimate: r >= 1 required")
    if g < 0.0 or f_scan < 0.0 or f_scan > 1.0:
        raise ValueError("speedup_estimate: need g >= 0 and f_scan in [0, 1]")
    denom = g / r + f_scan
    if denom == 0.0:
        raise ArithmeticError("speedup_estimate: g and f_scan both zero")  # std::domain_error
    return 1.0 / denom


@dataclasses.dataclass
class ThresholdSource:
    """bench.hpp:16-19: exactly one of these is set."""

    fixed_tau: Optional[float] = None
    oracle: Optional[OracleConfig] = None


@dataclasses.dataclass
class DecodeSimConfig:
    """bench.hpp:21-31."""

    build: BuildConfig = dataclasses.field(default_factory=BuildConfig)
    buffer_capacity: int = 128
    algo: FilterAlgo = FilterAlgo.Ta
    threshold: ThresholdSource = dataclasses.field(default_factory=ThresholdSource)
    reservoir_capacity: int = 256
    seed: int = 0
    verify: bool = False
    strict_threshold: bool = False
    recall_ks: List[int] = dataclasses.field(default_factory=list)


@dataclasses.dataclass
class MetricsReport:
    """bench.hpp:33-48."""

    steps: int = 0
    flushes: int = 0
    violations: int = 0
    mean_f_scan: float = 0.0
    mean_keys_scanned: float = 0.0
    mean_groups_tested: float = 0.0
    mean_gate_cost_equiv: float = 0.0
    mean_selected: float = 0.0
    mean_retrieved: float = 0.0
    mean_tau: float = 0.0
    mean_speedup_estimate: float = 0.0
    median_query_us: float = 0.0
    mean_query_us: float = 0.0  # extension: mean device time of the query launch
    recall: Dict[int, float] = dataclasses.field(default_factory=dict)


def _normative_scores(keys: np.ndarray, q: np.ndarray) -> np.ndarray:
    """core.hpp:17-21 for every row at once: float32 multiply, then add, in order."""
    s = np.zeros(keys.shape[0], np.float32)
    for c in range(keys.shape[1]):
        s = (s + keys[:, c] * q[c]).astype(np.float32)
    return s


def _exact_topk(scores: np.ndarray, k: int) -> np.ndarray:
    """bench.cpp:34-49: the k best by (score desc, id asc)."""
    order = np.lexsort((np.arange(scores.size), -scores.astype(np.float64)))
    return order[: min(k, scores.size)]


def run_decode_sim(keys, values, queries, cfg: DecodeSimConfig, prefill: int = 0) -> MetricsReport:
    """bench.hpp:50-58 / bench.cpp:54-136 on the device. keys, values, queries: [steps][d]
    float32; row t drives step t.

    ``prefill`` (an extension, 0 = the reference's loop): rows [0, prefill) form the
    initial store, indexed at once as by ``LouverCache(KeyStore, cfg, B)``
    (cache.hpp:31-36) and fed to the reservoir in order; steps prefill .. rows-1 then
    run the decode loop (an 8K prompt, then 32K query-then-insert steps)."""
    import torch  # plumbing: device buffers, the stream, events

    keys = np.ascontiguousarray(keys, np.float32)
    values = np.ascontiguousarray(values, np.float32)
    queries = np.ascontiguousarray(queries, np.float32)
    if keys.shape[0] != values.shape[0] or keys.shape[0] != queries.shape[0]:
        raise ValueError("run_decode_sim: keys/values/queries row mismatch")
    if cfg.threshold.fixed_tau is None and cfg.threshold.oracle is None:
        raise ValueError("run_decode_sim: no threshold source")
    rows, d = keys.shape
    if not 0 <= prefill <= rows:
        raise ValueError("run_decode_sim: prefill outside [0, rows]")
    oracle = cfg.threshold.oracle if cfg.threshold.fixed_tau is None else None
    if oracle is not None:
        oracle.validate()

    steps = rows
    layer = LouverLayer(d, 1, 1, 1, max(rows, 16), cfg.build, buffer_capacity=cfg.buffer_capacity, dtype="f32")
    reservoir = Reservoir(cfg.reservoir_capacity, cfg.seed)
    dev = torch.device("cuda")
    stream = torch.cuda.current_stream().cuda_stream
    k_d = torch.from_numpy(keys).to(dev)
    v_d = torch.from_numpy(values).to(dev)
    q_d = torch.from_numpy(queries).to(dev)
    fill = cfg.threshold.fixed_tau if oracle is None else -math.inf  # warm-up: retrieve all
    tau_d = torch.full((steps, 1), float(fill), dtype=torch.float32, device=dev)
    out_d = torch.zeros((steps, d), dtype=torch.float32, device=dev)
    counts_d = torch.zeros((steps, 4), dtype=torch.int32, device=dev)
    totals_d = torch.zeros((steps, 4), dtype=torch.int64, device=dev)
    ids_d = torch.zeros((1, cfg.reservoir_capacity), dtype=torch.int32, device=dev)
    words = layer.bitmap_words
    need_bits = cfg.verify or bool(cfg.recall_ks) or cfg.strict_threshold
    bits = torch.zeros((1, words), dtype=torch.int32, device=dev) if need_bits else None
    viol_d = torch.zeros((1,), dtype=torch.int32, device=dev)
    ev = [(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)) for _ in range(steps)]
    need = (oracle.m if oracle is not None and oracle.variant == OracleVariant.SampleTopK else 1)
    recall_sum: Dict[int, float] = {}
    recall_steps = 0
    retrieved_h = np.zeros(steps, np.int64)
    lib = _capi.lib()

    if prefill:
        layer.build(keys[:prefill].reshape(1, 1, prefill, d), values[:prefill].reshape(1, 1, prefill, d))
        for j in range(prefill):
            reservoir.update(j)
        ids0 = reservoir.ids().astype(np.int32)
        ids_d[0, : ids0.size] = torch.from_numpy(ids0).to(dev)
    for t in range(prefill, steps):
        n = t  # keys stored before this step's query
        size = reservoir.size()
        if oracle is not None and size >= 2 and size >= need:
            estimate_tau_layer(layer, ids_d, size, q_d[t].view(1, 1, d), oracle, tau_d[t].view(1, 1))
        if bits is not None:
            bits.zero_()
        # the timed query is queued behind a short device sleep, so the start event fires
        # once the launch is already in the stream: the interval is the query's device
        # time, not the host's launch latency (the loop is host-bound otherwise)
        torch.cuda._sleep(_SLEEP_CYCLES)
        ev[t][0].record()
        layer.query_device(q_d[t].view(1, 1, d), tau_d[t].view(1, 1), out_d[t].view(1, 1, d),
                           strict=cfg.strict_threshold, counts=counts_d[t], sel_bits=bits, totals=totals_d[t])
        ev[t][1].record()
        if cfg.verify and n > 0:
            ref_bits = layer.brute_force_bits(q_d[t].view(1, 1, d), tau_d[t].view(1, 1), n)
            check(lib.lv_bits_diff(bits.data_ptr(), ref_bits.data_ptr(), words, 1, viol_d.data_ptr(), stream),
                  "lv_bits_diff")
        if cfg.recall_ks or cfg.strict_threshold:
            sel = layer.ids_from_bits(bits, n)[0] if n else np.zeros((0,), np.uint32)
            indexed = layer.indexed_count
            retrieved = np.concatenate([sel[sel < indexed], np.arange(indexed, n, dtype=np.uint32)])
            retrieved_h[t] = retrieved.size
            if cfg.recall_ks and n > 0:
                scores = _normative_scores(keys[:n], queries[t])
                for k in cfg.recall_ks:
                    top = _exact_topk(scores, k)
                    if top.size:
                        recall_sum[k] = recall_sum.get(k, 0.0) + np.isin(top, retrieved).sum() / top.size
                recall_steps += 1
        layer.push_key(k_d[t].view(1, 1, d), v_d[t].view(1, 1, d))
        slot = reservoir.update(t)
        if slot >= 0:
            ids_d[0, slot] = t

    torch.cuda.synchronize()
    layer.sync_counters()
    counts = counts_d.cpu().numpy()
    totals = totals_d.cpu().numpy()
    taus = tau_d.cpu().numpy()[:, 0]
    rep = MetricsReport(steps=steps - prefill, flushes=layer.flush_count, violations=int(viol_d.item()))
    # statistics of the device index: its groups are cells of cell_keys contiguous keys with
    # one AABB each (gate cost 2 per cell), so gate_cost_equiv and the speed-up estimate
    # use that geometry (bench.cpp:13-20 with g = 2, r = cell_keys), not cfg.build's r
    g = 2.0
    r_dev = max(1, int(layer.geometry().get("cell_keys", cfg.build.r)))
    inv = 1.0 / rep.steps if rep.steps else 0.0
    sum_speedup = 0.0
    for t in range(prefill, steps):
        n = t
        scanned = float(counts[t, 2])
        f_scan = scanned / n if n > 0 else 1.0  # cache.cpp:58-65
        retrieved = float(retrieved_h[t]) if (cfg.recall_ks or cfg.strict_threshold) else float(counts[t, 1])
        if n == 0:
            retrieved = 0.0
        groups = float(totals[t, 0])
        rep.mean_f_scan += f_scan
        rep.mean_keys_scanned += scanned
        rep.mean_groups_tested += groups
        rep.mean_gate_cost_equiv += g * groups / r_dev
        rep.mean_selected += float(counts[t, 0])
        rep.mean_retrieved += retrieved
        rep.mean_tau += float(taus[t]) if math.isfinite(float(taus[t])) else 0.0
        sum_speedup += speedup_estimate(g, r_dev, min(max(f_scan, 0.0), 1.0))
        if cfg.verify and n == 0 and counts[t, 0] != 0:
            rep.violations += 1
    for f in ("mean_f_scan", "mean_keys_scanned", "mean_groups_tested", "mean_gate_cost_equiv", "mean_selected",
              "mean_retrieved", "mean_tau"):
        setattr(rep, f, getattr(rep, f) * inv)
    rep.mean_speedup_estimate = sum_speedup * inv
    if rep.steps:
        q_us = [a.elapsed_time(b) * 1e3 for a, b in ev[prefill:]]
        rep.median_query_us = statistics.median(q_us)
        rep.mean_query_us = statistics.mean(q_us)
    for k, total in recall_sum.items():
        rep.recall[k] = total / recall_steps if recall_steps else 0.0
    return rep


@dataclasses.dataclass
class GraphDecodeReport:
    """Statistics of ``run_decode_graph`` (per q head means over the decode steps)."""

    steps: int = 0
    flushes: int = 0
    n_final: int = 0
    violations: int = -1              # -1: not verified
    us_per_step: float = 0.0          # device time of the replayed step graphs / steps
    mean_selected: float = 0.0        # per q head per step
    mean_attended: float = 0.0
    mean_keys_scanned: float = 0.0
    mean_f_scan: float = 0.0          # keys scanned / keys stored before the step
    mean_tau: float = 0.0
    selected: Optional[np.ndarray] = None  # [steps][rows] per step and q head
    taus: Optional[np.ndarray] = None      # [steps][rows]


def run_decode_graph(keys, values, queries, H_kv: int, G: int, cfg: DecodeSimConfig, prefill: int,
                     batch: int = 1, dtype: str = "bf16", steps_per_graph: int = 16,
                     verify: bool = False) -> GraphDecodeReport:
    """The decode loop of bench.cpp:71-120 for a whole attention layer (``batch`` x ``H_kv``
    kv slots, ``G`` q heads each), captured as CUDA graphs and replayed with no host work
    per step. keys, values: [rows][batch * H_kv][d]; queries: [rows][batch * H_kv * G][d]
    (float32, row t drives step t). Rows [0, prefill) are the prompt, indexed at once;
    steps prefill .. rows - 1 each run, on the device:

      load q_t, k_t, v_t (a device step counter selects the slice)
      tau  = estimate_tau over the reservoir (oracle source) or the fixed tau
      lv_query (selected / attended / scanned counts logged per step)
      [verify: brute_force_range over every stored key, bitmap compare]
      lv_push_key(k_t, v_t)  (flush at B inside the insert kernel)
      the reservoir's write for row t (its draws are the reference's mt19937_64,
      made on the host in advance: they depend only on capacity, seed and t)

    With the oracle source the reservoir must be full after the prompt (prefill >=
    capacity), so every step samples the same number of rows, as a captured launch
    requires."""
    import torch

    keys = np.ascontiguousarray(keys, np.float32)
    values = np.ascontiguousarray(values, np.float32)
    queries = np.ascontiguousarray(queries, np.float32)
    rows, slots, d = keys.shape
    rq = queries.shape[1]
    if slots != batch * H_kv or rq != slots * G or values.shape != keys.shape or queries.shape[0] != rows:
        raise ValueError("run_decode_graph: shapes must be keys/values [rows][batch*H_kv][d], queries [rows][rows_q][d]")
    if not 0 < prefill < rows:
        raise ValueError("run_decode_graph: 0 < prefill < rows required")
    oracle = cfg.threshold.oracle if cfg.threshold.fixed_tau is None else None
    if oracle is None and cfg.threshold.fixed_tau is None:
        raise ValueError("run_decode_graph: no threshold source")
    if oracle is not None:
        oracle.validate()
        if prefill < cfg.reservoir_capacity:
            raise ValueError("run_decode_graph: the reservoir must be full after the prompt")
    steps = rows - prefill
    spg = max(1, min(steps_per_graph, steps))
    while steps % spg:
        spg -= 1
    dev = torch.device("cuda")
    lib = _capi.lib()
    layer = LouverLayer(d, H_kv, G, batch, rows, cfg.build, buffer_capacity=cfg.buffer_capacity, dtype=dtype)
    layer.build(np.ascontiguousarray(keys[:prefill].reshape(prefill, batch, H_kv, d).transpose(1, 2, 0, 3)),
                np.ascontiguousarray(values[:prefill].reshape(prefill, batch, H_kv, d).transpose(1, 2, 0, 3)))
    # the reservoir's admissions for every row, drawn now (threshold.cpp:40-55)
    res = Reservoir(cfg.reservoir_capacity, cfg.seed)
    slot_of = np.full((rows,), -1, np.int32)
    for t in range(rows):
        slot_of[t] = res.update(t)
    res0 = Reservoir(cfg.reservoir_capacity, cfg.seed)
    for t in range(prefill):
        res0.update(t)
    cap = cfg.reservoir_capacity
    ids_d = torch.from_numpy(np.tile(res0.ids().astype(np.int32)[None], (slots, 1))).to(dev)
    slot_d = torch.from_numpy(slot_of).to(dev)
    k_d, v_d, q_d = (torch.from_numpy(a).to(dev) for a in (keys, values, queries))
    q_buf = torch.zeros((batch, H_kv * G, d), dtype=torch.float32, device=dev)
    k_buf = torch.zeros((batch, H_kv, d), dtype=torch.float32, device=dev)
    v_buf = torch.zeros_like(k_buf)
    fill = float(cfg.threshold.fixed_tau) if oracle is None else 0.0
    tau_buf = torch.full((batch, H_kv * G), fill, dtype=torch.float32, device=dev)
    out_buf = torch.zeros((batch, H_kv * G, d), dtype=torch.float32, device=dev)
    counts = torch.zeros((batch, H_kv * G, 4), dtype=torch.int32, device=dev)
    cnt_log = torch.zeros((rows, rq, 4), dtype=torch.int32, device=dev)
    tau_log = torch.zeros((rows, rq), dtype=torch.float32, device=dev)
    step_d = torch.tensor([prefill], dtype=torch.int64, device=dev)
    words = layer.bitmap_words
    bits = torch.zeros((rq, words), dtype=torch.int32, device=dev) if verify else None
    ref_bits = torch.zeros_like(bits) if verify else None
    viol = torch.zeros((1,), dtype=torch.int32, device=dev)
    ctx = layer._ctx

    cp = _capi.lv_step_copy
    loads = (cp * 3)(cp(q_d.data_ptr(), q_buf.data_ptr(), rq * d * 4, rq * d * 4, 0),
                     cp(k_d.data_ptr(), k_buf.data_ptr(), slots * d * 4, slots * d * 4, 0),
                     cp(v_d.data_ptr(), v_buf.data_ptr(), slots * d * 4, slots * d * 4, 0))
    stores = (cp * 2)(cp(counts.data_ptr(), cnt_log.data_ptr(), rq * 16, rq * 16, 1),
                      cp(tau_buf.data_ptr(), tau_log.data_ptr(), rq * 4, rq * 4, 1))

    def one_step(st):
        sp = step_d.data_ptr()
        check(lib.lv_step_copies(sp, loads, 3, st), "lv_step_copies")
        if oracle is not None:
            estimate_tau_layer(layer, ids_d, cap, q_buf, oracle, tau_buf, stream=st)
        if verify:  # (lv_query zeroes counts itself)
            bits.zero_()
        layer.query_device(q_buf, tau_buf, out_buf, strict=cfg.strict_threshold, counts=counts, sel_bits=bits,
                           stream=st)
        if verify:
            check(lib.lv_brute_force_range(ctx.h, q_buf.data_ptr(), tau_buf.data_ptr(), -1, _capi.LV_DEVICE,
                                           ref_bits.data_ptr(), st), "lv_brute_force_range")
            check(lib.lv_bits_diff(bits.data_ptr(), ref_bits.data_ptr(), words, rq, viol.data_ptr(), st),
                  "lv_bits_diff")
        layer.push_key(k_buf, v_buf, stream=st)
        # the step's log, the reservoir's write for row t and the counter advance: one launch
        check(lib.lv_step_epilogue(sp, stores, 2, slot_d.data_ptr(), 0, ids_d.data_ptr(), slots, cap, st),
              "lv_step_epilogue")

    stream = torch.cuda.Stream()
    graph = torch.cuda.CUDAGraph()
    torch.cuda.synchronize()
    with torch.cuda.graph(graph, stream=stream):
        st = torch.cuda.current_stream().cuda_stream
        for _ in range(spg):
            one_step(st)
    layer.sync_counters()  # capture advanced the host mirrors; the device counters did not move
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    torch.cuda.synchronize()
    a.record()
    for _ in range(steps // spg):
        graph.replay()
    b.record()
    torch.cuda.synchronize()
    layer.sync_counters()
    rep = GraphDecodeReport(steps=steps, flushes=layer.flush_count, n_final=layer.n,
                            us_per_step=a.elapsed_time(b) * 1e3 / steps)
    if verify:
        rep.violations = int(viol.item())
    cl = cnt_log[prefill:].cpu().numpy().astype(np.float64)
    tl = tau_log[prefill:].cpu().numpy().astype(np.float64)
    n_before = np.arange(prefill, rows, dtype=np.float64)[:, None]
    rep.mean_selected = float(cl[..., 0].mean())
    rep.mean_attended = float(cl[..., 1].mean())
    rep.mean_keys_scanned = float(cl[..., 2].mean())
    rep.mean_f_scan = float((cl[..., 2] / n_before).mean())
    rep.mean_tau = float(tl.mean())
    rep.selected = cl[..., 0].astype(np.int64)
    rep.taus = tl.astype(np.float32)
    del graph
    return rep


__all__ = ["ThresholdSource", "DecodeSimConfig", "MetricsReport", "run_decode_sim", "speedup_estimate",
           "GraphDecodeReport", "run_decode_graph"]
