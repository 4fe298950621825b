"""SURVEY §8(d) C4 at the C2 head shape: an 8192-token prompt, then 32768 decode steps of
query-then-insert (bench.cpp:91-118) for a Llama-3-8B-shaped layer (32 q / 8 kv heads,
d = 128, bf16 KV), B = 128 (256 flushes), τ per step and q head from the device threshold
oracle (budget:0.05 over a 256-id reservoir), the reference key law (io.cpp:145-169) and
sign-aligned queries (io.cpp:186-202). The loop runs as CUDA graphs of 16 steps replayed
back to back (run_decode_graph): per step estimate_tau -> lv_query -> lv_push_key, inputs
selected on the device by a step counter, no host work per step.

Pass 1 (timed): device time of the whole loop / steps. Pass 2: the same loop with
on-device verification (brute-force range over every stored key, bitmap compare) —
violations must be 0. Also: the insert alone (a graph of 256 lv_push_key on the same
shape), and the per-step statistics. Prints one JSON line.

    python tools/decode_c4_graph.py [--steps 32768] [--prefill 8192]
"""
import argparse
import json
import os
import sys
import time

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import torch  # noqa: E402

from paper_2605_06763_b200 import BuildConfig, LouverLayer, OracleConfig, OracleVariant, synth  # noqa: E402
from paper_2605_06763_b200.decode_sim import DecodeSimConfig, ThresholdSource, run_decode_graph  # noqa: E402


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--steps", type=int, default=32768)
    ap.add_argument("--prefill", type=int, default=8192)
    ap.add_argument("--seed", type=int, default=4)
    ap.add_argument("--no-verify", action="store_true")
    a = ap.parse_args()
    H_kv, G, d, B = 8, 4, 128, 128
    rows = a.prefill + a.steps
    t0 = time.perf_counter()
    seeds = np.array([a.seed + 1000 * h for h in range(H_kv)], np.uint64)
    K = synth.keys_multi(rows, d, seeds, os.cpu_count()).transpose(1, 0, 2)                 # [rows][H][d]
    V = synth.keys_multi(rows, d, seeds + np.uint64(1), os.cpu_count()).transpose(1, 0, 2)
    Q = np.stack([synth.queries(rows * G, d, int(s)).reshape(rows, G, d) for s in seeds], axis=1)
    Q = Q.reshape(rows, H_kv * G, d)
    K, V, Q = (np.ascontiguousarray(x, np.float32) for x in (K, V, Q))
    gen_s = time.perf_counter() - t0
    cfg = DecodeSimConfig(build=BuildConfig(1, 16, "contiguous", "aabb", 0), buffer_capacity=B,
                          threshold=ThresholdSource(oracle=OracleConfig(OracleVariant.Budget, 0, 0.05)),
                          reservoir_capacity=256, seed=a.seed)
    rep = run_decode_graph(K, V, Q, H_kv, G, cfg, a.prefill, dtype="bf16", steps_per_graph=16)
    ver = None if a.no_verify else run_decode_graph(K, V, Q, H_kv, G, cfg, a.prefill, dtype="bf16",
                                                    steps_per_graph=16, verify=True)

    # the insert alone: a graph of 256 lv_push_key calls (one key per kv slot each) on the shape
    layer = LouverLayer(d, H_kv, G, 1, a.prefill + 4096, cfg.build, buffer_capacity=B)
    layer.build(np.ascontiguousarray(K[:a.prefill].transpose(1, 0, 2))[None],
                np.ascontiguousarray(V[:a.prefill].transpose(1, 0, 2))[None])
    kk = torch.from_numpy(K[a.prefill:a.prefill + 256]).cuda()
    vv = torch.from_numpy(V[a.prefill:a.prefill + 256]).cuda()
    s = torch.cuda.Stream()
    g = torch.cuda.CUDAGraph()
    torch.cuda.synchronize()
    with torch.cuda.graph(g, stream=s):
        for i in range(256):
            layer.push_key(kk[i].view(1, H_kv, d), vv[i].view(1, H_kv, d))
    layer.sync_counters()
    ev0, ev1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    reps = 8  # 8 x 256 inserts fit the capacity (prefill + 4096)
    ev0.record()
    for _ in range(reps):
        g.replay()
    ev1.record()
    torch.cuda.synchronize()
    insert_us = ev0.elapsed_time(ev1) * 1e3 / (reps * 256)
    layer.sync_counters()

    out = {
        "config": "C4 at the C2 head shape", "prefill": a.prefill, "decode_steps": rep.steps, "H_q": H_kv * G,
        "H_kv": H_kv, "d": d, "dtype": "bf16", "B": B, "oracle": "budget:0.05", "reservoir": 256,
        "us_per_step": rep.us_per_step, "insert_us": insert_us,
        "insert_how": "graph of 256 lv_push_key (8 kv slots each), replayed 8x, device time / inserts",
        "flushes": rep.flushes, "n_final": rep.n_final,
        "violations": None if ver is None else ver.violations,
        "verified_steps": 0 if ver is None else ver.steps,
        "verified_us_per_step": None if ver is None else ver.us_per_step,
        "mean_selected_per_q_head": rep.mean_selected, "mean_attended_per_q_head": rep.mean_attended,
        "mean_keys_scanned_per_q_head": rep.mean_keys_scanned, "mean_f_scan": rep.mean_f_scan,
        "mean_tau": rep.mean_tau, "data_gen_s": gen_s,
        "how": "run_decode_graph (paper_2605_06763_b200/decode_sim.py): CUDA graphs of 16 steps, each step "
               "step-counter loads of q/k/v, estimate_tau (32 q heads), lv_query, counts logged, lv_push_key, "
               "reservoir write, counter advance; us_per_step = device time of all replays / steps",
    }
    print(json.dumps(out))


if __name__ == "__main__":
    main()
