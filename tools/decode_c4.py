"""an 8192-token prompt, then 32768 decode steps of query-then-insert
(bench.cpp:91-118) with B = 128 (256 flushes), d = 128, fp32, the reference key law
(io.cpp:145-169) and sign-aligned queries (io.cpp:186-202), τ from the device threshold
oracle (budget:0.05 over a 256-id reservoir, the paper default). Every step is verified
against the brute-force range on the device. Prints one JSON line.

    python tools/decode_c4.py [--steps 32768] [--prefill 8192]
"""
import argparse
import json
import os
import sys
import time

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

from paper_2605_06763_b200 import BuildConfig, OracleConfig, OracleVariant, synth  # noqa: E402
from paper_2605_06763_b200.decode_sim import DecodeSimConfig, ThresholdSource, run_decode_sim  # noqa: E402


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--steps", type=int, default=32768)
    ap.add_argument("--prefill", type=int, default=8192)
    ap.add_argument("--seed", type=int, default=4)
    a = ap.parse_args()
    rows, d = a.prefill + a.steps, 128
    keys = synth.keys(rows, d, a.seed)
    values = synth.keys(rows, d, a.seed + 1)
    queries = synth.queries(rows, d, a.seed)
    cfg = DecodeSimConfig(build=BuildConfig(1, 16, "contiguous", "aabb", 0), buffer_capacity=128,
                          threshold=ThresholdSource(oracle=OracleConfig(OracleVariant.Budget, 0, 0.05)),
                          reservoir_capacity=256, seed=a.seed, verify=True)
    t0 = time.perf_counter()
    rep = run_decode_sim(keys, values, queries, cfg, prefill=a.prefill)
    wall = time.perf_counter() - t0
    out = {"config": "C4", "prefill": a.prefill, "decode_steps": rep.steps, "d": d, "dtype": "f32", "B": 128,
           "oracle": "budget:0.05", "reservoir": 256, "flushes": rep.flushes, "violations": rep.violations,
           "median_query_us": rep.median_query_us, "mean_query_us": rep.mean_query_us,
           "mean_keys_scanned": rep.mean_keys_scanned, "mean_f_scan": rep.mean_f_scan,
           "mean_selected": rep.mean_selected, "mean_retrieved": rep.mean_retrieved, "mean_tau": rep.mean_tau,
           "host_wall_s": wall, "host_wall_us_per_step": wall / max(1, rep.steps) * 1e6,
           "how": "run_decode_sim on the device (paper_2605_06763_b200/decode_sim.py): per step estimate_tau, "
                  "lv_query (timed with CUDA events), brute-force verification + bitmap compare, lv_push_key; "
                  "host wall includes verification and the Python loop"}
    print(json.dumps(out))


if __name__ == "__main__":
    main()
