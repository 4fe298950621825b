"""Per-CTA phase timing of the bf16 query kernel (lv_debug_trace) on one C2 layer.

Phases: 0 start, 1 summary tile landed, 2 probe done, 3 exact rounds done,
4 softmax prep done, 5 value rounds done, 6 partial written, 7 merged (last CTAs).
"""
import os
import sys

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import torch  # noqa: E402

import bench  # noqa: E402
from paper_2605_06763_b200 import BuildConfig, LouverLayer  # noqa: E402


def main():
    cfg = dict(bench.CONFIGS[os.environ.get("CONFIG", "c2")])
    K, V, Q = bench.gen_layer(cfg, 0, 0, os.cpu_count())
    G = cfg["G"]
    tau = bench.taus_device(torch, K, Q, G, bench.SELECTIVITY)
    layer = LouverLayer(cfg["d"], cfg["H_kv"], G, cfg["batch"], cfg["n"],
                        BuildConfig(S=1, r=bench.CELL, grouping="contiguous", enclosing="aabb"))
    layer.build(K, V)
    q, t = torch.from_numpy(Q).cuda(), torch.from_numpy(tau).cuda()
    out = torch.zeros((cfg["batch"], cfg["H_kv"] * G, cfg["d"]), device="cuda")
    geo = layer.geometry()
    nct = cfg["batch"] * cfg["H_kv"] * geo["splits"]
    buf = torch.zeros((nct, 8), dtype=torch.int64, device="cuda")
    for _ in range(3):
        layer.query_device(q, t, out)
    layer._ctx.lib.lv_debug_trace(layer._ctx.h, buf.data_ptr())
    buf.zero_()
    layer.query_device(q, t, out)
    torch.cuda.synchronize()
    layer._ctx.lib.lv_debug_trace(layer._ctx.h, None)
    tr = buf.cpu().numpy().astype(np.float64)
    t0 = tr[:, 0].min()
    rel = (tr - t0) / 1e3  # us
    names = ["tile", "probe", "exact", "prep", "values", "partial", "merge"]
    print(f"CTAs {nct}; kernel span {rel[:, 6].max():.2f} us (last partial), start spread {rel[:, 0].max():.2f} us")
    for i in range(1, 7):
        d = tr[:, i] - tr[:, i - 1]
        ok = tr[:, i] > 0
        d = d[ok & (tr[:, i - 1] > 0)] / 1e3
        if d.size:
            print(f"  {names[i - 1]:8s} mean {d.mean():7.3f} us  p50 {np.median(d):7.3f}  p90 {np.percentile(d, 90):7.3f}  max {d.max():7.3f}")
    life = (tr[:, 6] - tr[:, 0]) / 1e3
    print(f"  CTA life mean {life.mean():.2f} us p50 {np.median(life):.2f} max {life.max():.2f}")
    # concurrency over time
    starts = np.sort(rel[:, 0])
    print("  start-time quantiles (us):", np.percentile(starts, [0, 25, 50, 75, 100]).round(2))


if __name__ == "__main__":
    main()
