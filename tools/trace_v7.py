"""Per-CTA phase timing of the bf16 cell-stream kernel (louver_cells_v7) on one layer.

Phases: 0 start, 1 setup done, 2 griddepcontrol.wait returned (probe done),
3 survivor prefix done, 4 first task begins, 5 last warp finished its tasks,
6 CTA partial ready, 7 end (merge done).
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
    slots = cfg["batch"] * cfg["H_kv"]
    nb = -(-2 * 148 // slots)
    buf = torch.zeros((slots * nb, 32), dtype=torch.int64, device="cuda")
    for _ in range(int(os.environ.get("WARM", "300"))):  # keep the clocks up
        layer.query_device(q, t, out)
    torch.cuda.synchronize()
    st, en = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    layer._ctx.lib.lv_debug_trace(layer._ctx.h, buf.data_ptr())
    buf.zero_()
    if os.environ.get("FLUSH", "1") == "1":  # cold L2: the bench's regime (inputs >> L2)
        # read (not write) 512 MB: the L2 ends up holding clean lines, as after the
        # previous layer's query, so no dirty write-backs compete with the traced launch
        junk = torch.ones(128 << 20, dtype=torch.float32, device="cuda")
        torch.cuda.synchronize()
        junk.sum()
    torch.cuda.synchronize()
    st.record()
    layer.query_device(q, t, out)
    en.record()
    torch.cuda.synchronize()
    layer._ctx.lib.lv_debug_trace(layer._ctx.h, None)
    print(f"event time of traced query: {st.elapsed_time(en) * 1e3:.1f} us")
    tr = buf.cpu().numpy().astype(np.float64)
    tr = tr[tr[:, 0] > 0]  # CTAs that ran
    t0 = tr[:, 0].min()
    ns = tr[:, 15]
    print(f"  survivors per CTA: min {ns.min():.0f} p10 {np.percentile(ns, 10):.0f} p50 {np.median(ns):.0f} "
          f"p90 {np.percentile(ns, 90):.0f} max {ns.max():.0f}")
    life = (tr[:, 5] - tr[:, 4]) / 1e3
    print("  corr(survivors, task time) = %.2f; task-time per survivor p50 %.3f us" %
          (np.corrcoef(ns, life)[0, 1], np.median(life / np.maximum(ns, 1))))
    fin = tr[tr[:, 7] > 0]
    for row in fin:
        r = (row - t0) / 1e3
        print(f"  final CTA: partial {r[6]:.2f} won {r[8]:.2f} headers {r[11]:.2f} "
              f"chunk {r[13]:.2f} acc {r[14]:.2f} end {r[7]:.2f}")
    for i, nm in ((9, "q loaded"), (12, "colmax"), (10, "S ready"), (1, "frags done")):
        v = (tr[:, i] - t0) / 1e3
        print(f"  setup {nm:10s} quantiles " + " ".join(f"{x:6.2f}" for x in np.percentile(v, [0, 50, 100])))
    tr = tr[:, :8]
    rel = (tr - t0) / 1e3
    names = ["setup", "wait", "prefix", "cells", "tasks", "partial", "merge"]
    print(f"CTAs {len(tr)}; start spread {rel[:, 0].max():.2f} us; last end {rel[:, 7].max():.2f} us")
    for i in range(8):
        v = rel[:, i][tr[:, i] > 0]
        print(f"  t{i} abs quantiles " + " ".join(f"{x:7.2f}" for x in np.percentile(v, [0, 10, 50, 90, 100])))
    for i in range(1, 8):
        ok = (tr[:, i] > 0) & (tr[:, i - 1] > 0)
        d = (tr[ok, i] - tr[ok, i - 1]) / 1e3
        if d.size:
            print(f"  {names[i - 1]:8s} mean {d.mean():7.3f}  p50 {np.median(d):7.3f}  p90 {np.percentile(d, 90):7.3f}  max {d.max():7.3f}")


if __name__ == "__main__":
    main()
