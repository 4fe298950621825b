"""Per-CTA phase timing of the bf16 layer kernel (v10) on one C2 layer.

Stamps: 0 start, 1 setup done, 2 producer warp 0 done (probe), 3 consumer warp 0 starts
its first task, 4 consumer warp 0 done, 5 every warp done, 6 CTA partial written,
7 end (merge winners), 8 ticket won, 11 partial headers loaded, 15 tasks processed.
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
    buf = torch.zeros((slots * nb, 64), dtype=torch.int64, device="cuda")
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
    print(f"  tasks per CTA: min {ns.min():.0f} p10 {np.percentile(ns, 10):.0f} p50 {np.median(ns):.0f} "
          f"p90 {np.percentile(ns, 90):.0f} max {ns.max():.0f}  total {ns.sum():.0f}")
    names = {9: "setup loads in", 10: "S reduced", 1: "setup done", 12: "prologue issued", 13: "loader probe issued", 14: "loader keys done", 2: "probe done (pw0)", 3: "first task (cw0)", 4: "tasks done (cw0)",
             5: "all warps done", 6: "CTA partial", 8: "ticket won", 11: "headers", 7: "merge end"}
    print(f"CTAs {len(tr)}; last end {(tr[:, 7].max() - t0) / 1e3:.2f} us")
    for i, nm in names.items():
        v = (tr[:, i][tr[:, i] > 0] - t0) / 1e3
        if v.size:
            print(f"  {nm:18s} " + " ".join(f"{x:7.2f}" for x in np.percentile(v, [0, 10, 50, 90, 100])))
    for lab, off in (("iteration start, before V fold (w0)", 16), ("task issue->wait (w0)", 32), ("task K ready (w0)", 48)):
        print(f"  {lab}: p50 over CTAs per index")
        row = []
        for i in range(16):
            v = tr[:, off + i]
            v = (v[v > 0] - t0) / 1e3
            row.append(f"{np.median(v):6.2f}" if v.size else "   -  ")
        print("    " + " ".join(row))


if __name__ == "__main__":
    main()
