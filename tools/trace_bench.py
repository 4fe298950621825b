"""Per-layer timeline of the bench's CUDA graph (C2, 8 layers back to back): every layer
kernel writes per-CTA phase stamps; prints, per layer, when its CTAs start (before the
PDL wait), pass griddepcontrol.wait, finish setup / probe / tasks / partial, and when
the merge ends, relative to the first layer's first CTA."""
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
    L = int(os.environ.get("LAYERS", "8"))
    G = cfg["G"]
    layers, qs, taus, outs, bufs = [], [], [], [], []
    for l in range(L):
        K, V, Q = bench.gen_layer(cfg, l, 0, os.cpu_count())
        layer = LouverLayer(cfg["d"], cfg["H_kv"], G, cfg["batch"], cfg["n"],
                            BuildConfig(S=1, r=bench.CELL, grouping="contiguous", enclosing="aabb"))
        layer.build(K, V)
        layers.append(layer)
        qs.append(torch.from_numpy(Q).cuda())
        taus.append(torch.from_numpy(bench.taus_device(torch, K, Q, G, bench.SELECTIVITY)).cuda())
        outs.append(torch.zeros((cfg["batch"], cfg["H_kv"] * G, cfg["d"]), device="cuda"))
        slots = cfg["batch"] * cfg["H_kv"]
        buf = torch.zeros((slots * 148, 64), dtype=torch.int64, device="cuda")
        layer._ctx.lib.lv_debug_trace(layer._ctx.h, buf.data_ptr())
        bufs.append(buf)

    def step():
        for l in range(L):
            layers[l].query_device(qs[l], taus[l], outs[l])

    s = torch.cuda.Stream()
    s.wait_stream(torch.cuda.current_stream())
    with torch.cuda.stream(s):
        step()
    torch.cuda.current_stream().wait_stream(s)
    torch.cuda.synchronize()
    g = torch.cuda.CUDAGraph()
    with torch.cuda.graph(g):
        step()
    for _ in range(200):
        g.replay()
    torch.cuda.synchronize()
    for b in bufs:
        b.zero_()
    torch.cuda.synchronize()
    g.replay()
    torch.cuda.synchronize()
    trs = [b.cpu().numpy().astype(np.float64) for b in bufs]
    trs = [t[t[:, 0] > 0] for t in trs]
    t0 = min(t[:, 0].min() for t in trs)
    cols = [(0, "start"), (13, "waited"), (1, "setup"), (2, "probe"), (5, "tasks w0"), (6, "partial"),
            (8, "won"), (7, "end")]
    print("layer  " + " ".join(f"{nm:>16s}" for _, nm in cols) + "   (min/max over CTAs, us)")
    for l, t in enumerate(trs):
        row = []
        for i, _ in cols:
            v = t[:, i][t[:, i] > 0]
            row.append(f"{(v.min() - t0) / 1e3:7.2f}/{(v.max() - t0) / 1e3:7.2f}" if v.size else " " * 15)
        print(f"{l:5d}  " + " ".join(f"{x:>16s}" for x in row))
    ends = [t[:, 7][t[:, 7] > 0].max() for t in trs]
    print(f"per-layer period (end to end): {np.diff(ends).mean() / 1e3:.2f} us")
    # merge body of the ticket winners: won -> partials staged (11) -> combined (14) -> end (7)
    seg = []
    for t in trs:
        w = t[(t[:, 8] > 0) & (t[:, 11] > 0) & (t[:, 14] > 0)]
        for r in w:
            seg.append(((r[11] - r[8]) / 1e3, (r[14] - r[11]) / 1e3, (r[7] - r[14]) / 1e3))
    if seg:
        a = np.median(np.array(seg), axis=0)
        print(f"merge (median over winners): stage partials {a[0]:.2f} us, headers + accumulate {a[1]:.2f} us, "
              f"write {a[2]:.2f} us")
    # CTA partial: the CTA's last warp done (5 is warp 0 only) -> partial written (6)
    par = []
    for t in trs:
        w = t[(t[:, 5] > 0) & (t[:, 6] > 0)]
        par.extend(((w[:, 6] - w[:, 5]) / 1e3).tolist())
    if par:
        print(f"warp 0 tasks done -> CTA partial written: median {np.median(par):.2f} us")
    # per CTA: first / last warp done with its tasks (16..31), last warp -> partial written
    spread, red = [], []
    for t in trs:
        w = t[(t[:, 16] > 0) & (t[:, 6] > 0)]
        wd = w[:, 16:32]
        wd = np.where(wd > 0, wd, np.nan)
        spread.extend(((np.nanmax(wd, 1) - np.nanmin(wd, 1)) / 1e3).tolist())
        red.extend(((w[:, 6] - np.nanmax(wd, 1)) / 1e3).tolist())
    # probe: setup done (1) -> first sub-block available (48..63) / warp's probe done (32..47)
    a0, pe = [], []
    for t in trs:
        w = t[(t[:, 1] > 0) & (t[:, 48] > 0)]
        f0 = np.where(w[:, 48:64] > 0, w[:, 48:64], np.nan)
        pd = np.where(w[:, 32:48] > 0, w[:, 32:48], np.nan)
        a0.extend((np.nanmax(f0, 1) - w[:, 1]).tolist())
        pe.extend(((np.nanmax(pd, 1) - w[:, 1]) / 1e3).tolist())
    if a0:
        print(f"probe: setup done -> slowest warp's first sub-block available: median {np.median(a0) / 1e3:.2f} us; "
              f"-> last warp's probe done: median {np.median(pe):.2f} us (max {np.max(pe):.2f})")
    if spread:
        print(f"per CTA: warps' task-finish spread median {np.median(spread):.2f} us (max {np.max(spread):.2f}), "
              f"last warp -> partial written median {np.median(red):.2f} us")
    # per slot (kv head): the team's survivor cells and when its last CTA finished its tasks
    nb = int(layers[0].geometry().get("team_ctas_per_slot", 18)) if hasattr(layers[0], "geometry") else 18
    # the CTA of each slot whose wait returned last (dispatched onto a merging SM of the
    # previous layer): how often it is also the slot's last partial, and how the slot's
    # partial times follow its survivor counts
    late_last, late_gap, corr = 0, [], []
    nslots = 0
    for l in range(1, L):
        t = bufs[l].cpu().numpy().astype(np.float64)
        for sl in range(t.shape[0] // nb):
            tt = t[sl * nb:(sl + 1) * nb]
            tt = tt[(tt[:, 13] > 0) & (tt[:, 6] > 0)]
            if tt.shape[0] < 3:
                continue
            nslots += 1
            il = int(np.argmax(tt[:, 13]))
            late_last += int(il == int(np.argmax(tt[:, 6])))
            late_gap.append((tt[il, 6] - np.median(tt[:, 6])) / 1e3)
            corr.append(np.corrcoef(tt[:, 15], tt[:, 6])[0, 1])
    if nslots:
        print(f"late CTA (last wait) is the slot's last partial in {late_last}/{nslots} slots; its partial vs the "
              f"team median: {np.median(late_gap):+.2f} us; corr(survivor cells, partial time) median "
              f"{np.nanmedian(corr):.2f}")
    for l in (1, 4):
        t = bufs[l].cpu().numpy().astype(np.float64)
        p0 = t[:, 2][t[:, 2] > 0].min()
        print(f"layer {l} per slot: surviving cells (sum / max CTA), last partial after probe (us)")
        for sl in range(t.shape[0] // nb):
            tt = t[sl * nb:(sl + 1) * nb]
            tt = tt[tt[:, 0] > 0]
            if not tt.size:
                continue
            print(f"   slot {sl}: {int(tt[:, 15].sum()):5d} / {int(tt[:, 15].max()):4d}   "
                  f"{(tt[:, 6].max() - p0) / 1e3:6.2f}  (first CTA {(tt[:, 6].min() - p0) / 1e3:6.2f})")


if __name__ == "__main__":
    main()
