import os, sys, time, json
sys.path.insert(0, os.getcwd())
import numpy as np, torch
import bench
from paper_2605_06763_b200 import BuildConfig, LouverLayer, LayersStep
cfg = dict(bench.CONFIGS["c2"]); L = 8
layers, qs, taus = [], [], []
for l in range(L):
    K, V, Q = bench.gen_layer(cfg, l, 0, os.cpu_count())
    ly = LouverLayer(cfg["d"], cfg["H_kv"], cfg["G"], cfg["batch"], cfg["n"], BuildConfig(S=1, r=bench.CELL, grouping="contiguous", enclosing="aabb"), dtype="bf16")
    ly.build(K, V); layers.append(ly)
    qs.append(torch.from_numpy(Q)); taus.append(torch.from_numpy(bench.taus_device(torch, K, Q, cfg["G"], 0.05)))
qh = torch.stack(qs).pin_memory(); th = torch.stack(taus).pin_memory(); oh = torch.empty_like(qh).pin_memory()
s = torch.cuda.Stream()
step = LayersStep(layers, qh.numpy(), th.numpy(), oh.numpy(), stream=s.cuda_stream)
for _ in range(20): step()
e0 = torch.cuda.Event(enable_timing=True); e1 = torch.cuda.Event(enable_timing=True)
walls, devs = [], []
for _ in range(200):
    t = time.perf_counter()
    e0.record(s); step(); e1.record(s); e1.synchronize()
    walls.append((time.perf_counter() - t) * 1e6); devs.append(e0.elapsed_time(e1) * 1e3)
print("wall per step", np.median(walls), "device (events around the graph)", np.median(devs))
# host-only cost of the call: launch without waiting (graph replays queue up)
t = time.perf_counter()
for _ in range(50): step()
print("back-to-back steps", (time.perf_counter() - t) * 1e6 / 50)
# the bench's device graph (8 query_device calls), replayed one at a time with a sync
qd = [q.cuda() for q in qs]; td = [t.cuda() for t in taus]; od = [torch.zeros_like(q) for q in qd]
def dstep():
    for l in range(L):
        layers[l].query_device(qd[l], td[l], od[l])
def cstep():
    for l in range(L):
        qd[l].copy_(qh[l], non_blocking=True); td[l].copy_(th[l], non_blocking=True)
    dstep()
    for l in range(L):
        oh[l].copy_(od[l], non_blocking=True)
for name, fn in (("kernels only", dstep), ("copies + kernels", cstep)):
    s2 = torch.cuda.Stream(); s2.wait_stream(torch.cuda.current_stream())
    with torch.cuda.stream(s2):
        fn(); fn()
    torch.cuda.current_stream().wait_stream(s2); torch.cuda.synchronize()
    g = torch.cuda.CUDAGraph()
    with torch.cuda.graph(g):
        fn()
    for _ in range(20): g.replay()
    torch.cuda.synchronize()
    devs, walls = [], []
    for _ in range(200):
        t = time.perf_counter()
        e0.record(); g.replay(); e1.record(); e1.synchronize(); devs.append(e0.elapsed_time(e1) * 1e3)
        walls.append((time.perf_counter() - t) * 1e6)
    e0.record()
    for _ in range(50): g.replay()
    e1.record(); e1.synchronize()
    print(name, ": one replay at a time: device", np.median(devs), "wall", np.median(walls), "; back to back", e0.elapsed_time(e1) * 1e3 / 50)
