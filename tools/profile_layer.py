"""One C2 layer (8 kv x 4 q heads, 128K keys, bf16): run the Louver query and the
dense decode a few times — a short command for ncu captures."""
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import torch  # noqa: E402

import bench  # noqa: E402
from paper_2605_06763_b200 import BuildConfig, LouverLayer  # noqa: E402


def main():
    reps = int(os.environ.get("REPS", "3"))
    which = os.environ.get("WHICH", "both")
    cfg = dict(bench.CONFIGS[os.environ.get("CONFIG", "c2")])
    K, V, Q = bench.gen_layer(cfg, 0, 0, os.cpu_count())
    G = cfg["G"]
    tau = bench.taus_device(torch, K, Q, G, bench.SELECTIVITY)
    layer = LouverLayer(cfg["d"], cfg["H_kv"], G, cfg["batch"], cfg["n"],
                        BuildConfig(S=1, r=bench.CELL, grouping="contiguous", enclosing="aabb"),
                        dtype=cfg["dtype"])
    layer.build(K, V)
    q, t = torch.from_numpy(Q).cuda(), torch.from_numpy(tau).cuda()
    out = torch.zeros((cfg["batch"], cfg["H_kv"] * G, cfg["d"]), device="cuda")
    if which == "insert":  # one decode step's key per kv slot, a few steps
        kk = torch.from_numpy(K[:, :, :reps].transpose(2, 0, 1, 3).copy()).cuda()  # [reps][B][H][d]
        layer2 = LouverLayer(cfg["d"], cfg["H_kv"], G, cfg["batch"], cfg["n"] + 1024,
                             BuildConfig(S=1, r=bench.CELL, grouping="contiguous", enclosing="aabb"),
                             dtype=cfg["dtype"])
        layer2.build(K, V)
        for i in range(reps):
            layer2.push_key(kk[i], kk[i])
        torch.cuda.synchronize()
        print("done insert")
        return
    for _ in range(reps):
        if which in ("both", "query"):
            layer.query_device(q, t, out)
        if which in ("both", "dense"):
            layer.dense_decode(q, out)
    torch.cuda.synchronize()
    print("done", layer.geometry())


if __name__ == "__main__":
    main()
