"""Diagnostic: attention-output error of the bf16 layer path vs float64 exact attention
over the same attended set, next to the oracle's (normative fp32) error, for several d."""
import math
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
sys.path.insert(0, os.path.join(ROOT, "tests"))
import numpy as np  # noqa: E402
import torch  # noqa: E402

from oracle import pyoracle as oracle  # noqa: E402
from test_gpu_parity import make_layer, taus_at  # noqa: E402

for d in (128, 200, 256):
    layer, K, V, Q = make_layer(torch, oracle, H_kv=2, G=4, batch=2, n=1500, d=d, r=16, seed=300 + d)
    tau = taus_at(oracle, K, Q, 4, 0.05)
    out = torch.zeros((2, 8, d), device="cuda")
    layer.query_device(torch.from_numpy(Q).cuda(), torch.from_numpy(tau).cuda(), out)
    torch.cuda.synchronize()
    o = out.cpu().numpy()
    worst = (0, 0, 0)
    for b in range(2):
        for hq in range(8):
            kh, vh = K[b, hq // 4].astype(np.float64), V[b, hq // 4].astype(np.float64)
            q = Q[b, hq].astype(np.float64)
            sel = oracle.brute_force_range(K[b, hq // 4], Q[b, hq], tau[b, hq])
            att = np.union1d(sel[sel < layer.indexed_count], np.arange(layer.indexed_count, layer.n))
            s = (kh[att] @ q) / math.sqrt(d)
            w = np.exp(s - s.max())
            exact = (w[:, None] * vh[att]).sum(0) / w.sum()
            ow = oracle.sparse_attention(K[b, hq // 4], V[b, hq // 4], [], att, Q[b, hq], np.float32(1 / math.sqrt(d)))
            e_dev = np.linalg.norm(o[b, hq] - exact) / np.linalg.norm(exact)
            e_or = np.linalg.norm(ow[2] - exact) / np.linalg.norm(exact)
            if e_dev > worst[0]:
                worst = (e_dev, e_or, float(s.max() - np.sort(s)[-2]) if s.size > 1 else 0.0, float(np.abs(s).max()))
    print(f"d={d}: worst device rel err vs fp64 {worst[0]:.2e}, oracle {worst[1]:.2e}; max |s| {worst[3]:.1f}")
