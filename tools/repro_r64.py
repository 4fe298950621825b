import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
from paper_2605_06763_b200 import BuildConfig, LouverLayer, synth
n, d, G, H = int(os.environ.get("N", "3000")), 128, 4, 2
r = int(os.environ.get("R", "64"))
K = np.stack([synth.keys(n, d, 100 + h) for h in range(H)])[None]
V = np.stack([synth.keys(n, d, 200 + h) for h in range(H)])[None]
Q = np.stack([synth.queries(G, d, 100 + h) for h in range(H)]).reshape(1, H * G, d)
layer = LouverLayer(d, H, G, 1, n, BuildConfig(S=1, r=r, grouping="contiguous", enclosing="aabb"))
layer.build(K, V)
tau = torch.full((1, H * G), 1e3, device="cuda")
out = torch.zeros((1, H * G, d), device="cuda")
layer.query_device(torch.from_numpy(Q).cuda(), tau, out)
torch.cuda.synchronize()
print("ok", layer.geometry())
