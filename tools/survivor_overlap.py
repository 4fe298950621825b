"""How stable are the surviving cells along a decode stream? For one C2 slot (131,072 keys
of the reference's decode-trace law, 16-key cells), consecutive decode queries (rows of
gen_synthetic_queries, G = 4 per step) each with its own tau = the 5 % score: the overlap of
the surviving-cell sets between steps, and the per-CTA survivor counts (18 team CTAs) under
the fine interleave vs under an ownership dealt from the previous step's survivors."""
import os
import sys

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import bench  # noqa: E402
from paper_2605_06763_b200 import synth  # noqa: E402


def main():
    n, d, G, nb, steps = 131072, 128, 4, 18, 6
    seed = int(bench.layer_seeds(0, 0, 0, 0, 8))
    K = synth.keys(n, d, seed)
    Q = synth.queries(G * steps, d, seed)
    lo, hi = K.reshape(-1, 16, d).min(1), K.reshape(-1, 16, d).max(1)

    def survivors(q):
        m = np.zeros(len(lo), bool)
        for g in range(G):
            s = K @ q[g]
            tau = np.sort(s)[-int(np.ceil(0.05 * n))]
            m |= np.maximum(hi * q[g], lo * q[g]).sum(1) >= tau
        return m

    S = [survivors(Q[G * i:G * (i + 1)]) for i in range(steps)]
    C = len(lo)
    inter = np.arange(C) % nb

    def dealt(prev):
        own = np.empty(C, int)
        for mask in (prev, ~prev):
            idx = np.nonzero(mask)[0]
            own[idx] = np.arange(len(idx)) % nb
        return own

    for i in range(1, steps):
        ci = np.bincount(inter[S[i]], minlength=nb)
        cp = np.bincount(dealt(S[i - 1])[S[i]], minlength=nb)
        print(f"step {i}: surviving cells {S[i].sum()}, overlap with step {i - 1}: "
              f"{np.sum(S[i] & S[i - 1]) / S[i].sum():.3f}; max/mean per CTA: interleave {ci.max()}/{ci.mean():.1f}, "
              f"dealt from the previous step {cp.max()}/{cp.mean():.1f}")


if __name__ == "__main__":
    main()
