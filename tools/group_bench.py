"""Grouped index at the C2 shape (8 kv slots x 131072 keys, d=128, bf16 arena) with the
reference's default BuildConfig (S=4, r=4, PCA tree, ball): device build time (lv_build
with and without the grouped index), query_ta / query_full_subspace candidate time per
slot, and slot 0 checked against the reference library built here on the same bf16-rounded
keys (assignments, member lists, centers, radii of every subspace; TA candidate set)."""
import ctypes as C
import json
import os
import sys
import time

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import torch  # noqa: E402

import bench  # noqa: E402
from oracle import pyoracle as rest  # noqa: E402
from paper_2605_06763_b200 import BuildConfig, LouverLayer, _capi  # noqa: E402


def main():
    cfgd = dict(bench.CONFIGS["c2"])
    n = int(os.environ.get("N", cfgd["n"]))
    cfgd["n"] = n
    K, V, Q = bench.gen_layer(cfgd, 0, 0, os.cpu_count())
    H, G, d = cfgd["H_kv"], cfgd["G"], cfgd["d"]
    bc = BuildConfig(S=4, r=4, grouping="pca_tree", enclosing="ball")
    Kt = torch.from_numpy(K).cuda().to(torch.bfloat16)
    Vt = torch.from_numpy(V).cuda().to(torch.bfloat16)
    res = {"config": f"C2 shape: {H} kv slots x {n} keys, d={d}, bf16 arena; BuildConfig S=4 r=4 pca_tree ball"}
    times = {}
    for gi in (False, True):
        ly = LouverLayer(d, H, G, 1, n, bc, dtype="bf16", group_index=gi)
        ly.build(Kt, Vt)
        torch.cuda.synchronize()
        ts = []
        for _ in range(3):
            t0 = time.perf_counter()
            ly.build(Kt, Vt)
            torch.cuda.synchronize()
            ts.append(time.perf_counter() - t0)
        times[gi] = min(ts)
        if gi:
            layer = ly
    res["build_s_cells_only"] = times[False]
    res["build_s_with_grouped_index"] = times[True]
    res["grouped_index_build_s"] = times[True] - times[False]
    lib = _capi.lib()
    h = layer._ctx.h
    q0 = np.ascontiguousarray(Q[0, 0], np.float32)
    Kb = Kt[0, 0].float().cpu().numpy()  # slot 0 as stored (bf16-rounded)
    tau = float(rest.kth_score(Kb, q0, int(0.05 * n)))
    st = _capi.lv_group_stats()
    ids = np.zeros((n,), np.uint32)
    nl = C.c_int64()
    for algo in (1, 0):
        ts = np.zeros((4,), np.float32)
        if algo == 0:
            assert lib.lv_group_thresholds(h, 0, q0.ctypes.data, tau, ts.ctypes.data, None) == 0
        reps = []
        for _ in range(5):
            t0 = time.perf_counter()
            assert lib.lv_group_candidates(h, 0, q0.ctypes.data, tau, ts.ctypes.data if algo == 0 else None, algo,
                                           None, ids.ctypes.data, n, C.byref(nl), C.byref(st), None) == 0
            reps.append(time.perf_counter() - t0)
        name = "ta" if algo else "full_subspace"
        res[f"{name}_candidates_ms"] = 1e3 * min(reps)
        res[f"{name}_keys_scanned"] = int(st.keys_scanned)
        res[f"{name}_f_scan"] = st.f_scan
        if algo:
            res["ta_stop_depth"] = int(st.ta_stop_depth)
            dev_ta = ids[: nl.value].copy()
    ref = rest.reference_module()
    if ref is not None:  # slot 0 against the reference's own build (index.cpp) on the same keys
        t0 = time.perf_counter()
        rc = ref.Cache(d, ref.cfg(4, 4, "pca_tree", "ball"), 128, Kb, Kb)
        res["reference_build_s_one_slot"] = time.perf_counter() - t0
        ok = True
        for s in range(4):
            w = d // 4
            asg, off, mem, a, _, rad, nb = rc.subspace(s, w, "ball")
            A = np.zeros((n,), np.uint32)
            O = np.zeros((rc.groups(s) + 1,), np.uint32)
            M = np.zeros((n,), np.uint32)
            Ac = np.zeros((w, rc.groups(s)), np.float32)
            R = np.zeros((rc.groups(s),), np.float32)
            nbd = C.c_double()
            assert lib.lv_group_export(h, 0, s, A.ctypes.data, O.ctypes.data, M.ctypes.data, Ac.ctypes.data, None,
                                       R.ctypes.data, C.byref(nbd)) == 0
            ok &= (np.array_equal(A, asg) and np.array_equal(O, off) and np.array_equal(M, mem)
                   and np.array_equal(Ac.view(np.uint32), a.view(np.uint32))
                   and np.array_equal(R.view(np.uint32), rad.view(np.uint32)) and nbd.value == nb)
        rids, rst = rc.candidates(q0, tau, 1)
        res["slot0_index_equals_reference"] = bool(ok)
        res["slot0_ta_candidates_equal_reference"] = bool(np.array_equal(rids, dev_ta))
        res["reference_ta_keys_scanned"] = int(rst["keys_scanned"])
    print(json.dumps(res))


if __name__ == "__main__":
    main()
