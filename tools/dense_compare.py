"""Full-scan dense decode at C2 (32 q / 8 kv heads, d = 128, 131072 keys, bf16): this repo's
kernel (lv_dense_decode: the layer kernel in DENSE mode) against the library kernels in the
image (torch SDPA, FlashInfer single_decode_with_kv_cache, flash_attn_with_kvcache).

Each variant runs L independent layers (4 GiB of KV, larger than L2) captured in one CUDA
graph; per-layer time = replay time / L, median of REPS replays after warm-up. Output
error of each against float64 attention on layer 0 is printed too."""
import json
import math
import os
import statistics
import sys

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import torch  # noqa: E402

import bench  # noqa: E402
from paper_2605_06763_b200 import BuildConfig, LouverLayer  # noqa: E402

L = int(os.environ.get("LAYERS", "8"))
REPS = int(os.environ.get("REPS", "50"))


def graph_time(fn):
    s = torch.cuda.Stream()
    s.wait_stream(torch.cuda.current_stream())
    with torch.cuda.stream(s):
        for _ in range(2):
            fn()
    torch.cuda.current_stream().wait_stream(s)
    torch.cuda.synchronize()
    g = torch.cuda.CUDAGraph()
    with torch.cuda.graph(g):
        fn()
    for _ in range(5):
        g.replay()
    torch.cuda.synchronize()
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    ts = []
    for _ in range(REPS):
        a.record()
        g.replay()
        b.record()
        b.synchronize()
        ts.append(a.elapsed_time(b) * 1e3 / L)
    return statistics.median(ts)


def main():
    cfg = dict(bench.CONFIGS["c2"])
    B, H, G, d, n = cfg["batch"], cfg["H_kv"], cfg["G"], cfg["d"], cfg["n"]
    Hq = H * G
    layers, qs, outs, kts, vts = [], [], [], [], []
    for l in range(L):
        K, V, Q = bench.gen_layer(cfg, l, 0, os.cpu_count())
        layer = LouverLayer(d, H, G, B, n, BuildConfig(S=1, r=16, grouping="contiguous", enclosing="aabb"))
        layer.build(K, V)
        layers.append(layer)
        qs.append(torch.from_numpy(Q).cuda())
        outs.append(torch.zeros((B, Hq, d), device="cuda"))
        kts.append(torch.from_numpy(K).to("cuda", torch.bfloat16))  # [B][H][n][d]
        vts.append(torch.from_numpy(V).to("cuda", torch.bfloat16))
    # float64 reference on layer 0
    k0, v0, q0 = kts[0][0].double(), vts[0][0].double(), qs[0][0].double()
    ref = torch.empty((Hq, d), dtype=torch.float64, device="cuda")
    for hq in range(Hq):
        s = (k0[hq // G] @ q0[hq]) / math.sqrt(d)
        w = torch.softmax(s, 0)
        ref[hq] = w @ v0[hq // G]

    def err(o):
        o = o.reshape(Hq, d).double()
        return float(((o - ref).norm(dim=1) / ref.norm(dim=1)).max())

    res = {}
    bytes_ = B * H * n * d * 2 * 2

    def own():
        for l in range(L):
            layers[l].dense_decode(qs[l], outs[l])

    own()
    torch.cuda.synchronize()
    res["own_lv_dense_decode"] = {"us": graph_time(own), "max_rel_err": err(outs[0])}

    import torch.nn.functional as F
    qb = [q.to(torch.bfloat16).view(B, Hq, 1, d) for q in qs]
    so = [None] * L

    def sdpa():
        for l in range(L):
            so[l] = F.scaled_dot_product_attention(qb[l], kts[l], vts[l], enable_gqa=True)

    try:
        sdpa()
        torch.cuda.synchronize()
        res["torch_sdpa"] = {"us": graph_time(sdpa), "max_rel_err": err(so[0].float())}
    except Exception as e:  # pragma: no cover
        res["torch_sdpa"] = {"error": str(e)[:200]}

    try:
        import flashinfer

        kf = [k[0].transpose(0, 1).contiguous() for k in kts]  # [n][H][d] (NHD)
        vf = [v[0].transpose(0, 1).contiguous() for v in vts]
        qf = [q.to(torch.bfloat16)[0] for q in qs]  # [Hq][d]
        fo = [None] * L

        def fi():
            for l in range(L):
                fo[l] = flashinfer.single_decode_with_kv_cache(qf[l], kf[l], vf[l], kv_layout="NHD")

        fi()
        torch.cuda.synchronize()
        res["flashinfer_single_decode"] = {"us": graph_time(fi), "max_rel_err": err(fo[0].float())}
        del kf, vf
    except Exception as e:  # pragma: no cover
        res["flashinfer_single_decode"] = {"error": str(e)[:300]}

    try:  # TensorRT-LLM-gen decode kernels shipped as sm_100 cubins (flashinfer-cubin), paged HND
        import flashinfer

        page = 128
        npg = n // page
        # [pages][H][page][d] strided views of the [B=1][H][n][d] caches (no copy)
        kp = [k[0].view(H, npg, page, d).permute(1, 0, 2, 3) for k in kts]
        vp = [v[0].view(H, npg, page, d).permute(1, 0, 2, 3) for v in vts]
        qt = [q.to(torch.bfloat16)[0] for q in qs]  # [Hq][d]
        ws = torch.zeros(256 << 20, dtype=torch.uint8, device="cuda")
        bt = torch.arange(npg, dtype=torch.int32, device="cuda").view(1, npg)
        sl = torch.tensor([n], dtype=torch.int32, device="cuda")
        to = [torch.empty((Hq, d), dtype=torch.bfloat16, device="cuda") for _ in range(L)]

        def trt():
            for l in range(L):
                flashinfer.decode.trtllm_batch_decode_with_kv_cache(
                    qt[l], (kp[l], vp[l]), ws, bt, sl, n, bmm1_scale=1.0 / math.sqrt(d), bmm2_scale=1.0,
                    out=to[l], kv_layout="HND")

        trt()
        torch.cuda.synchronize()
        res["flashinfer_trtllm_gen_decode"] = {"us": graph_time(trt), "max_rel_err": err(to[0].float())}
    except Exception as e:  # pragma: no cover
        res["flashinfer_trtllm_gen_decode"] = {"error": str(e)[:300]}

    try:
        from flash_attn import flash_attn_with_kvcache

        kc = [k.transpose(1, 2).contiguous() for k in kts]  # [B][n][H][d]
        vc = [v.transpose(1, 2).contiguous() for v in vts]
        qc = [q.to(torch.bfloat16).view(B, 1, Hq, d) for q in qs]
        fa = [None] * L

        def fa2():
            for l in range(L):
                fa[l] = flash_attn_with_kvcache(qc[l], kc[l], vc[l])

        fa2()
        torch.cuda.synchronize()
        res["flash_attn_with_kvcache"] = {"us": graph_time(fa2), "max_rel_err": err(fa[0].float())}
    except Exception as e:  # pragma: no cover
        res["flash_attn_with_kvcache"] = {"error": str(e)[:300]}

    for k, v in res.items():
        if "us" in v:
            v["achieved_gbs"] = bytes_ / (v["us"] * 1e-6) / 1e9
    print(json.dumps({"config": "C2 dense full scan", "layers": L, "kv_bytes_per_layer": bytes_, "results": res},
                     indent=1))


if __name__ == "__main__":
    main()
