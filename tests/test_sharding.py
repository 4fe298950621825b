"""Sequence sharding: contiguous partition, one all-gather of
(m, l, o) partials, log-sum-exp combine.

CPU: a world_size-2 gloo job runs the rank-side host logic
(paper_2605_06763_b200.sharding: shard_range + gather_partials) with each
rank's partial computed by the CPU oracle on its shard; the combined output
must equal the oracle's attention over the whole context.
GPU: two shards on one device through the product path (LouverLayer partials
-> lv_lse_merge) against the same unsharded oracle."""
import math
import os
import socket
import tempfile

import numpy as np
import pytest

from paper_2605_06763_b200 import shard_range, synth

N, D = 3000, 64


def test_shard_range_partitions_the_context():
    for n in (0, 1, 7, 3000, 131072):
        for world in (1, 2, 3, 8):
            parts = [shard_range(n, world, r) for r in range(world)]
            assert parts[0][0] == 0
            assert sum(c for _, c in parts) == n
            for (f0, c0), (f1, _) in zip(parts, parts[1:]):
                assert f1 == f0 + c0
            assert max(c for _, c in parts) - min(c for _, c in parts) <= 1
    with pytest.raises(ValueError):
        shard_range(10, 2, 2)


def _inputs():
    K = synth.keys(N, D, 41)
    V = synth.keys(N, D, 42)
    q = synth.queries(1, D, 43)[0]
    return K, V, q


def _oracle_partial(oracle, K, V, q, tau, first, count, scale):
    """(m, l, o[d]) over the selected keys of [first, first + count): o unnormalised."""
    if count == 0:
        return np.concatenate([[-np.inf, 0.0], np.zeros(D)]).astype(np.float32)
    ids = oracle.brute_force_range(K[first:first + count], q, tau)
    if ids.size == 0:
        return np.concatenate([[-np.inf, 0.0], np.zeros(D)]).astype(np.float32)
    s = scale * oracle.scores(K[first:first + count][ids], q).astype(np.float64)
    m = s.max()
    w = np.exp(s - m)
    o = (w[:, None] * V[first:first + count][ids].astype(np.float64)).sum(0)
    return np.concatenate([[m, w.sum()], o]).astype(np.float32)


def _lse_combine(parts):
    m = parts[:, 0].max()
    if not np.isfinite(m):
        return np.zeros(parts.shape[1] - 2)
    w = np.where(np.isfinite(parts[:, 0]), np.exp(parts[:, 0] - m), 0.0)
    return (w[:, None] * parts[:, 2:]).sum(0) / (w * parts[:, 1]).sum()


def _rank_main(rank, world, port, tau, out_path):
    import torch
    import torch.distributed as dist

    from oracle import pyoracle as oracle
    from paper_2605_06763_b200 import gather_partials

    dist.init_process_group("gloo", init_method=f"tcp://127.0.0.1:{port}", rank=rank, world_size=world)
    K, V, q = _inputs()
    first, count = shard_range(N, world, rank)
    part = torch.from_numpy(_oracle_partial(oracle, K, V, q, tau, first, count, np.float32(1 / math.sqrt(D))))
    gathered = gather_partials(part.view(1, D + 2))
    if rank == 0:
        np.save(out_path, gathered.numpy())
    dist.barrier()
    dist.destroy_process_group()


def _free_port():
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


@pytest.mark.parametrize("frac", [0.05, 0.0])
def test_gloo_two_ranks_merge_equals_unsharded(oracle, frac):
    import torch.multiprocessing as mp

    K, V, q = _inputs()
    sc = oracle.scores(K, q)
    # frac 0: tau = the top score of the second shard (few or no keys of the first shard pass)
    tau = np.sort(sc)[::-1][int(0.05 * N)] if frac else np.float32(sc[N // 2:].max())
    with tempfile.TemporaryDirectory() as tmp:
        path = os.path.join(tmp, "g.npy")
        mp.start_processes(_rank_main, args=(2, _free_port(), float(tau), path), nprocs=2, join=True,
                           start_method="spawn")
        parts = np.load(path)[:, 0, :]
    assert parts.shape == (2, D + 2)
    want = oracle.sparse_attention(K, V, [], oracle.brute_force_range(K, q, tau), q, np.float32(1 / math.sqrt(D)))
    got = _lse_combine(parts.astype(np.float64))
    assert want is not None
    assert np.linalg.norm(got - want[2]) <= 1e-5 * np.linalg.norm(want[2])


@pytest.mark.gpu
@pytest.mark.parametrize("empty_shard", [False, True])
def test_two_shards_on_device_lse_merge(oracle, empty_shard):
    import torch

    from paper_2605_06763_b200 import BuildConfig, LouverLayer, lse_merge

    d, H, G, n = 128, 2, 4, 8192
    K = np.stack([synth.keys(n, d, 500 + h) for h in range(H)])[None]
    V = np.stack([synth.keys(n, d, 600 + h) for h in range(H)])[None]
    K = torch.from_numpy(K).to(torch.bfloat16).float().numpy()
    V = torch.from_numpy(V).to(torch.bfloat16).float().numpy()
    Q = synth.queries(H * G, d, 700).reshape(1, H * G, d)
    Q = torch.from_numpy(Q).to(torch.bfloat16).float().numpy()
    tau = np.zeros((1, H * G), np.float32)
    for hq in range(H * G):
        sc = oracle.scores(K[0, hq // G], Q[0, hq])
        tau[0, hq] = np.float32(sc[n // 2:].max()) if empty_shard else np.sort(sc)[::-1][n // 20]
    parts = []
    for rank in range(2):
        first, count = shard_range(n, 2, rank)
        layer = LouverLayer(d, H, G, 1, count, BuildConfig(S=1, r=16, grouping="contiguous", enclosing="aabb"),
                            buffer_capacity=128, dtype="bf16")
        layer.build(np.ascontiguousarray(K[:, :, first:first + count]), np.ascontiguousarray(V[:, :, first:first + count]))
        part = torch.zeros((1, H * G, d + 2), dtype=torch.float32, device="cuda")
        layer.query_device(torch.from_numpy(Q).cuda(), torch.from_numpy(tau).cuda(), None, partial=part)
        parts.append(part.view(H * G, d + 2))
    out = torch.zeros((H * G, d), dtype=torch.float32, device="cuda")
    lse_merge(torch.stack(parts), out)
    torch.cuda.synchronize()
    o = out.cpu().numpy()
    for hq in range(H * G):
        ids = oracle.brute_force_range(K[0, hq // G], Q[0, hq], tau[0, hq])
        want = oracle.sparse_attention(K[0, hq // G], V[0, hq // G], [], ids, Q[0, hq], np.float32(1 / math.sqrt(d)))
        assert want is not None
        assert np.linalg.norm(o[hq] - want[2]) <= 1e-4 * np.linalg.norm(want[2]), hq


# ---------------------------------------------------------------------------------------------
# ShardedLayer end to end: two processes on one GPU (gloo, partials staged through host
# memory), the product kernels on each shard, decode-step inserts into the tail shard across
# a flush, against the unsharded oracle cache (LouverCache with the same prompt and pushes).

_SH = dict(d=128, H=2, G=4, n0=4000, extra=96, B=64)


def _sharded_inputs():
    import torch

    c = _SH
    n = c["n0"] + c["extra"]
    K = np.stack([synth.keys(n, c["d"], 900 + h) for h in range(c["H"])])  # [H][n][d]
    V = np.stack([synth.keys(n, c["d"], 950 + h) for h in range(c["H"])])
    Q = np.stack([synth.queries(c["G"], c["d"], 900 + h) for h in range(c["H"])]).reshape(c["H"] * c["G"], c["d"])
    K = torch.from_numpy(K).to(torch.bfloat16).float().numpy()
    V = torch.from_numpy(V).to(torch.bfloat16).float().numpy()
    return K, V, Q.astype(np.float32)


def _sharded_rank(rank, world, port, tau, out_path):
    import torch
    import torch.distributed as dist

    from paper_2605_06763_b200 import BuildConfig, LouverLayer, ShardedLayer

    c = _SH
    torch.cuda.set_device(0)
    dist.init_process_group("gloo", init_method=f"tcp://127.0.0.1:{port}", rank=rank, world_size=world)
    K, V, Q = _sharded_inputs()
    first, count = shard_range(c["n0"], world, rank)
    layer = LouverLayer(c["d"], c["H"], c["G"], 1, count + c["extra"] + 16,
                        BuildConfig(S=1, r=16, grouping="contiguous", enclosing="aabb"), buffer_capacity=c["B"])
    layer.build(np.ascontiguousarray(K[None, :, first:first + count]), np.ascontiguousarray(V[None, :, first:first + count]))
    sh = ShardedLayer(layer)
    for j in range(c["n0"], c["n0"] + c["extra"]):
        sh.push_key(torch.from_numpy(np.ascontiguousarray(K[None, :, j])).cuda(),
                    torch.from_numpy(np.ascontiguousarray(V[None, :, j])).cuda())
    q = torch.from_numpy(Q[None]).cuda()
    t = torch.from_numpy(np.asarray(tau, np.float32)[None]).cuda()
    out = torch.zeros((1, c["H"] * c["G"], c["d"]), device="cuda")
    bits = torch.zeros((c["H"] * c["G"], layer.bitmap_words), dtype=torch.int32, device="cuda")
    sh.query(q, t, out, sel_bits=bits)
    torch.cuda.synchronize()
    ids = [np.asarray(x, np.int64) + first for x in layer.ids_from_bits(bits)]
    allids = [None] * world
    dist.all_gather_object(allids, ids)
    if rank == 0:
        np.savez(out_path, out=out.cpu().numpy()[0], flushes=layer.flush_count,
                 **{f"ids{r}_{h}": allids[r][h] for r in range(world) for h in range(len(ids))})
    else:
        np.save(out_path + ".tail.npy", np.array([layer.flush_count, layer.indexed_count, layer.n]))
    dist.barrier()
    dist.destroy_process_group()


@pytest.mark.gpu
def test_sharded_layer_two_processes_with_tail_inserts(oracle):
    import torch.multiprocessing as mp

    c = _SH
    K, V, Q = _sharded_inputs()
    n = c["n0"] + c["extra"]
    rq = c["H"] * c["G"]
    # the global ceil(0.05 n)-th score per q head over the whole (sharded) context
    tau = [float(np.sort(oracle.scores(K[hq // c["G"]], Q[hq]))[::-1][int(math.ceil(0.05 * n)) - 1]) for hq in range(rq)]
    with tempfile.TemporaryDirectory() as tmp:
        path = os.path.join(tmp, "sh.npz")
        mp.start_processes(_sharded_rank, args=(2, _free_port(), tau, path), nprocs=2, join=True, start_method="spawn")
        got = np.load(path)
        tail = np.load(path + ".tail.npy")
        out = got["out"]
        ids = [np.sort(np.concatenate([got[f"ids{r}_{h}"] for r in range(2)])) for h in range(rq)]
    # the tail shard flushed once (96 pushes, B = 64) and holds 32 buffer keys
    assert tail[0] == c["extra"] // c["B"] and tail[2] - tail[1] == c["extra"] % c["B"]
    for h in range(c["H"]):
        cache = oracle.Cache(c["d"], oracle.cfg(1, 16, "contiguous", "aabb"), c["B"], keys=K[h, :c["n0"]],
                             values=V[h, :c["n0"]])
        for j in range(c["n0"], n):
            cache.push_key(K[h, j], V[h, j])
        for g in range(c["G"]):
            hq = h * c["G"] + g
            r = cache.query(Q[hq], tau[hq])
            sel, o_want = r["selected"], r["output"]
            assert np.array_equal(ids[hq], np.asarray(sel, np.int64)), hq
            assert np.linalg.norm(out[hq] - o_want) <= 1e-4 * np.linalg.norm(o_want), hq
