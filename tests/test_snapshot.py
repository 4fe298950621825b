"""Snapshots: the reference's LVKD / LVIX formats
(io.hpp:40-51, io.cpp:205-317). Ports test_io.cpp:74-123; the LVIX files are
checked with an independent reader restated from io.cpp:270-317 here, and a
reference-style snapshot of the oracle's own PCA-tree / ball index (S = 4) is
written with a writer restated from io.cpp:236-268 and loaded by the device cache."""
import math
import struct

import numpy as np
import pytest

from paper_2605_06763_b200 import BuildConfig, LouverCache, LouverError, QueryRequest
from paper_2605_06763_b200.snapshot import load_dataset, load_index, save_dataset, save_index


def rmat(n, d, seed):
    return np.random.default_rng(seed).standard_normal((n, d)).astype(np.float32)


def test_dataset_round_trip_and_corruption(tmp_path):  # test_io.cpp:74-92
    data = rmat(100, 12, 3)
    p = tmp_path / "data.lvkd"
    save_dataset(p, data)
    raw = p.read_bytes()
    assert raw[:4] == b"LVKD" and struct.unpack("<III", raw[4:16]) == (1, 100, 12)
    assert np.array_equal(load_dataset(p), data)
    (tmp_path / "trunc.lvkd").write_bytes(raw[: len(raw) // 2])
    with pytest.raises(LouverError, match="corrupt"):
        load_dataset(tmp_path / "trunc.lvkd")
    (tmp_path / "bad.lvkd").write_bytes(b"NOPE" + raw[4:])
    with pytest.raises(LouverError, match="magic"):
        load_dataset(tmp_path / "bad.lvkd")
    (tmp_path / "trail.lvkd").write_bytes(raw + b"\0")
    with pytest.raises(LouverError, match="trailing"):
        load_dataset(tmp_path / "trail.lvkd")


# ------------------------------------------------- LVIX reader / writer restated (test-only)


def read_lvix(raw: bytes):
    """io.cpp:270-317."""
    o = 0

    def get(fmt):
        nonlocal o
        v = struct.unpack_from("<" + fmt, raw, o)
        o += struct.calcsize("<" + fmt)
        return v if len(v) > 1 else v[0]

    assert raw[:4] == b"LVIX"
    o = 4
    ver, d, S, r, grouping, enclosing = get("IIIIII")
    seed, m = get("QQ")
    subs = []
    for _ in range(S):
        asz = get("Q")
        asg = np.frombuffer(raw, np.uint32, asz, o)
        o += 4 * asz
        groups = []
        for _ in range(get("I")):
            kind = get("I")
            vecs = []
            for _ in range(2 if kind == 1 else 1):
                ln = get("I")
                vecs.append(np.frombuffer(raw, np.float32, ln, o))
                o += 4 * ln
            rad = None if kind == 1 else get("f")
            msz = get("I")
            mem = np.frombuffer(raw, np.uint32, msz, o)
            o += 4 * msz
            groups.append((kind, vecs, rad, mem))
        subs.append((asg, groups))
    assert o == len(raw)
    return dict(version=ver, d=d, S=S, r=r, grouping=grouping, enclosing=enclosing, seed=seed, m=m, subs=subs)


def write_lvix(d, S, r, grouping, enclosing, seed, m, subs) -> bytes:
    """io.cpp:236-268; subs = [(assignments, [(kind, [vecs], radius, members)])]."""
    out = [b"LVIX", struct.pack("<IIIIIIQQ", 1, d, S, r, grouping, enclosing, seed, m)]
    for asg, groups in subs:
        out.append(struct.pack("<Q", len(asg)) + np.asarray(asg, np.uint32).tobytes())
        out.append(struct.pack("<I", len(groups)))
        for kind, vecs, rad, mem in groups:
            out.append(struct.pack("<I", kind))
            for v in vecs:
                out.append(struct.pack("<I", len(v)) + np.asarray(v, np.float32).tobytes())
            if kind != 1:
                out.append(struct.pack("<f", rad))
            out.append(struct.pack("<I", len(mem)) + np.asarray(mem, np.uint32).tobytes())
    return b"".join(out)


@pytest.fixture(scope="module")
def torch():
    import torch

    assert torch.cuda.is_available(), "GPU tests need a CUDA device"
    return torch


def answers(cache, d, trials=25):
    res = []
    for t in range(trials):
        q = np.random.default_rng(600 + t).standard_normal(d).astype(np.float32)
        a = cache.query(QueryRequest(q=q, tau=float(t) - 5.0))
        res.append((list(a.selected), list(a.retrieved)))
    return res


@pytest.mark.gpu
def test_index_snapshot_round_trips(torch, tmp_path):  # test_io.cpp:94-123
    d, n0, extra = 32, 512, 40
    keys = rmat(n0 + extra, d, 5)
    # without the grouped index the snapshot is the device cells (tests/test_groups.py covers
    # the grouped index's snapshot, byte-equal to the reference's)
    c = LouverCache.adopt(keys[:n0], keys[:n0].copy(), BuildConfig(S=1, r=16), 64, group_index=False)
    for j in range(n0, n0 + extra):
        c.push_key(keys[j], keys[j])
    m = c.indexed_count()
    p = tmp_path / "index.lvix"
    save_index(c, p)
    f = read_lvix(p.read_bytes())
    assert (f["version"], f["d"], f["S"], f["r"], f["grouping"], f["enclosing"], f["m"]) == (1, d, 1, 16, 0, 1, m)
    asg, groups = f["subs"][0]
    assert np.array_equal(asg, np.arange(m) // 16)
    for g, (kind, (lo, hi), _, mem) in enumerate(groups):
        rows = keys[g * 16: min(m, g * 16 + 16)]
        assert kind == 1 and np.array_equal(mem, np.arange(g * 16, g * 16 + rows.shape[0]))
        assert np.array_equal(lo, rows.min(0)) and np.array_equal(hi, rows.max(0))
    # a fresh cache over the same rows adopts the snapshot's indexed_count: same answers
    c2 = LouverCache.adopt(keys, keys.copy(), BuildConfig(S=1, r=16), 64)
    assert c2.indexed_count() == n0 + extra
    assert load_index(c2, p) == m and c2.indexed_count() == m and c2.pending_count() == c.pending_count()
    assert answers(c2, d) == answers(c, d)
    raw = p.read_bytes()
    for name, blob, err in [("trunc", raw[:-7], "corrupt"), ("magic", b"NOPE" + raw[4:], "magic"),
                            ("trail", raw + b"\0", "trailing")]:
        (tmp_path / f"{name}.lvix").write_bytes(blob)
        with pytest.raises(LouverError, match=err):
            load_index(c2, tmp_path / f"{name}.lvix")
    assert c2.indexed_count() == m  # no partial state
    with pytest.raises(ValueError):
        load_index(LouverCache.adopt(rmat(8, 16, 1), rmat(8, 16, 2), BuildConfig(S=1, r=4), 8), p)


@pytest.mark.gpu
def test_loads_reference_pca_ball_snapshot(torch, oracle, tmp_path):
    """A reference-style LVIX of the oracle's PCA-tree / ball index (S = 4) is accepted and
    gives the same final sets as the oracle cache it describes."""
    d, n = 32, 600
    keys = rmat(n, d, 8)
    oc = oracle.Cache(d, oracle.cfg(4, 4, "pca_tree", "ball", 1), 64, keys=keys[:512], values=keys[:512])
    for j in range(512, n):
        oc.push_key(keys[j], keys[j])
    m = oc.indexed_count()
    subs = []
    for s in range(4):
        G = oc.groups(s)
        asg = np.zeros(m, np.uint32)
        groups = []
        for g in range(G):
            mem = oc.group_members(s, g)
            asg[mem] = g
            groups.append((0, [np.zeros(d // 4, np.float32)], 1.0, mem))
        subs.append((asg, groups))
    p = tmp_path / "ref.lvix"
    p.write_bytes(write_lvix(d, 4, 4, 3, 0, 1, m, subs))
    c = LouverCache.adopt(keys, keys.copy(), BuildConfig(S=4, r=4), 64)
    assert load_index(c, p) == m
    for t in range(20):
        q = np.random.default_rng(900 + t).standard_normal(d).astype(np.float32)
        tau = float(t) - 4.0
        a = c.query(QueryRequest(q=q, tau=tau))
        b = oc.query(q, tau)
        assert list(a.selected) == list(b["selected"]) and list(a.retrieved) == list(b["retrieved"])
    # a snapshot whose groups do not partition the indexed keys is rejected
    bad = [(subs[0][0], subs[0][1][:-1])] + subs[1:]
    (tmp_path / "bad.lvix").write_bytes(write_lvix(d, 4, 4, 3, 0, 1, m, bad))
    with pytest.raises(LouverError, match="partition"):
        load_index(c, tmp_path / "bad.lvix")
