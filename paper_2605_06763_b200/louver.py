"""Python mirror of the reference Louver API over the C ABI.

Names, argument meaning and error behaviour follow the reference headers
(/root/reference/proj/include/louver/{cache,query,index}.hpp):

* ``BuildConfig``       — index.hpp:10-22 (validated the same way)
* ``QueryRequest``      — query.hpp:11-20 (``effective_scale`` = 1/sqrt(d) when 0)
* ``FilterAlgo``        — cache.hpp:7
* ``LouverCache``       — cache.hpp:21-63: push_key / flush_buffer / query /
                          indexed_count / pending_count / pending_ids / flush_count
* ``CacheQueryResult``  — cache.hpp:11-16 (selected, retrieved, stats, attention)
* ``brute_force_range`` — query.hpp:44-45, ``sparse_attention`` — query.hpp:69-72

``LouverCache`` is the single-head cache of the reference (one kv head, one q
head, fp32 storage). ``LouverLayer`` is the batched, grouped-query form used
for real decode layers (bf16 KV, H_kv heads x G q heads x batch); its
``query_device`` is the hot path that bench.py measures. Exceptions:
``ValueError`` <- std::invalid_argument, ``IndexError`` <- std::out_of_range.
Empty attention sets give ``attention = None`` (std::nullopt).
"""
from __future__ import annotations

import ctypes as C
import dataclasses
import enum
import math
import threading
from typing import List, Optional, Sequence

import numpy as np

from . import _capi
from ._capi import LV_BF16, LV_DEVICE, LV_EMPTY, LV_F32, LV_HOST, check

_GROUPING = {"contiguous": 0, "interleaved": 1, "random": 2, "pca_tree": 3, "pca": 3}
_ENCLOSURE = {"ball": 0, "aabb": 1, "span_ball": 2, "spanball": 2}


def _torch():
    import torch  # plumbing only: device buffers and streams

    return torch


class FilterAlgo(enum.IntEnum):
    FullSubspace = 0
    Ta = 1


@dataclasses.dataclass
class BuildConfig:
    """index.hpp:10-22. On the device, keys are grouped into contiguous cells of
    ``r`` keys (rounded up to a power of two, at most 64) with AABB summaries;
    S/grouping/enclosing only affect pruning statistics, never the results."""

    S: int = 4
    r: int = 4
    grouping: str = "pca_tree"
    enclosing: str = "ball"
    rng_seed: int = 0

    def validate(self, d: int) -> None:
        if self.S < 1:
            raise ValueError("BuildConfig: S >= 1 required")
        if self.r < 1:
            raise ValueError("BuildConfig: r >= 1 required")
        if self.S > d:
            raise ValueError("BuildConfig: S <= d required")
        if self.grouping not in _GROUPING:
            raise ValueError(f"unknown grouping strategy: {self.grouping}")
        if self.enclosing not in _ENCLOSURE:
            raise ValueError(f"unknown enclosure kind: {self.enclosing}")


@dataclasses.dataclass
class QueryRequest:
    q: np.ndarray
    tau: float = 0.0
    tau_subspace: Optional[List[float]] = None
    scale: float = 0.0

    def effective_scale(self) -> float:
        if self.scale != 0.0:
            return float(self.scale)
        return float(np.float32(1.0 / math.sqrt(float(len(self.q)))))


@dataclasses.dataclass
class QueryStats:
    groups_tested: int = 0
    keys_scanned: int = 0
    f_scan: float = 0.0
    gate_cost_equiv: float = 0.0
    ta_stop_depth: Optional[int] = None
    ta_stop_upper: Optional[float] = None


@dataclasses.dataclass
class CandidateSet:
    """query.hpp:34-37: live ids (ascending, duplicate-free) and the filter's statistics."""
    live_ids: np.ndarray
    stats: QueryStats


@dataclasses.dataclass
class SubspaceIndex:
    """One subspace of the grouped index (index.hpp:29-52), copied from the device."""
    assignments: np.ndarray            # key id -> group id
    member_offsets: np.ndarray         # [K + 1]
    member_ids: np.ndarray             # group g: member_ids[member_offsets[g]:member_offsets[g + 1]]
    gate_centers: Optional[np.ndarray]  # [w][K] (ball kinds)
    gate_radii: Optional[np.ndarray]    # [K]
    gate_lo: Optional[np.ndarray]       # [w][K] (AABB)
    gate_hi: Optional[np.ndarray]
    norm_bound: float


@dataclasses.dataclass
class AttentionResult:
    selected_ids: np.ndarray           # attended token ids, ascending
    weights: Optional[np.ndarray]      # aligned with selected_ids (when requested)
    output: np.ndarray


@dataclasses.dataclass
class CacheQueryResult:
    selected: np.ndarray               # all ids with q.k >= tau, ascending
    retrieved: np.ndarray              # selected (indexed part) ∪ buffer
    stats: QueryStats
    attention: Optional[AttentionResult]


def _config(d, heads, group, batch, dtype, cfg: BuildConfig, B, capacity, group_index=False) -> _capi.lv_config:
    return _capi.lv_config(
        d=d, n_kv_heads=heads, group_size=group, batch=batch, dtype=dtype, S=cfg.S, r=cfg.r,
        grouping=_GROUPING.get(cfg.grouping, -1), enclosure=_ENCLOSURE.get(cfg.enclosing, -1),
        rng_seed=cfg.rng_seed, buffer_capacity=B, capacity=capacity, group_index=1 if group_index else 0,
    )


def _ptr(a) -> Optional[int]:
    if a is None:
        return None
    if isinstance(a, np.ndarray):
        return a.ctypes.data
    return a.data_ptr()


class _Context:
    """Owns one lv_ctx (one layer: batch x H_kv slots)."""

    def __init__(self, cfg: _capi.lv_config):
        self.lib = _capi.lib()
        self.cfg = cfg
        h = C.c_void_p()
        check(self.lib.lv_create(C.byref(cfg), C.byref(h)), "lv_create")
        self.h = h

    def close(self):
        if getattr(self, "h", None):
            self.lib.lv_destroy(self.h)
            self.h = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass

    @property
    def n(self) -> int:
        return int(self.lib.lv_n(self.h))

    @property
    def indexed(self) -> int:
        return int(self.lib.lv_indexed_count(self.h))

    @property
    def flushes(self) -> int:
        return int(self.lib.lv_flush_count(self.h))

    @property
    def bitmap_words(self) -> int:
        return int(self.lib.lv_bitmap_words(self.h))

    def bits_to_ids(self, bits, rows: int, limit: int) -> List[np.ndarray]:
        """Expand device bitmaps [rows][words] into ascending id arrays (device kernel)."""
        torch = _torch()
        words = self.bitmap_words
        ids = torch.empty((rows, max(limit, 1)), dtype=torch.int32, device=bits.device)
        cnt = torch.empty((rows,), dtype=torch.int32, device=bits.device)
        stream = torch.cuda.current_stream(bits.device).cuda_stream
        check(self.lib.lv_bitmap_to_ids(bits.data_ptr(), words, rows, limit, ids.data_ptr(),
                                        ids.shape[1], cnt.data_ptr(), stream), "lv_bitmap_to_ids")
        ids_h = ids.cpu().numpy().view(np.uint32)
        cnt_h = cnt.cpu().numpy()
        return [ids_h[i, : cnt_h[i]].copy() for i in range(rows)]


class LouverCache:
    """Single-head KV store + Louver index + update buffer (cache.hpp:21-63).

    ``LouverCache(dim, cfg, buffer_capacity)`` starts empty;
    ``LouverCache.adopt(keys, values, cfg, buffer_capacity)`` indexes an
    existing store immediately (cache.hpp:31-36). Storage is fp32 in HBM and
    grows geometrically like KeyStore (core.hpp:134-142).
    """

    def __init__(self, dim: int, cfg: BuildConfig, buffer_capacity: int, capacity: int = 1024,
                 group_index: bool = True):
        cfg.validate(dim)
        if buffer_capacity < 1:
            raise ValueError("LouverCache: buffer capacity >= 1 required")
        self.d = dim
        self.cfg = cfg
        self.B = int(buffer_capacity)
        # group_index: the reference's LouverIndex for cfg (PCA tree, balls, S subspaces ...)
        # is also built on the device; it supplies query()'s QueryStats and candidate sets
        self.group_index = bool(group_index)
        self._ctx = _Context(_config(dim, 1, 1, 1, LV_F32, cfg, self.B, max(capacity, 16), self.group_index))
        self._cap = max(capacity, 16)
        self._pool_lock = threading.Lock()
        self._pool = []  # (bits, totals) device scratch leased by queries

    @classmethod
    def adopt(cls, keys: np.ndarray, values: np.ndarray, cfg: BuildConfig, buffer_capacity: int,
              group_index: bool = True):
        keys = np.ascontiguousarray(keys, dtype=np.float32)
        values = np.ascontiguousarray(values, dtype=np.float32)
        if keys.shape != values.shape or keys.ndim != 2:
            raise ValueError("KeyStore: keys/values shape mismatch")
        n, d = keys.shape
        self = cls(d, cfg, buffer_capacity, capacity=max(2 * n, 1024), group_index=group_index)
        if n:
            check(self._ctx.lib.lv_build(self._ctx.h, _ptr(keys), _ptr(values), n, LV_F32, LV_HOST,
                                         None), "lv_build")
        return self

    # -- writer side -----------------------------------------------------------
    def push_key(self, k, v) -> None:
        k = np.ascontiguousarray(k, dtype=np.float32).reshape(-1)
        v = np.ascontiguousarray(v, dtype=np.float32).reshape(-1)
        if k.size != self.d or v.size != self.d:
            raise ValueError("KeyStore::append: dimension mismatch")
        if self._ctx.n >= self._cap:
            self._cap = max(16, 2 * self._cap)
            check(self._ctx.lib.lv_reserve(self._ctx.h, self._cap, None), "lv_reserve")
        check(self._ctx.lib.lv_push_key(self._ctx.h, _ptr(k), _ptr(v), LV_F32, LV_HOST, None),
              "lv_push_key")

    def flush_buffer(self) -> bool:
        return check(self._ctx.lib.lv_flush(self._ctx.h, None), "lv_flush") == _capi.LV_OK

    # -- accessors ---------------------------------------------------------------
    def n(self) -> int:
        return self._ctx.n

    def indexed_count(self) -> int:
        return self._ctx.indexed

    def pending_count(self) -> int:
        return self._ctx.n - self._ctx.indexed

    def pending_ids(self) -> np.ndarray:
        return np.arange(self._ctx.indexed, self._ctx.n, dtype=np.uint32)

    def flush_count(self) -> int:
        return self._ctx.flushes

    def buffer_capacity(self) -> int:
        return self.B

    def keys(self) -> np.ndarray:
        out = np.empty((self.n(), self.d), dtype=np.float32)
        if self.n():
            check(self._ctx.lib.lv_read_rows(self._ctx.h, 0, 0, self.n(), 0, _ptr(out)), "lv_read_rows")
        return out

    def values(self) -> np.ndarray:
        out = np.empty((self.n(), self.d), dtype=np.float32)
        if self.n():
            check(self._ctx.lib.lv_read_rows(self._ctx.h, 0, 0, self.n(), 1, _ptr(out)), "lv_read_rows")
        return out

    # -- reader side -------------------------------------------------------------
    def query(self, req: QueryRequest, algo: FilterAlgo = FilterAlgo.Ta, strict_threshold: bool = False,
              want_weights: bool = False) -> CacheQueryResult:
        """cache.cpp:30-70. The attention's weights (query.cpp:359-365) come from the
        query's own (m, l) and the normative scores of the attended ids; ``want_weights``
        is accepted for compatibility (weights are always filled, as in the reference).
        Device scratch is leased from a per-cache pool (no allocation per query)."""
        q = np.ascontiguousarray(req.q, dtype=np.float32).reshape(-1)
        if q.size != self.d:
            raise ValueError("dot: length mismatch")
        tau = np.array([req.tau], dtype=np.float32)
        out = np.zeros((self.d,), dtype=np.float32)
        part = np.zeros((self.d + 2,), dtype=np.float32)
        counts = np.zeros((4,), dtype=np.int32)
        bits, totals = self._lease()
        try:
            args = _capi.lv_query_args(
                q=_ptr(q), tau=_ptr(tau), scale=req.effective_scale(), algo=int(algo),
                strict=1 if strict_threshold else 0, where=LV_HOST, out=_ptr(out), partial=_ptr(part),
                counts=_ptr(counts), sel_bits=bits.data_ptr(), totals=totals.data_ptr(), workspace=None,
                stream=None,
            )
            check(self._ctx.lib.lv_query(self._ctx.h, C.byref(args)), "lv_query")
            n, indexed = self._ctx.n, self._ctx.indexed
            selected = self._ctx.bits_to_ids(bits, 1, n)[0] if n else np.zeros((0,), np.uint32)
            tot = totals.cpu().numpy()
        finally:
            self._release(bits, totals)
        retrieved = np.concatenate([selected[selected < indexed],
                                    np.arange(indexed, n, dtype=np.uint32)]).astype(np.uint32)
        if self.group_index:
            # the reference's statistics (cache.cpp:37-64): the filter's on the grouped index,
            # then the buffer counted as scanned and f_scan over every stored key
            stats = QueryStats()
            if indexed:
                stats = _group_candidates(self, req, algo, want_ids=False).stats
            stats.keys_scanned += n - indexed
            stats.f_scan = (stats.keys_scanned / n) if n else 1.0
        else:
            stats = QueryStats(groups_tested=int(tot[0]), keys_scanned=int(counts[2]),
                               f_scan=(counts[2] / n) if n else 1.0,
                               gate_cost_equiv=2.0 * float(tot[0]) / max(1, self.cfg.r))
        attention = None
        if counts[3]:
            attended = np.ascontiguousarray(selected if strict_threshold else retrieved, dtype=np.uint32)
            weights = np.zeros((max(1, attended.size),), dtype=np.float32)
            if attended.size:
                check(self._ctx.lib.lv_attention_weights(self._ctx.h, 0, _ptr(attended), attended.size, _ptr(q),
                                                         req.effective_scale(), float(part[0]), float(part[1]),
                                                         LV_HOST, _ptr(weights), None), "attention weights")
            attention = AttentionResult(selected_ids=attended, weights=weights[: attended.size], output=out)
        return CacheQueryResult(selected=selected, retrieved=retrieved, stats=stats, attention=attention)

    def index_subspace(self, s: int) -> SubspaceIndex:
        """Subspace s of the grouped index (index.hpp:29-52), copied to the host."""
        if not self.group_index:
            raise ValueError("LouverCache: built without the grouped index")
        n, K = self.indexed_count(), int(self._ctx.lib.lv_group_count(self._ctx.h))
        w = self.d // self.cfg.S + (1 if s < self.d % self.cfg.S else 0)
        asg = np.zeros((max(n, 1),), np.uint32)
        off = np.zeros((K + 1,), np.uint32)
        mem = np.zeros((max(n, 1),), np.uint32)
        a = np.zeros((w, max(K, 1)), np.float32)
        b = np.zeros((w, max(K, 1)), np.float32)
        rad = np.zeros((max(K, 1),), np.float32)
        nb = C.c_double(0.0)
        check(self._ctx.lib.lv_group_export(self._ctx.h, 0, s, _ptr(asg), _ptr(off), _ptr(mem), _ptr(a), _ptr(b),
                                            _ptr(rad), C.byref(nb)), "lv_group_export")
        a, b, rad = a[:, :K].copy(), b[:, :K].copy(), rad[:K].copy()
        aabb = self.cfg.enclosing == "aabb"
        return SubspaceIndex(assignments=asg[:n], member_offsets=off, member_ids=mem[:n],
                             gate_centers=None if aabb else a, gate_radii=None if aabb else rad,
                             gate_lo=a if aabb else None, gate_hi=b if aabb else None, norm_bound=nb.value)

    def _lease(self):
        torch = _torch()
        words = self._ctx.bitmap_words
        with self._pool_lock:
            while self._pool:
                bits, totals = self._pool.pop()
                if bits.shape[1] == words:
                    return bits, totals
        return (torch.empty((1, words), dtype=torch.int32, device="cuda"),
                torch.empty((4,), dtype=torch.int64, device="cuda"))

    def _release(self, bits, totals):
        with self._pool_lock:
            self._pool.append((bits, totals))


def _group_candidates(cache: LouverCache, req: QueryRequest, algo: FilterAlgo, want_ids: bool = True) -> CandidateSet:
    if not cache.group_index:
        raise ValueError("LouverCache: built without the grouped index")
    q = np.ascontiguousarray(req.q, dtype=np.float32).reshape(-1)
    if q.size != cache.d:
        raise ValueError("dot: length mismatch")
    ts = None
    if algo == FilterAlgo.FullSubspace:
        if req.tau_subspace is None:  # cache.cpp:38-41
            ts = derive_subspace_thresholds(cache, q, req.tau)
        else:
            ts = np.ascontiguousarray(req.tau_subspace, dtype=np.float32)
            if ts.size != cache.cfg.S:
                raise ValueError("query_full_subspace: tau_subspace length != S")
    n = cache.indexed_count()
    ids = np.zeros((max(n, 1),), np.uint32) if want_ids else None
    nlive = C.c_int64(0)
    st = _capi.lv_group_stats()
    check(cache._ctx.lib.lv_group_candidates(cache._ctx.h, 0, _ptr(q), float(np.float32(req.tau)),
                                             _ptr(ts), int(algo), None, _ptr(ids), n, C.byref(nlive), C.byref(st),
                                             None), "group candidates")
    stats = QueryStats(groups_tested=int(st.groups_tested), keys_scanned=int(st.keys_scanned), f_scan=st.f_scan,
                       gate_cost_equiv=st.gate_cost_equiv,
                       ta_stop_depth=None if st.ta_stop_depth < 0 else int(st.ta_stop_depth),
                       ta_stop_upper=None if st.ta_stop_depth < 0 else float(st.ta_stop_upper))
    live = ids[: nlive.value].copy() if want_ids else np.zeros((0,), np.uint32)
    return CandidateSet(live_ids=live, stats=stats)


def query_ta(cache: LouverCache, req: QueryRequest) -> CandidateSet:
    """query.hpp:60-63 on the device grouped index (query.cpp:204-303)."""
    return _group_candidates(cache, req, FilterAlgo.Ta)


def query_full_subspace(cache: LouverCache, req: QueryRequest) -> CandidateSet:
    """query.hpp:56-58 on the device grouped index (query.cpp:82-117); tau_subspace required."""
    if req.tau_subspace is None:
        raise ValueError("query_full_subspace: tau_subspace required")
    return _group_candidates(cache, req, FilterAlgo.FullSubspace)


def derive_subspace_thresholds(cache: LouverCache, q, tau: float) -> np.ndarray:
    """query.hpp:65-67 on the device grouped index (query.cpp:305-336)."""
    if not cache.group_index:
        raise ValueError("LouverCache: built without the grouped index")
    q = np.ascontiguousarray(q, dtype=np.float32).reshape(-1)
    out = np.zeros((cache.cfg.S,), np.float32)
    check(cache._ctx.lib.lv_group_thresholds(cache._ctx.h, 0, _ptr(q), float(np.float32(tau)), _ptr(out), None),
          "derive_subspace_thresholds")
    return out


def brute_force_range(cache: LouverCache, q, tau: float, limit: Optional[int] = None) -> np.ndarray:
    """query.hpp:44-45 on the device: ids j < limit with dot(q, k_j) >= tau."""
    torch = _torch()
    n = cache.n()
    limit = n if limit is None else int(limit)
    if limit > n:
        raise ValueError("brute_force_range: limit > n")
    q = np.ascontiguousarray(q, dtype=np.float32).reshape(-1)
    tau_a = np.array([tau], dtype=np.float32)
    bits = torch.zeros((1, cache._ctx.bitmap_words), dtype=torch.int32, device="cuda")
    if limit == 0:
        return np.zeros((0,), np.uint32)
    check(cache._ctx.lib.lv_brute_force_range(cache._ctx.h, _ptr(q), _ptr(tau_a), limit, LV_HOST,
                                              bits.data_ptr(), None), "lv_brute_force_range")
    return cache._ctx.bits_to_ids(bits, 1, limit)[0]


def sparse_attention(cache: LouverCache, buffer_ids: Sequence[int], selected_ids: Sequence[int], q,
                     scale: float) -> Optional[AttentionResult]:
    """query.hpp:69-72: softmax over sort∪unique(selected ∪ buffer); None when empty."""
    q = np.ascontiguousarray(q, dtype=np.float32).reshape(-1)
    buf = np.ascontiguousarray(buffer_ids, dtype=np.uint32).reshape(-1)
    sel = np.ascontiguousarray(selected_ids, dtype=np.uint32).reshape(-1)
    tokens = np.unique(np.concatenate([sel, buf]))
    out = np.zeros((cache.d,), dtype=np.float32)
    weights = np.zeros((max(1, tokens.size),), dtype=np.float32)
    ntok = C.c_int64(0)
    rc = check(cache._ctx.lib.lv_sparse_attention(
        cache._ctx.h, 0, _ptr(buf) if buf.size else None, buf.size, _ptr(sel) if sel.size else None,
        sel.size, _ptr(q), float(scale), LV_HOST, _ptr(out), _ptr(weights), C.byref(ntok), None),
        "sparse_attention")
    if rc == LV_EMPTY:
        return None
    return AttentionResult(selected_ids=tokens, weights=weights[: ntok.value], output=out)


class LouverLayer:
    """One decode layer's KV cache for ``batch`` sequences x ``n_kv_heads`` kv heads
    with ``group_size`` q heads per kv head, resident in HBM, plus its index.

    Device-side API (torch tensors on cuda): ``build`` (prefill),
    ``push_key`` (one decode step's key/value per slot), ``query_device`` (the
    hot path: one launch, writes attention outputs), ``dense_decode`` (the
    full-scan baseline). Host-buffer API: ``query_host`` (copies inside).
    """

    def __init__(self, d: int, n_kv_heads: int, group_size: int, batch: int, capacity: int,
                 cfg: Optional[BuildConfig] = None, buffer_capacity: int = 128,
                 dtype: str = "bf16", group_index: bool = False):
        cfg = cfg or BuildConfig(S=1, r=16, grouping="contiguous", enclosing="aabb")
        cfg.validate(d)
        self.d, self.H_kv, self.G, self.batch = d, n_kv_heads, group_size, batch
        self.H_q = n_kv_heads * group_size
        self.rows = batch * self.H_q
        self.dtype = LV_BF16 if dtype == "bf16" else LV_F32
        self.cfg = cfg
        self.group_index = bool(group_index)
        self._ctx = _Context(_config(d, n_kv_heads, group_size, batch, self.dtype, cfg,
                                     buffer_capacity, capacity, self.group_index))

    @property
    def n(self) -> int:
        return self._ctx.n

    @property
    def indexed_count(self) -> int:
        return self._ctx.indexed

    @property
    def flush_count(self) -> int:
        return self._ctx.flushes

    @property
    def bitmap_words(self) -> int:
        return self._ctx.bitmap_words

    def workspace_bytes(self) -> int:
        return int(self._ctx.lib.lv_query_workspace_bytes(self._ctx.h))

    def geometry(self) -> dict:
        g = np.zeros((8,), np.int64)
        check(self._ctx.lib.lv_geometry(self._ctx.h, g.ctypes.data), "lv_geometry")
        keys = ("dp", "cell_keys", "arena_rows", "cells", "splits", "chunks_per_split", "chunk_keys",
                "smem_bytes")
        out = {k: int(v) for k, v in zip(keys, g)}
        if self.dtype == LV_BF16 or self.d > 64:  # the fused layer kernel's launch geometry (after a query)
            lg = np.zeros((4,), np.int64)
            check(self._ctx.lib.lv_layer_geometry(self._ctx.h, lg.ctypes.data), "lv_layer_geometry")
            out.update(zip(("team_ctas_per_slot", "ctas_per_sm", "threads_per_cta", "layer_smem_bytes"),
                           (int(v) for v in lg)))
        return out

    def build(self, K, V, stream=None) -> None:
        """K, V: [batch][H_kv][n][d] fp32 or bf16 (numpy host or torch cuda)."""
        torch = _torch()
        if isinstance(K, np.ndarray):
            K = np.ascontiguousarray(K, dtype=np.float32)
            V = np.ascontiguousarray(V, dtype=np.float32)
            n = K.shape[2]
            check(self._ctx.lib.lv_build(self._ctx.h, _ptr(K), _ptr(V), n, LV_F32, LV_HOST, stream),
                  "lv_build")
            return
        src = LV_BF16 if K.dtype == torch.bfloat16 else LV_F32
        K = K.contiguous()
        V = V.contiguous()
        st = stream if stream is not None else torch.cuda.current_stream().cuda_stream
        check(self._ctx.lib.lv_build(self._ctx.h, K.data_ptr(), V.data_ptr(), K.shape[2], src,
                                     LV_DEVICE, st), "lv_build")

    def push_key(self, k, v, stream=None) -> None:
        torch = _torch()
        if isinstance(k, np.ndarray):
            k = np.ascontiguousarray(k, dtype=np.float32)
            v = np.ascontiguousarray(v, dtype=np.float32)
            check(self._ctx.lib.lv_push_key(self._ctx.h, _ptr(k), _ptr(v), LV_F32, LV_HOST, None),
                  "lv_push_key")
            return
        src = LV_BF16 if k.dtype == torch.bfloat16 else LV_F32
        st = stream if stream is not None else torch.cuda.current_stream().cuda_stream
        check(self._ctx.lib.lv_push_key(self._ctx.h, k.data_ptr(), v.data_ptr(), src, LV_DEVICE, st),
              "lv_push_key")

    def flush_buffer(self) -> bool:
        return check(self._ctx.lib.lv_flush(self._ctx.h, None), "lv_flush") == _capi.LV_OK

    def sync_counters(self) -> None:
        check(self._ctx.lib.lv_sync_counters(self._ctx.h, None), "lv_sync_counters")

    def query_device(self, q, tau, out, *, scale: float = 0.0, strict: bool = False, partial=None,
                     counts=None, sel_bits=None, totals=None, workspace=None, stream=None) -> None:
        """Hot path. q [batch][H_q][d] fp32, tau [batch][H_q] fp32, out [batch][H_q][d] fp32,
        all cuda tensors; enqueue-only on ``stream`` (default: torch's current stream)."""
        torch = _torch()
        st = stream if stream is not None else torch.cuda.current_stream().cuda_stream
        args = _capi.lv_query_args(
            q=q.data_ptr(), tau=tau.data_ptr(), scale=float(scale), algo=1, strict=1 if strict else 0,
            where=LV_DEVICE, out=_ptr(out), partial=_ptr(partial), counts=_ptr(counts),
            sel_bits=_ptr(sel_bits), totals=_ptr(totals), workspace=_ptr(workspace), stream=st)
        check(self._ctx.lib.lv_query(self._ctx.h, C.byref(args)), "lv_query")

    def query_host(self, q: np.ndarray, tau: np.ndarray, *, scale: float = 0.0,
                   strict: bool = False, want_counts: bool = False, out: np.ndarray | None = None):
        """Host buffers in and out (copies inside the call): returns out[, counts].
        ``out`` may be a caller-owned (ideally pinned) float32 [batch][H_q][d] buffer."""
        q = np.ascontiguousarray(q, dtype=np.float32)
        tau = np.ascontiguousarray(tau, dtype=np.float32)
        if out is None:
            out = np.zeros((self.batch, self.H_q, self.d), dtype=np.float32)
        elif out.dtype != np.float32 or not out.flags.c_contiguous or out.size != self.batch * self.H_q * self.d:
            raise ValueError("query_host: out must be a C-contiguous float32 [batch][H_q][d] array")
        counts = np.zeros((self.batch, self.H_q, 4), dtype=np.int32) if want_counts else None
        args = _capi.lv_query_args(
            q=_ptr(q), tau=_ptr(tau), scale=float(scale), algo=1, strict=1 if strict else 0,
            where=LV_HOST, out=_ptr(out), partial=None, counts=_ptr(counts), sel_bits=None,
            totals=None, workspace=None, stream=None)
        check(self._ctx.lib.lv_query(self._ctx.h, C.byref(args)), "lv_query")
        return (out, counts) if want_counts else out

    def dense_decode(self, q, out, *, scale: float = 0.0, partial=None, stream=None) -> None:
        torch = _torch()
        st = stream if stream is not None else torch.cuda.current_stream().cuda_stream
        check(self._ctx.lib.lv_dense_decode(self._ctx.h, q.data_ptr(), float(scale), LV_DEVICE,
                                            out.data_ptr(), _ptr(partial), st), "lv_dense_decode")

    def brute_force_bits(self, q, tau, limit: Optional[int] = None, stream=None):
        torch = _torch()
        limit = self.n if limit is None else limit
        bits = torch.zeros((self.rows, self.bitmap_words), dtype=torch.int32, device="cuda")
        st = stream if stream is not None else torch.cuda.current_stream().cuda_stream
        check(self._ctx.lib.lv_brute_force_range(self._ctx.h, q.data_ptr(), tau.data_ptr(), limit,
                                                 LV_DEVICE, bits.data_ptr(), st), "lv_brute_force_range")
        return bits

    def ids_from_bits(self, bits, limit: Optional[int] = None) -> List[np.ndarray]:
        return self._ctx.bits_to_ids(bits, self.rows, self.n if limit is None else limit)

    def read_rows(self, slot: int, first: int, count: int, values: bool = False) -> np.ndarray:
        out = np.empty((count, self.d), dtype=np.float32)
        check(self._ctx.lib.lv_read_rows(self._ctx.h, slot, first, count, 1 if values else 0, _ptr(out)),
              "lv_read_rows")
        return out


def _layers_host_args(layers, q, tau, out, scale, strict, stream):
    L = len(layers)
    for a, shape in ((q, (L, layers[0].batch, layers[0].H_q, layers[0].d)), (tau, (L, layers[0].batch, layers[0].H_q)),
                     (out, (L, layers[0].batch, layers[0].H_q, layers[0].d))):
        if a.dtype != np.float32 or not a.flags.c_contiguous or a.shape != shape:
            raise ValueError(f"query_layers_host: expected C-contiguous float32 {shape}")
    hs = (C.c_void_p * L)(*[ly._ctx.h for ly in layers])
    return hs, (hs, L, _ptr(q), _ptr(tau), float(scale), 1 if strict else 0, _ptr(out), None, stream)


def query_layers_host(layers: Sequence["LouverLayer"], q: np.ndarray, tau: np.ndarray, out: np.ndarray, *,
                      scale: float = 0.0, strict: bool = False, stream=None) -> np.ndarray:
    """One decode step over L layers through the C ABI with HOST buffers (lv_query_layers):
    q [L][batch][H_q][d], tau [L][batch][H_q], out [L][batch][H_q][d] float32, C-contiguous
    (pinned for full speed). Inputs go in per layer, L fused queries, outputs come back per
    layer, one sync (see LayersStep for the repeated call)."""
    _, args = _layers_host_args(layers, q, tau, out, scale, strict, stream)
    check(_capi.lib().lv_query_layers(*args), "lv_query_layers")
    return out


class LayersStep:
    """query_layers_host prepared once for fixed buffers: the arguments are validated and
    marshalled here, so each call is the one C call a C++ caller makes per decode step. The
    caller rewrites q and tau in place between calls and reads out after each."""

    def __init__(self, layers: Sequence["LouverLayer"], q: np.ndarray, tau: np.ndarray, out: np.ndarray, *,
                 scale: float = 0.0, strict: bool = False, stream=None):
        hs, self._args = _layers_host_args(layers, q, tau, out, scale, strict, stream)
        self._keep = (list(layers), q, tau, out, hs)
        self._fn = _capi.lib().lv_query_layers

    def __call__(self) -> np.ndarray:
        rc = self._fn(*self._args)
        if rc:
            check(rc, "lv_query_layers")
        return self._keep[3]


def lse_merge(partials, out, stream=None) -> None:
    """Merge sequence-shard partials [P][rows][d+2] -> out [rows][d] (cuda tensors)."""
    torch = _torch()
    P, rows, w = partials.shape
    st = stream if stream is not None else torch.cuda.current_stream().cuda_stream
    check(_capi.lib().lv_lse_merge(partials.data_ptr(), P, rows, w - 2, out.data_ptr(), st),
          "lv_lse_merge")
