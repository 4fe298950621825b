"""TEST INFRASTRUCTURE — ctypes binding of the CPU oracle (liblouver_oracle.so).

Only tests/, __graft_entry__.smoke() and bench.py's CPU legs import this
module. It restates the reference library (see louver_oracle.h); nothing in
the product package imports it.
"""
from __future__ import annotations

import ctypes as C
import os
import subprocess
from typing import Optional

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
_LIB_PATH = os.path.join(_HERE, "liblouver_oracle.so")

GROUPING = {"contiguous": 0, "interleaved": 1, "random": 2, "pca_tree": 3}
ENCLOSURE = {"ball": 0, "aabb": 1, "span_ball": 2}


class lvo_build_config(C.Structure):
    _fields_ = [("S", C.c_int), ("r", C.c_int), ("grouping", C.c_int), ("enclosure", C.c_int),
                ("rng_seed", C.c_uint64)]


class lvo_stats(C.Structure):
    _fields_ = [("groups_tested", C.c_int64), ("keys_scanned", C.c_int64), ("f_scan", C.c_double),
                ("gate_cost_equiv", C.c_double), ("ta_stop_depth", C.c_int),
                ("ta_stop_upper", C.c_double)]


_P = C.c_void_p
_I64P = C.POINTER(C.c_int64)
_SIGS = {
    "lvo_last_error": (C.c_char_p, []),
    "lvo_dot": (C.c_float, [_P, _P, C.c_int64]),
    "lvo_brute_force_range": (C.c_int, [_P, C.c_int64, C.c_int, _P, C.c_float, C.c_int64, _P, C.c_int64, _I64P]),
    "lvo_exact_check": (C.c_int, [_P, C.c_int64, C.c_int, _P, C.c_int64, _P, C.c_float, _P, _I64P]),
    "lvo_layout": (C.c_int, [C.c_int, C.c_int, _P]),
    "lvo_scores": (C.c_int, [_P, C.c_int64, C.c_int, _P, _P]),
    "lvo_kth_score": (C.c_float, [_P, C.c_int64, C.c_int, _P, C.c_int64]),
    "lvo_reservoir_create": (_P, [C.c_int64, C.c_uint64]),
    "lvo_reservoir_destroy": (None, [_P]),
    "lvo_reservoir_update": (C.c_int64, [_P, C.c_uint32]),
    "lvo_reservoir_size": (C.c_int64, [_P]),
    "lvo_reservoir_seen": (C.c_int64, [_P]),
    "lvo_reservoir_ids": (None, [_P, _P]),
    "lvo_estimate_tau": (C.c_int, [_P, C.c_int64, C.c_int, _P, C.c_int, C.c_int, C.c_double, _P]),
    "lvo_sparse_attention": (C.c_int, [_P, _P, C.c_int64, C.c_int, _P, C.c_int64, _P, C.c_int64, _P,
                                       C.c_float, _P, _P, _I64P]),
    "lvo_cache_create": (C.c_int, [C.c_int, C.POINTER(lvo_build_config), C.c_int64, C.POINTER(_P)]),
    "lvo_cache_adopt": (C.c_int, [_P, _P, C.c_int64, C.c_int, C.POINTER(lvo_build_config), C.c_int64,
                                  C.POINTER(_P)]),
    "lvo_cache_destroy": (None, [_P]),
    "lvo_cache_push_key": (C.c_int, [_P, _P, _P]),
    "lvo_cache_flush": (C.c_int, [_P]),
    "lvo_cache_n": (C.c_int64, [_P]),
    "lvo_cache_indexed_count": (C.c_int64, [_P]),
    "lvo_cache_flush_count": (C.c_int64, [_P]),
    "lvo_cache_groups": (C.c_int64, [_P, C.c_int]),
    "lvo_cache_group_members": (C.c_int64, [_P, C.c_int, C.c_int64, _P, C.c_int64]),
    "lvo_cache_query": (C.c_int, [_P, _P, C.c_float, C.c_float, C.c_int, C.c_int, _P, _I64P, _P, _I64P,
                                  C.c_int64, _P, C.POINTER(C.c_int), C.POINTER(lvo_stats)]),
    "lvo_cache_candidates": (C.c_int, [_P, _P, C.c_float, _P, C.c_int, _P, C.c_int64, _I64P,
                                       C.POINTER(lvo_stats)]),
    "lvo_cache_thresholds": (C.c_int, [_P, _P, C.c_float, _P]),
    "lvo_cache_subspace": (C.c_int, [_P, C.c_int, _P, _P, _P, _P, _P, _P, C.POINTER(C.c_double)]),
    "lvo_balanced_pca_tree": (C.c_int, [_P, C.c_int64, C.c_int, C.c_int, _P]),
    "lvo_assign_groups": (C.c_int, [_P, C.c_int64, C.c_int, C.POINTER(lvo_build_config), C.c_int,
                                    C.c_uint32, _P]),
    "lvo_enclose_group": (C.c_int, [_P, C.c_int64, C.c_int, C.c_int, _P, _P, _P, _P]),
}

_lib = None


def reference_module():
    """This module's API bound to oracle/_ref/liblouver_ref.so — the reference sources
    themselves (/root/reference/proj/src/*.cpp, unmodified) compiled against the Eigen shim
    in oracle/ref (``make -C oracle ref``) — or None when that build is absent."""
    import importlib.util

    path = os.path.join(_HERE, "_ref", "liblouver_ref.so")
    if not os.path.exists(path):
        return None
    spec = importlib.util.spec_from_file_location("oracle._pyoracle_reference", os.path.abspath(__file__))
    mod = importlib.util.module_from_spec(spec)
    spec.loader.exec_module(mod)
    mod._LIB_PATH = path
    mod.IS_REFERENCE = True
    return mod


IS_REFERENCE = False


def build() -> None:
    subprocess.run(["make", "-s", "-C", _HERE], check=True)


def lib() -> C.CDLL:
    global _lib
    if _lib is None:
        if not os.path.exists(_LIB_PATH):
            build()
        L = C.CDLL(_LIB_PATH)
        for name, (res, args) in _SIGS.items():
            fn = getattr(L, name)
            fn.restype = res
            fn.argtypes = args
        _lib = L
    return _lib


def _f32(a) -> np.ndarray:
    return np.ascontiguousarray(a, dtype=np.float32)


def _u32(a) -> np.ndarray:
    return np.ascontiguousarray(a, dtype=np.uint32).reshape(-1)


def _check(rc: int) -> int:
    if rc < 0:
        msg = (lib().lvo_last_error() or b"").decode()
        if rc == -2:
            raise IndexError(msg)
        raise ValueError(msg)
    return rc


def cfg(S=4, r=4, grouping="pca_tree", enclosure="ball", seed=0) -> lvo_build_config:
    g = GROUPING[grouping] if isinstance(grouping, str) else grouping
    e = ENCLOSURE[enclosure] if isinstance(enclosure, str) else enclosure
    return lvo_build_config(S, r, g, e, seed)


def dot(a, b) -> np.float32:
    a, b = _f32(a), _f32(b)
    if a.size != b.size:
        raise ValueError("dot: length mismatch")
    return np.float32(lib().lvo_dot(a.ctypes.data, b.ctypes.data, a.size))


def brute_force_range(keys, q, tau, limit: Optional[int] = None) -> np.ndarray:
    keys, q = _f32(keys), _f32(q)
    n, d = keys.shape
    limit = n if limit is None else limit
    out = np.empty((max(1, limit),), np.uint32)
    cnt = C.c_int64()
    _check(lib().lvo_brute_force_range(keys.ctypes.data, n, d, q.ctypes.data, float(tau), limit,
                                       out.ctypes.data, out.size, C.byref(cnt)))
    return out[: cnt.value].copy()


def exact_check(keys, cand, q, tau) -> np.ndarray:
    keys, q, cand = _f32(keys), _f32(q), _u32(cand)
    n, d = keys.shape
    out = np.empty((max(1, cand.size),), np.uint32)
    cnt = C.c_int64()
    _check(lib().lvo_exact_check(keys.ctypes.data, n, d, cand.ctypes.data if cand.size else None,
                                 cand.size, q.ctypes.data, float(tau), out.ctypes.data, C.byref(cnt)))
    return out[: cnt.value].copy()


def layout(d: int, S: int) -> np.ndarray:
    off = np.zeros((S + 1,), np.int32)
    _check(lib().lvo_layout(d, S, off.ctypes.data))
    return off


def scores(keys, q) -> np.ndarray:
    keys, q = _f32(keys), _f32(q)
    n, d = keys.shape
    out = np.empty((n,), np.float32)
    lib().lvo_scores(keys.ctypes.data, n, d, q.ctypes.data, out.ctypes.data)
    return out


def kth_score(keys, q, k: int) -> np.float32:
    keys, q = _f32(keys), _f32(q)
    n, d = keys.shape
    return np.float32(lib().lvo_kth_score(keys.ctypes.data, n, d, q.ctypes.data, k))


class Reservoir:
    """threshold.hpp:29-50 over ids (the oracle's restatement; test-only)."""

    def __init__(self, capacity: int = 256, seed: int = 0):
        if capacity < 1:
            raise ValueError("Reservoir: capacity >= 1 required")
        self._h = lib().lvo_reservoir_create(capacity, seed)

    def __del__(self):
        if getattr(self, "_h", None):
            lib().lvo_reservoir_destroy(self._h)
            self._h = None

    def update(self, key_id: int) -> int:
        return int(lib().lvo_reservoir_update(self._h, key_id))

    def size(self) -> int:
        return int(lib().lvo_reservoir_size(self._h))

    def seen(self) -> int:
        return int(lib().lvo_reservoir_seen(self._h))

    def ids(self) -> np.ndarray:
        out = np.empty((self.size(),), np.uint32)
        lib().lvo_reservoir_ids(self._h, out.ctypes.data)
        return out


def estimate_tau(sample_keys, q, variant: int, m: int = 2, alpha: float = 0.1) -> np.float32:
    """threshold.cpp:63-103 over the sampled keys [n][d]; variant as OracleVariant."""
    keys, q = _f32(sample_keys), _f32(q)
    n, d = keys.shape if keys.ndim == 2 else (0, q.shape[0])
    out = np.zeros((1,), np.float32)
    _check(lib().lvo_estimate_tau(keys.ctypes.data if n else None, n, d, q.ctypes.data, variant, m, alpha,
                                  out.ctypes.data))
    return out[0]


def sparse_attention(keys, values, buffer_ids, selected_ids, q, scale):
    """Returns (tokens, weights, output) or None when the token set is empty."""
    keys, values, q = _f32(keys), _f32(values), _f32(q)
    buf, sel = _u32(buffer_ids), _u32(selected_ids)
    n, d = keys.shape
    tokens = np.unique(np.concatenate([sel, buf]))
    out = np.zeros((d,), np.float32)
    w = np.zeros((max(1, tokens.size),), np.float32)
    nt = C.c_int64()
    rc = _check(lib().lvo_sparse_attention(
        keys.ctypes.data, values.ctypes.data, n, d, buf.ctypes.data if buf.size else None, buf.size,
        sel.ctypes.data if sel.size else None, sel.size, q.ctypes.data, float(scale), out.ctypes.data,
        w.ctypes.data, C.byref(nt)))
    if rc == 1:
        return None
    return tokens, w[: nt.value].copy(), out


def balanced_pca_tree(points, r: int) -> np.ndarray:
    points = _f32(points)
    m, w = points.shape
    out = np.zeros((m,), np.uint32)
    _check(lib().lvo_balanced_pca_tree(points.ctypes.data if m else None, m, w, r, out.ctypes.data))
    return out


def assign_groups(points, config: lvo_build_config, subspace: int = 0, base_id: int = 0) -> np.ndarray:
    points = _f32(points)
    m, w = points.shape
    out = np.zeros((m,), np.uint32)
    _check(lib().lvo_assign_groups(points.ctypes.data, m, w, C.byref(config), subspace, base_id,
                                   out.ctypes.data))
    return out


def enclose_group(points, kind: str):
    points = _f32(points)
    m, w = points.shape
    k = ENCLOSURE[kind]
    center = np.zeros((w,), np.float32)
    lo = np.zeros((w,), np.float32)
    hi = np.zeros((w,), np.float32)
    rad = C.c_float()
    _check(lib().lvo_enclose_group(points.ctypes.data if m else None, m, w, k, center.ctypes.data,
                                   C.byref(rad), lo.ctypes.data, hi.ctypes.data))
    if k == 1:
        return lo, hi
    return center, np.float32(rad.value)


class Cache:
    """Oracle LouverCache (cache.hpp:21-63)."""

    def __init__(self, d: int, config: lvo_build_config, B: int, keys=None, values=None):
        self.d = d
        h = C.c_void_p()
        if keys is None:
            _check(lib().lvo_cache_create(d, C.byref(config), B, C.byref(h)))
        else:
            k, v = _f32(keys), _f32(values)
            _check(lib().lvo_cache_adopt(k.ctypes.data, v.ctypes.data, k.shape[0], d, C.byref(config),
                                         B, C.byref(h)))
        self.h = h

    def __del__(self):
        if getattr(self, "h", None):
            lib().lvo_cache_destroy(self.h)
            self.h = None

    def push_key(self, k, v) -> None:
        k, v = _f32(k).reshape(-1), _f32(v).reshape(-1)
        _check(lib().lvo_cache_push_key(self.h, k.ctypes.data, v.ctypes.data))

    def flush_buffer(self) -> bool:
        return _check(lib().lvo_cache_flush(self.h)) == 0

    def n(self) -> int:
        return int(lib().lvo_cache_n(self.h))

    def indexed_count(self) -> int:
        return int(lib().lvo_cache_indexed_count(self.h))

    def pending_count(self) -> int:
        return self.n() - self.indexed_count()

    def flush_count(self) -> int:
        return int(lib().lvo_cache_flush_count(self.h))

    def groups(self, s: int) -> int:
        return int(lib().lvo_cache_groups(self.h, s))

    def group_members(self, s: int, g: int) -> np.ndarray:
        out = np.zeros((4096,), np.uint32)
        cnt = lib().lvo_cache_group_members(self.h, s, g, out.ctypes.data, out.size)
        return out[:cnt].copy()

    def candidates(self, q, tau, algo: int = 1, tau_s=None):
        """query_full_subspace (algo 0, tau_s required) / query_ta (algo 1) on the cache's
        index: (live ids, stats dict)."""
        q = _f32(q).reshape(-1)
        n = max(1, self.indexed_count())
        ids = np.empty((n,), np.uint32)
        cnt = C.c_int64()
        st = lvo_stats()
        ts = None if tau_s is None else _f32(tau_s)
        _check(lib().lvo_cache_candidates(self.h, q.ctypes.data, float(np.float32(tau)),
                                          None if ts is None else ts.ctypes.data, algo, ids.ctypes.data, n,
                                          C.byref(cnt), C.byref(st)))
        stats = dict(groups_tested=st.groups_tested, keys_scanned=st.keys_scanned, f_scan=st.f_scan,
                     gate_cost_equiv=st.gate_cost_equiv, ta_stop_depth=st.ta_stop_depth,
                     ta_stop_upper=st.ta_stop_upper)
        return ids[: cnt.value].copy(), stats

    def thresholds(self, q, tau, S: int) -> np.ndarray:
        q = _f32(q).reshape(-1)
        out = np.zeros((S,), np.float32)
        _check(lib().lvo_cache_thresholds(self.h, q.ctypes.data, float(np.float32(tau)), out.ctypes.data))
        return out

    def subspace(self, s: int, w: int, enclosure: str):
        """(assignments, member offsets, member ids, a [w][K], b [w][K] | None, radii | None, norm_bound)"""
        n, K = self.indexed_count(), self.groups(s)
        asg = np.zeros((max(n, 1),), np.uint32)
        off = np.zeros((K + 1,), np.uint32)
        mem = np.zeros((max(n, 1),), np.uint32)
        a = np.zeros((w, max(K, 1)), np.float32)
        b = np.zeros((w, max(K, 1)), np.float32)
        rad = np.zeros((max(K, 1),), np.float32)
        nb = C.c_double()
        _check(lib().lvo_cache_subspace(self.h, s, asg.ctypes.data, off.ctypes.data, mem.ctypes.data,
                                        a.ctypes.data, b.ctypes.data, rad.ctypes.data, C.byref(nb)))
        box = enclosure == "aabb"
        return (asg[:n], off, mem[:n], a[:, :K].copy(), b[:, :K].copy() if box else None,
                None if box else rad[:K].copy(), nb.value)

    def query(self, q, tau, algo: int = 1, strict: bool = False, scale: float = 0.0):
        """Returns dict(selected, retrieved, output|None, stats)."""
        q = _f32(q).reshape(-1)
        n = self.n()
        sel = np.empty((max(1, n),), np.uint32)
        ret = np.empty((max(1, n),), np.uint32)
        ns, nr = C.c_int64(), C.c_int64()
        out = np.zeros((self.d,), np.float32)
        has = C.c_int()
        st = lvo_stats()
        _check(lib().lvo_cache_query(self.h, q.ctypes.data, float(tau), float(scale), algo,
                                     1 if strict else 0, sel.ctypes.data, C.byref(ns), ret.ctypes.data,
                                     C.byref(nr), sel.size, out.ctypes.data, C.byref(has), C.byref(st)))
        return {
            "selected": sel[: ns.value].copy(),
            "retrieved": ret[: nr.value].copy(),
            "output": out if has.value else None,
            "stats": {
                "groups_tested": st.groups_tested, "keys_scanned": st.keys_scanned, "f_scan": st.f_scan,
                "gate_cost_equiv": st.gate_cost_equiv,
                "ta_stop_depth": None if st.ta_stop_depth < 0 else st.ta_stop_depth,
                "ta_stop_upper": st.ta_stop_upper,
            },
        }
