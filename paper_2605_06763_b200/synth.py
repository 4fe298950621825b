"""Synthetic decode-trace streams with the reference data laws (io.cpp:89-206).

Thin numpy wrappers over liblouver_synth.so (std::mt19937_64 +
std::normal_distribution<double>, so libstdc++ reproduces the reference's
bytes). ``keys(n, d, seed)`` is ``gen_synthetic(n, d, gaussian, seed)``;
``queries(nq, d, seed)`` is ``gen_synthetic_queries(nq, d, gaussian, seed)``.
"""
from __future__ import annotations

import numpy as np

from . import _capi


def keys(n: int, d: int, seed: int) -> np.ndarray:
    out = np.empty((n, d), dtype=np.float32)
    _capi.check(_capi.synth_lib().lv_synth_keys(n, d, seed, out.ctypes.data), "lv_synth_keys")
    return out


def queries(nq: int, d: int, seed: int) -> np.ndarray:
    out = np.empty((nq, d), dtype=np.float32)
    _capi.check(_capi.synth_lib().lv_synth_queries(nq, d, seed, out.ctypes.data), "lv_synth_queries")
    return out


def mixture(n: int, d: int, seed: int, k: int = 8, spread: float = 0.25, queries: bool = False) -> np.ndarray:
    out = np.empty((n, d), dtype=np.float32)
    _capi.check(_capi.synth_lib().lv_synth_mixture(n, d, k, spread, seed, 1 if queries else 0,
                                                   out.ctypes.data), "lv_synth_mixture")
    return out


def keys_multi(n: int, d: int, seeds, threads: int = 0) -> np.ndarray:
    """One independent key stream per seed, generated in parallel: [len(seeds)][n][d]."""
    seeds = np.ascontiguousarray(seeds, dtype=np.uint64)
    out = np.empty((seeds.size, n, d), dtype=np.float32)
    _capi.check(_capi.synth_lib().lv_synth_keys_multi(n, d, seeds.ctypes.data, seeds.size,
                                                      out.ctypes.data, threads), "lv_synth_keys_multi")
    return out


def iid_normal(n: int, d: int, seed: int) -> np.ndarray:
    """The unit tests' iid N(0,1) query law (test_util.hpp:18-24) — numpy RNG, not bit-identical."""
    return np.random.default_rng(seed).standard_normal((n, d)).astype(np.float32)
