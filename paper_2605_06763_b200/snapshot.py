"""Snapshots: the reference's ``louver/io.hpp`` file formats (io.hpp:40-51, io.cpp:205-317).

``save_dataset`` / ``load_dataset``: the "LVKD" row-major f32 matrix container.
``save_index`` writes a cache's device index as a reference "LVIX" snapshot (one
subspace, contiguous groups = the device cells, exact fp32 AABBs, the member lists);
``load_index`` reads any reference LVIX file (every grouping, enclosure and S),
validates it against the cache and adopts its ``indexed_count`` — the cell summaries
already cover every stored key, so no re-indexing happens on restart. Errors follow
the reference: std::runtime_error (bad magic, truncation, trailing bytes, version) →
``LouverError`` (a RuntimeError); argument errors → ValueError.
"""
from __future__ import annotations

import ctypes as C
import os

import numpy as np

from . import _capi
from ._capi import check


def _path(p) -> bytes:
    return os.fsencode(os.fspath(p))


def save_dataset(path, data) -> None:
    """io.cpp:208-217."""
    data = np.ascontiguousarray(data, dtype=np.float32)
    if data.ndim != 2:
        raise ValueError("save_dataset: a [n][d] matrix is required")
    check(_capi.lib().lv_save_dataset(_path(path), data.ctypes.data, data.shape[0], data.shape[1]), "save_dataset")


def load_dataset(path) -> np.ndarray:
    """io.cpp:219-234."""
    lib = _capi.lib()
    n, d = C.c_int64(), C.c_int()
    check(lib.lv_load_dataset(_path(path), None, 0, C.byref(n), C.byref(d)), "load_dataset")
    out = np.empty((n.value, d.value), np.float32)
    check(lib.lv_load_dataset(_path(path), out.ctypes.data if out.size else None, n.value, C.byref(n),
                              C.byref(d)), "load_dataset")
    return out


def save_index(cache, path, slot: int = 0) -> None:
    """io.cpp:236-268 for the device index of ``cache`` (a LouverCache or LouverLayer)."""
    ctx = cache._ctx
    check(ctx.lib.lv_save_index(ctx.h, int(slot), _path(path)), "save_index")


def load_index(cache, path) -> int:
    """io.cpp:270-317: validates the snapshot against ``cache`` and adopts its
    indexed_count; returns it."""
    ctx = cache._ctx
    m = C.c_int64()
    check(ctx.lib.lv_load_index(ctx.h, _path(path), C.byref(m), None), "load_index")
    return int(m.value)


__all__ = ["save_dataset", "load_dataset", "save_index", "load_index"]
