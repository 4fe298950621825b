"""Threshold oracle: the reference's ``louver/threshold.hpp`` interface on the device.

Mirrors proj/include/louver/threshold.hpp:9-53 and proj/src/threshold.cpp:
``OracleVariant``, ``OracleConfig`` (with ``validate``), ``parse_oracle``,
``to_string``, ``Reservoir`` (Algorithm R, the reference's mt19937_64 draws, in
the C library) and ``estimate_tau``. The reservoir samples arena row ids of one
cache (rows are append-only, so an id names the same key forever); the
estimate gathers those rows on the device and runs the normative dot, the sort
and the variant's pick there (csrc/louver_threshold.cuh), so an adaptive τ
never leaves HBM in a decode loop. ``LouverLayer``-wide estimates for every q
head at once: :func:`estimate_tau_layer`.
"""
from __future__ import annotations

import ctypes as C
import dataclasses
import enum
import numpy as np

from . import _capi
from ._capi import LV_DEVICE, LV_HOST, check


class OracleVariant(enum.IntEnum):
    """threshold.hpp:9 (same order as LV_TAU_*)."""

    SampleMax = 0
    SampleTopK = 1
    SampleGap = 2
    SampleMeanMax = 3
    Budget = 4


@dataclasses.dataclass
class OracleConfig:
    """threshold.hpp:11-23."""

    variant: OracleVariant = OracleVariant.SampleMax
    m: int = 2
    alpha: float = 0.1

    def validate(self) -> None:
        if self.variant == OracleVariant.SampleTopK and self.m < 1:
            raise ValueError("OracleConfig: m >= 1 required")
        if self.variant == OracleVariant.Budget and not (0.0 < self.alpha < 1.0):
            raise ValueError("OracleConfig: 0 < alpha < 1 required")


def parse_oracle(text: str) -> OracleConfig:
    """threshold.cpp:8-27: "max", "topk:m", "gap", "meanmax", "budget:alpha"."""
    cfg = OracleConfig()
    if text == "max":
        cfg.variant = OracleVariant.SampleMax
    elif text == "gap":
        cfg.variant = OracleVariant.SampleGap
    elif text == "meanmax":
        cfg.variant = OracleVariant.SampleMeanMax
    elif text.startswith("topk:"):
        cfg.variant = OracleVariant.SampleTopK
        cfg.m = int(text[5:])
    elif text.startswith("budget:"):
        cfg.variant = OracleVariant.Budget
        cfg.alpha = float(text[7:])
    else:
        raise ValueError("unknown oracle variant: " + text)
    cfg.validate()
    return cfg


def to_string(cfg: OracleConfig) -> str:
    """threshold.cpp:29-38 (std::to_string(double) prints six decimals)."""
    v = cfg.variant
    if v == OracleVariant.SampleMax:
        return "max"
    if v == OracleVariant.SampleGap:
        return "gap"
    if v == OracleVariant.SampleMeanMax:
        return "meanmax"
    if v == OracleVariant.SampleTopK:
        return f"topk:{cfg.m}"
    return f"budget:{cfg.alpha:.6f}"


class Reservoir:
    """threshold.hpp:29-50: fixed-capacity uniform sample of a key stream.

    ``update(id, key=None)`` follows Reservoir::update (threshold.cpp:40-55); the
    key argument is accepted for signature parity, the sample keeps the id (the
    key is the arena row ``id`` of the cache the reservoir samples).
    """

    def __init__(self, capacity: int = 256, seed: int = 0, cache=None):
        lib = _capi.lib()
        h = C.c_void_p()
        check(lib.lv_reservoir_create(int(capacity), int(seed) & (2**64 - 1), C.byref(h)), "Reservoir")
        self._lib, self._h, self.cache = lib, h, cache

    def close(self) -> None:
        if getattr(self, "_h", None) is not None and self._h.value:
            self._lib.lv_reservoir_destroy(self._h)
            self._h = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass

    def update(self, key_id: int, key=None) -> int:
        """Returns the position written, or -1 when the id was not admitted."""
        slot = C.c_int64()
        check(self._lib.lv_reservoir_update(self._h, int(key_id), C.byref(slot)), "Reservoir::update")
        return int(slot.value)

    def size(self) -> int:
        return int(self._lib.lv_reservoir_size(self._h))

    def seen(self) -> int:
        return int(self._lib.lv_reservoir_seen(self._h))

    def capacity(self) -> int:
        return int(self._lib.lv_reservoir_capacity(self._h))

    def ids(self) -> np.ndarray:
        out = np.empty((self.size(),), np.uint32)
        if out.size:
            check(self._lib.lv_reservoir_ids(self._h, out.ctypes.data), "Reservoir::ids")
        return out


def _variant_args(cfg: OracleConfig):
    return int(cfg.variant), int(cfg.m), float(cfg.alpha)


def estimate_tau(res: Reservoir, q, cfg: OracleConfig, cache=None) -> float:
    """threshold.cpp:63-103 for one query against a reservoir of a ``LouverCache``
    (the reservoir's own ``cache`` unless one is passed). Runs on the device."""
    cache = cache if cache is not None else res.cache
    if cache is None:
        raise ValueError("estimate_tau: the reservoir samples no cache")
    cfg.validate()
    q = np.ascontiguousarray(q, dtype=np.float32).reshape(-1)
    if q.size != cache.d:
        raise ValueError("dot: length mismatch")
    ids = res.ids()
    tau = np.zeros((1,), np.float32)
    v, m, a = _variant_args(cfg)
    ctx = cache._ctx
    check(ctx.lib.lv_estimate_tau(ctx.h, ids.ctypes.data if ids.size else q.ctypes.data, ids.size,
                                  max(ids.size, 1), q.ctypes.data, v, m, a, LV_HOST, tau.ctypes.data, None),
          "estimate_tau")
    return float(tau[0])


def estimate_tau_layer(layer, ids, count: int, q, cfg: OracleConfig, tau_out=None, stream=None):
    """Every q head of a ``LouverLayer`` at once: ``ids`` holds the reservoir of each kv
    slot, [batch * H_kv][ld] uint32 (a cuda tensor for the device path, or a numpy
    array), the first ``count`` entries of each row valid; ``q`` [batch][H_q][d].
    Device tensors in → enqueue-only, τ written to ``tau_out`` [batch][H_q] on the
    device; numpy in → returns τ as numpy."""
    cfg.validate()
    v, m, a = _variant_args(cfg)
    ctx = layer._ctx
    if isinstance(ids, np.ndarray):
        ids = np.ascontiguousarray(ids, dtype=np.uint32)
        q = np.ascontiguousarray(q, dtype=np.float32)
        tau = np.zeros((layer.batch, layer.H_q), np.float32) if tau_out is None else tau_out
        check(ctx.lib.lv_estimate_tau(ctx.h, ids.ctypes.data, int(count), ids.shape[-1], q.ctypes.data, v, m, a,
                                      LV_HOST, tau.ctypes.data, None), "estimate_tau")
        return tau
    import torch  # plumbing only

    st = stream if stream is not None else torch.cuda.current_stream().cuda_stream
    if tau_out is None:
        tau_out = torch.empty((layer.batch, layer.H_q), dtype=torch.float32, device="cuda")
    check(ctx.lib.lv_estimate_tau(ctx.h, ids.data_ptr(), int(count), ids.shape[-1], q.data_ptr(), v, m, a,
                                  LV_DEVICE, tau_out.data_ptr(), st), "estimate_tau")
    return tau_out


__all__ = ["OracleVariant", "OracleConfig", "parse_oracle", "to_string", "Reservoir", "estimate_tau",
           "estimate_tau_layer"]
