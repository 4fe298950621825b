"""ctypes binding of the C ABI in include/louver_b200.h.

The shared libraries are built in-tree by ``__graft_entry__.build()`` (or
``make -C paper_2605_06763_b200/csrc``). Loading fails loudly when they are
missing: the hot path has no CPU fallback.
"""
from __future__ import annotations

import ctypes as C
import os

_HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.environ.get("LOUVER_B200_LIB") or os.path.join(_HERE, "liblouver_b200.so")  # env: A/B builds (tools only)
SYNTH_PATH = os.path.join(_HERE, "liblouver_synth.so")

LV_OK, LV_EMPTY, LV_EINVAL, LV_ERANGE, LV_ERUNTIME, LV_ENODEV = 0, 1, -1, -2, -3, -4
LV_F32, LV_BF16 = 0, 1
LV_HOST, LV_DEVICE = 0, 1
LV_ALGO_FULL_SUBSPACE, LV_ALGO_TA = 0, 1
LV_TAU_MAX, LV_TAU_TOPK, LV_TAU_GAP, LV_TAU_MEANMAX, LV_TAU_BUDGET = 0, 1, 2, 3, 4


class lv_config(C.Structure):
    _fields_ = [
        ("d", C.c_int),
        ("n_kv_heads", C.c_int),
        ("group_size", C.c_int),
        ("batch", C.c_int),
        ("dtype", C.c_int),
        ("S", C.c_int),
        ("r", C.c_int),
        ("grouping", C.c_int),
        ("enclosure", C.c_int),
        ("rng_seed", C.c_uint64),
        ("buffer_capacity", C.c_int64),
        ("capacity", C.c_int64),
        ("group_index", C.c_int),
    ]


class lv_group_stats(C.Structure):
    _fields_ = [
        ("groups_tested", C.c_int64),
        ("keys_scanned", C.c_int64),
        ("f_scan", C.c_double),
        ("gate_cost_equiv", C.c_double),
        ("ta_stop_depth", C.c_int32),
        ("ta_stop_upper", C.c_double),
    ]


class lv_query_args(C.Structure):
    _fields_ = [
        ("q", C.c_void_p),
        ("tau", C.c_void_p),
        ("scale", C.c_float),
        ("algo", C.c_int),
        ("strict", C.c_int),
        ("where", C.c_int),
        ("out", C.c_void_p),
        ("partial", C.c_void_p),
        ("counts", C.c_void_p),
        ("sel_bits", C.c_void_p),
        ("totals", C.c_void_p),
        ("workspace", C.c_void_p),
        ("stream", C.c_void_p),
        ("cand_bits", C.c_void_p),
    ]


class LouverError(RuntimeError):
    pass


def _load(path: str) -> C.CDLL:
    if not os.path.exists(path):
        raise ImportError(
            f"{os.path.basename(path)} is not built ({path}); run __graft_entry__.build() — "
            "the Louver hot path has no CPU fallback"
        )
    return C.CDLL(path)


class lv_step_copy(C.Structure):
    _fields_ = [("src", C.c_void_p), ("dst", C.c_void_p), ("stride", C.c_int64), ("bytes", C.c_int64),
                ("dir", C.c_int)]


_lib = None
_synth = None

_P = C.c_void_p
_SIGS = {
    "lv_last_error": (C.c_char_p, []),
    "lv_build_info": (C.c_char_p, []),
    "lv_create": (C.c_int, [C.POINTER(lv_config), C.POINTER(_P)]),
    "lv_destroy": (C.c_int, [_P]),
    "lv_build": (C.c_int, [_P, _P, _P, C.c_int64, C.c_int, C.c_int, _P]),
    "lv_push_key": (C.c_int, [_P, _P, _P, C.c_int, C.c_int, _P]),
    "lv_flush": (C.c_int, [_P, _P]),
    "lv_reserve": (C.c_int, [_P, C.c_int64, _P]),
    "lv_sync_counters": (C.c_int, [_P, _P]),
    "lv_query": (C.c_int, [_P, C.POINTER(lv_query_args)]),
    "lv_query_workspace_bytes": (C.c_size_t, [_P]),
    "lv_query_layers": (C.c_int, [_P, C.c_int, _P, _P, C.c_float, C.c_int, _P, _P, _P]),
    "lv_query_layers_staging_bytes": (C.c_size_t, [_P, C.c_int]),
    "lv_geometry": (C.c_int, [_P, _P]),
    "lv_debug_trace": (C.c_int, [_P, _P]),
    "lv_layer_geometry": (C.c_int, [_P, _P]),
    "lv_bitmap_words": (C.c_int64, [_P]),
    "lv_n": (C.c_int64, [_P]),
    "lv_indexed_count": (C.c_int64, [_P]),
    "lv_pending_count": (C.c_int64, [_P]),
    "lv_flush_count": (C.c_int64, [_P]),
    "lv_read_rows": (C.c_int, [_P, C.c_int, C.c_int64, C.c_int64, C.c_int, _P]),
    "lv_brute_force_range": (C.c_int, [_P, _P, _P, C.c_int64, C.c_int, _P, _P]),
    "lv_bitmap_to_ids": (C.c_int, [_P, C.c_int64, C.c_int64, C.c_int64, _P, C.c_int64, _P, _P]),
    "lv_sparse_attention": (
        C.c_int,
        [_P, C.c_int, _P, C.c_int64, _P, C.c_int64, _P, C.c_float, C.c_int, _P, _P,
         C.POINTER(C.c_int64), _P],
    ),
    "lv_dense_decode": (C.c_int, [_P, _P, C.c_float, C.c_int, _P, _P, _P]),
    "lv_exact_check": (C.c_int, [_P, C.c_int, _P, C.c_int64, _P, C.c_float, C.c_int, _P, _P]),
    "lv_subspace_thresholds": (C.c_int, [_P, C.c_int, _P, C.c_float, C.c_int, C.c_int, _P, _P]),
    "lv_attention_weights": (C.c_int, [_P, C.c_int, _P, C.c_int64, _P, C.c_float, C.c_float, C.c_float, C.c_int,
                                       _P, _P]),
    "lv_lse_merge": (C.c_int, [_P, C.c_int, C.c_int64, C.c_int, _P, _P]),
    "lv_reservoir_create": (C.c_int, [C.c_int64, C.c_uint64, C.POINTER(_P)]),
    "lv_reservoir_destroy": (C.c_int, [_P]),
    "lv_reservoir_update": (C.c_int, [_P, C.c_uint32, C.POINTER(C.c_int64)]),
    "lv_reservoir_size": (C.c_int64, [_P]),
    "lv_reservoir_seen": (C.c_int64, [_P]),
    "lv_reservoir_capacity": (C.c_int64, [_P]),
    "lv_reservoir_ids": (C.c_int, [_P, _P]),
    "lv_save_dataset": (C.c_int, [C.c_char_p, _P, C.c_int64, C.c_int]),
    "lv_load_dataset": (C.c_int, [C.c_char_p, _P, C.c_int64, C.POINTER(C.c_int64), C.POINTER(C.c_int)]),
    "lv_save_index": (C.c_int, [_P, C.c_int, C.c_char_p]),
    "lv_load_index": (C.c_int, [_P, C.c_char_p, C.POINTER(C.c_int64), _P]),
    "lv_bits_diff": (C.c_int, [_P, _P, C.c_int64, C.c_int64, _P, _P]),
    "lv_step_copies": (C.c_int, [_P, _P, C.c_int, _P]),
    "lv_step_load": (C.c_int, [_P, _P, C.c_int64, _P, C.c_int64, _P]),
    "lv_step_store": (C.c_int, [_P, _P, _P, C.c_int64, C.c_int64, _P]),
    "lv_step_reservoir": (C.c_int, [_P, _P, C.c_int64, _P, C.c_int, C.c_int64, _P]),
    "lv_step_advance": (C.c_int, [_P, _P]),
    "lv_step_epilogue": (C.c_int, [_P, _P, C.c_int, _P, C.c_int64, _P, C.c_int, C.c_int64, _P]),
    "lv_group_candidates": (C.c_int, [_P, C.c_int, _P, C.c_float, _P, C.c_int, _P, _P, C.c_int64,
                                      C.POINTER(C.c_int64), C.POINTER(lv_group_stats), _P]),
    "lv_group_thresholds": (C.c_int, [_P, C.c_int, _P, C.c_float, _P, _P]),
    "lv_group_count": (C.c_int64, [_P]),
    "lv_group_export": (C.c_int, [_P, C.c_int, C.c_int, _P, _P, _P, _P, _P, _P, C.POINTER(C.c_double)]),
    "lv_estimate_tau": (C.c_int, [_P, _P, C.c_int64, C.c_int64, _P, C.c_int, C.c_int, C.c_double, C.c_int, _P, _P]),
}

_SYNTH_SIGS = {
    "lv_synth_keys": (C.c_int, [C.c_int64, C.c_int, C.c_uint64, _P]),
    "lv_synth_queries": (C.c_int, [C.c_int64, C.c_int, C.c_uint64, _P]),
    "lv_synth_mixture": (C.c_int, [C.c_int64, C.c_int, C.c_int, C.c_double, C.c_uint64, C.c_int, _P]),
    "lv_synth_keys_multi": (C.c_int, [C.c_int64, C.c_int, _P, C.c_int64, _P, C.c_int]),
}


def lib() -> C.CDLL:
    global _lib
    if _lib is None:
        L = _load(LIB_PATH)
        for name, (res, args) in _SIGS.items():
            fn = getattr(L, name)
            fn.restype = res
            fn.argtypes = args
        _lib = L
    return _lib


def synth_lib() -> C.CDLL:
    global _synth
    if _synth is None:
        L = _load(SYNTH_PATH)
        for name, (res, args) in _SYNTH_SIGS.items():
            fn = getattr(L, name)
            fn.restype = res
            fn.argtypes = args
        _synth = L
    return _synth


def check(rc: int, what: str = "") -> int:
    """Map status codes onto the reference's exception types.

    LV_EINVAL -> ValueError (std::invalid_argument), LV_ERANGE -> IndexError
    (std::out_of_range), LV_ERUNTIME/LV_ENODEV -> LouverError. LV_EMPTY is
    returned to the caller (it means nullopt / false, not an error).
    """
    if rc >= 0:
        return rc
    msg = (lib().lv_last_error() or b"").decode() or what
    if rc == LV_EINVAL:
        raise ValueError(msg)
    if rc == LV_ERANGE:
        raise IndexError(msg)
    raise LouverError(f"{what}: {msg} (status {rc})")
