"""The C-ABI library loads on a CPU-only box and exports every entry point
include/*.h declares (no compute calls — those need a GPU)."""
import ctypes
import os
import re

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def declared_functions(header):
    text = open(header).read()
    text = re.sub(r"/\*.*?\*/", "", text, flags=re.S)
    return sorted(set(re.findall(r"^\s*(?:const\s+)?[a-z_0-9]+\s*\*?\s*(lv_[a-z_0-9]+)\s*\(", text, flags=re.M)))


def test_header_declares_the_boundary():
    names = declared_functions(os.path.join(ROOT, "include", "louver_b200.h"))
    for must in ("lv_create", "lv_build", "lv_push_key", "lv_flush", "lv_query", "lv_brute_force_range",
                 "lv_sparse_attention", "lv_dense_decode", "lv_lse_merge", "lv_last_error"):
        assert must in names


def test_libraries_export_every_declared_symbol():
    from paper_2605_06763_b200 import _capi

    main = ctypes.CDLL(_capi.LIB_PATH)
    synth = ctypes.CDLL(_capi.SYNTH_PATH)
    missing = []
    for name in declared_functions(os.path.join(ROOT, "include", "louver_b200.h")):
        lib = synth if name.startswith("lv_synth") else main
        if not hasattr(lib, name):
            missing.append(name)
    assert not missing, missing


def test_build_info_and_no_device_error():
    from paper_2605_06763_b200 import _capi

    L = _capi.lib()
    assert b"sm_100a" in L.lv_build_info()
    import torch

    if torch.cuda.is_available():
        pytest.skip("device present: the no-device path is not reachable")
    cfg = _capi.lv_config(d=8, n_kv_heads=1, group_size=1, batch=1, dtype=0, S=1, r=4, grouping=0,
                          enclosure=1, rng_seed=0, buffer_capacity=4, capacity=64)
    h = ctypes.c_void_p()
    rc = L.lv_create(ctypes.byref(cfg), ctypes.byref(h))
    assert rc == _capi.LV_ENODEV  # fails loudly: no CPU fallback
    with pytest.raises(_capi.LouverError):
        _capi.check(rc, "lv_create")


def test_config_validation_matches_reference():
    """BuildConfig::validate (index.hpp:17-21) errors surface before any device work."""
    from paper_2605_06763_b200 import BuildConfig

    with pytest.raises(ValueError):
        BuildConfig(S=0).validate(8)
    with pytest.raises(ValueError):
        BuildConfig(r=0).validate(8)
    with pytest.raises(ValueError):
        BuildConfig(S=9).validate(8)
    BuildConfig(S=8, r=1).validate(8)
