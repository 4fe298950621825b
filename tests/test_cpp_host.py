"""The C++ host layer (include/louver_b200.hpp, the reference-shaped API) builds
against the C-ABI library, and on a GPU matches the CPU oracle
(tests/cpp/test_host.cpp: cache query vs brute force, strict toggle,
flush-at-B, sparse_attention known answers, error mapping, bf16 GQA layer)."""
import os
import subprocess

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
CPP = os.path.join(ROOT, "tests", "cpp")


def _build():
    r = subprocess.run(["make", "-s", "-C", CPP], capture_output=True, text=True)
    assert r.returncode == 0, r.stdout + r.stderr
    return os.path.join(CPP, "test_host")


def test_cpp_host_layer_compiles_and_links():
    exe = _build()
    r = subprocess.run([exe, "--compile-only"], capture_output=True, text=True, timeout=120)
    assert r.returncode == 0, r.stdout + r.stderr
    assert "sm_100a" in r.stdout


@pytest.mark.gpu
def test_cpp_host_layer_matches_oracle():
    exe = _build()
    r = subprocess.run([exe], capture_output=True, text=True, timeout=600)
    assert r.returncode == 0 and r.stdout.strip().endswith("OK"), r.stdout + r.stderr


def test_cpp_sharded_layer_compiles_and_links():  # include/louver_b200_nccl.hpp
    _build()
    exe = os.path.join(CPP, "test_sharded")
    r = subprocess.run([exe, "--compile-only"], capture_output=True, text=True, timeout=120)
    assert r.returncode == 0 and "nccl" in r.stdout, r.stdout + r.stderr


@pytest.mark.gpu
def test_cpp_sharded_layer_matches_unsharded():
    _build()
    r = subprocess.run([os.path.join(CPP, "test_sharded")], capture_output=True, text=True, timeout=600)
    assert r.returncode == 0 and r.stdout.strip().endswith("OK"), r.stdout + r.stderr
