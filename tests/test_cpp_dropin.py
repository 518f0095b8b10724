"""The C++ drop-in (include/cuboid/gpu.hpp) against the reference's own C++ API:
cpp/test_dropin.cpp, compiled by `make -C cpp` from the unmodified reference
headers (build time only) and libcuboid_gpu.so."""
from __future__ import annotations

import os
import subprocess

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
BIN = os.path.join(ROOT, "cpp", "_build", "test_dropin")

needs_bin = pytest.mark.skipif(not os.path.exists(BIN), reason="cpp/_build/test_dropin not built")


@needs_bin
@pytest.mark.gpu
def test_cpp_dropin_matches_reference():
    r = subprocess.run([BIN], capture_output=True, text=True, timeout=600)
    assert r.returncode == 0, r.stdout + r.stderr
    assert " 0 failed" in r.stdout


@needs_bin
def test_cpp_dropin_fails_loudly_without_gpu():
    import torch
    if torch.cuda.is_available():
        pytest.skip("a GPU is visible")
    r = subprocess.run([BIN], capture_output=True, text=True, timeout=60)
    assert r.returncode != 0
    assert "no CPU fallback" in r.stderr
