"""Shared fixtures. `-m gpu` tests need a B200 (they run through the C ABI of
libcuboid_gpu.so); everything else runs on the CPU build container."""
from __future__ import annotations

import json
import os
import sys

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
if ROOT not in sys.path:
    sys.path.insert(0, ROOT)

GOLDEN_PATH = os.path.join(ROOT, "tests", "golden", "golden.json")


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: needs a CUDA device (B200, sm_100a)")
    config.addinivalue_line("markers", "slow: long-running CPU oracle case")
    # a fresh checkout has no built libraries (they are not committed): build
    # them once, here, the same way the driver's build() does
    libs = [os.path.join(ROOT, "paper_1601_00636_b200", "libcuboid_gpu.so"),
            os.path.join(ROOT, "oracle", "libcuboid_oracle.so")]
    if not all(os.path.exists(p) for p in libs):
        import __graft_entry__
        __graft_entry__.build()


@pytest.fixture(scope="session")
def golden():
    with open(GOLDEN_PATH) as f:
        return json.load(f)


@pytest.fixture(scope="session")
def sets():
    from paper_1601_00636_b200.primes import default_primes, odd_primes
    return {"odd32": odd_primes(32), "odd64": odd_primes(64), "odd128": odd_primes(128),
            "odd256": odd_primes(256), "default96": default_primes(), "weak11": [11]}
