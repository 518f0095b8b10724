"""The C-ABI library loads and exports every symbol include/cuboid_gpu.h
declares; host-only entry points behave like the reference's validation; with
no GPU every device entry point fails loudly (there is no CPU fallback).
CPU only."""
from __future__ import annotations

import ctypes as C
import os
import re

import numpy as np
import pytest

from oracle import port
from paper_1601_00636_b200 import _native as N
from paper_1601_00636_b200.primes import default_primes, odd_primes

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
HEADER = os.path.join(ROOT, "include", "cuboid_gpu.h")


def header_symbols():
    src = open(HEADER).read()
    src = re.sub(r"/\*.*?\*/", "", src, flags=re.S)
    return sorted(set(re.findall(r"\b(cgpu_[a-z_0-9]+)\s*\(", src)))


def test_header_declares_abi():
    syms = header_symbols()
    assert "cgpu_sieve_launch" in syms and "cgpu_tables_build" in syms
    assert set(syms) == set(N.SIGNATURES), "ctypes table and header disagree"


def test_library_exports_every_symbol():
    lib = N.lib()
    for s in header_symbols():
        assert hasattr(lib, s), s


def test_library_is_sm100a_only():
    out = os.popen(f"cuobjdump --list-elf {N.LIB_PATH} 2>&1").read()
    assert "sm_100a" in out
    assert not re.search(r"sm_(?!100a)\d+", out), out


def test_version_string():
    assert "sm_100a" in N.lib().cgpu_version().decode()


@pytest.mark.parametrize("name", ["odd32", "odd256", "default96"])
def test_table_layout_matches_oracle(sets, name):
    P = np.array(sets[name], np.uint32)
    offs = np.zeros(len(P), np.uint32)
    total = C.c_uint64()
    assert N.lib().cgpu_table_layout(P.ctypes.data_as(C.c_void_p), len(P),
                                     offs.ctypes.data_as(C.c_void_p), C.byref(total)) == N.OK
    tb, o = port.build_set(sets[name]) if name != "odd256" else (None, None)
    if tb is not None:
        assert total.value == len(tb)
        assert offs.tolist() == list(o)
    assert offs[0] == 0 and all((int(r) * int(r) + 7) // 8 == int(b) - int(a)
                                for r, a, b in zip(P, offs, list(offs[1:]) + [total.value]))


@pytest.mark.parametrize("primes", [[13, 11], [11, 11], [11, 15], [9697], [1], [2, 9699]])
def test_table_layout_rejects_like_reference(primes):
    """SieveSet::build / build_table validation (sievetable.hpp:83-87, 159-176)."""
    P = np.array(primes, np.uint32)
    total = C.c_uint64()
    rc = N.lib().cgpu_table_layout(P.ctypes.data_as(C.c_void_p), len(P), None, C.byref(total))
    assert rc == N.ERR_INVALID


def test_table_layout_overflow():
    """std::overflow_error once the set passes 2^32 bytes (sievetable.hpp:169-170):
    the largest legal list, every prime below 9697, is checked against the sum."""
    P = np.array([p for p in range(2, 9697) if port.lib().co_is_prime(p)], np.uint32)
    total = C.c_uint64()
    rc = N.lib().cgpu_table_layout(P.ctypes.data_as(C.c_void_p), len(P), None, C.byref(total))
    expect = sum((int(r) * int(r) + 7) // 8 for r in P)
    if expect > 0xFFFFFFFF:
        assert rc == N.ERR_OVERFLOW
    else:
        assert rc == N.OK and total.value == expect


def test_q_bounds_host():
    lo, hi = C.c_uint64(), C.c_uint64()
    for p in (1, 58, 59, 60, 151, 152, 153, 10**6, 72796055, 10**12):
        assert N.lib().cgpu_q_bounds(p, C.byref(lo), C.byref(hi)) == N.OK
        assert (lo.value, hi.value) == port.q_bounds(p)
    assert N.lib().cgpu_q_bounds(0, C.byref(lo), C.byref(hi)) == N.ERR_INVALID


def test_no_cpu_fallback_without_gpu():
    """On a box without a CUDA device the product path refuses to run."""
    import torch
    if torch.cuda.is_available():
        pytest.skip("a GPU is visible")
    ctx = C.c_void_p()
    rc = N.lib().cgpu_create(0, None, C.byref(ctx))
    assert rc == N.ERR_NO_DEVICE
    assert "no CPU fallback" in N.last_error()
    from paper_1601_00636_b200 import cuboid
    with pytest.raises(N.CudaSieveError):
        cuboid.SieveSet.build(odd_primes(4))


def test_multi_gpu_refuses_without_gpu():
    import torch
    if torch.cuda.is_available():
        pytest.skip("a GPU is visible")
    m = C.c_void_p()
    assert N.lib().cgpu_multi_create(2, None, C.byref(m)) == N.ERR_NO_DEVICE
    assert not m.value


def test_multi_null_handles_are_errors():
    assert N.lib().cgpu_multi_sieve(None, 2, 0, 10, 0, N.TRIANGLE, None, None, None, 0, None, 0) == N.ERR_INVALID
    assert N.lib().cgpu_multi_tables_load(None, None, 0, None, 0) == N.ERR_INVALID
    assert N.lib().cgpu_multi_destroy(None) == N.OK


def test_null_context_is_an_error():
    assert N.lib().cgpu_sieve_launch(None, 2, 0, 10, N.TRIANGLE, 1, 0, 0) == N.ERR_INVALID
    assert N.lib().cgpu_destroy(None) == N.OK


def test_product_package_never_imports_oracle():
    pkg = os.path.join(ROOT, "paper_1601_00636_b200")
    for dirpath, _, files in os.walk(pkg):
        for f in files:
            if f.endswith((".py", ".cu", ".cuh", ".cpp", ".h")):
                src = open(os.path.join(dirpath, f)).read()
                assert "oracle" not in re.findall(r"^\s*(?:from|import)\s+(\w+)", src, re.M), f


def test_region_advance_matches_the_visiting_order():
    """cgpu_region_advance (host) walks scan()'s q order like a row-by-row
    count (engine.hpp:225-248), including the small-p rows and a mid-row start."""
    import random
    from paper_1601_00636_b200 import cuboid
    rng = random.Random(5)
    for _ in range(40):
        p = rng.choice([1, 7, 150, 151, 152, 153, 999, 12345, 400000])
        lo, hi = cuboid.q_bounds(p)
        q = rng.randrange(lo, hi + 1)
        k = rng.choice([0, 1, 5, hi - q, hi - q + 1, 10**5, 3 * 10**6])
        p_end = p + rng.randrange(0, 50)
        want = cuboid.stop_point((p, q), p_end, k + 1)  # the (k+1)-th q visited
        assert cuboid.region_advance((p, q), k, p_end) == want
