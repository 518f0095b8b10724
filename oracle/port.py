"""ctypes front-end for oracle/libcuboid_oracle.so, the plain-C restatement of
the reference hot path (oracle/cuboid_oracle.c).

TEST INFRASTRUCTURE ONLY: used by tests/ and bench.py's cpu_baseline leg as
the checker. Never imported by the product package.
"""
from __future__ import annotations

import ctypes as C
import os

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.path.join(_HERE, "libcuboid_oracle.so")
_lib = None


def lib():
    global _lib
    if _lib is None:
        if not os.path.exists(LIB_PATH):
            raise FileNotFoundError(f"{LIB_PATH} missing: run `make -C oracle liboracle`")
        L = C.CDLL(LIB_PATH)
        L.co_is_prime.argtypes = [C.c_uint32]
        L.co_mod_inverse.restype = C.c_uint32
        L.co_mod_inverse.argtypes = [C.c_uint32, C.c_uint32]
        L.co_mod_coeffs.argtypes = [C.c_uint32, C.c_uint32, C.c_uint32, C.c_void_p]
        L.co_horner_mod.restype = C.c_uint32
        L.co_horner_mod.argtypes = [C.c_void_p, C.c_uint32, C.c_uint32]
        L.co_eval_q_mod.restype = C.c_int64
        L.co_eval_q_mod.argtypes = [C.c_uint32] * 4
        L.co_table_bytes.restype = C.c_uint64
        L.co_table_bytes.argtypes = [C.c_uint32]
        L.co_build_table.argtypes = [C.c_uint32, C.c_void_p]
        L.co_build_table_oracle.argtypes = [C.c_uint32, C.c_void_p, C.POINTER(C.c_uint64)]
        L.co_build_set.restype = C.c_int64
        L.co_build_set.argtypes = [C.c_void_p, C.c_uint32, C.c_void_p, C.c_void_p]
        L.co_q_lower_cubic.restype = C.c_uint64
        L.co_q_lower_cubic.argtypes = [C.c_uint64]
        L.co_q_bounds.argtypes = [C.c_uint64, C.POINTER(C.c_uint64), C.POINTER(C.c_uint64)]
        L.co_sieve.argtypes = [C.c_void_p, C.c_void_p, C.c_void_p, C.c_uint32, C.c_uint64,
                               C.c_uint64, C.c_uint64, C.c_int, C.POINTER(C.c_uint64),
                               C.POINTER(C.c_uint64), C.c_void_p, C.c_void_p, C.c_void_p,
                               C.c_uint64, C.POINTER(C.c_uint64)]
        _lib = L
    return _lib


def _ptr(a: np.ndarray):
    return a.ctypes.data_as(C.c_void_p)


def eval_q_mod(p, q, t, r) -> int:
    return int(lib().co_eval_q_mod(p, q, t, r))


def mod_coeffs(p, q, r):
    c = np.zeros(5, np.uint32)
    lib().co_mod_coeffs(p, q, r, _ptr(c))
    return c


def build_table(r: int) -> bytes:
    out = np.zeros((r * r + 7) // 8, np.uint8)
    if lib().co_build_table(r, _ptr(out)) != 0:
        raise ValueError(f"bad modulus {r}")
    return out.tobytes()


def build_table_oracle(r: int):
    out = np.zeros((r * r + 7) // 8, np.uint8)
    ev = C.c_uint64()
    if lib().co_build_table_oracle(r, _ptr(out), C.byref(ev)) != 0:
        raise ValueError(f"bad modulus {r}")
    return out.tobytes(), ev.value


def build_set(primes):
    pr = np.ascontiguousarray(primes, dtype=np.uint32)
    total = lib().co_build_set(_ptr(pr), len(pr), None, None)
    if total < 0:
        raise ValueError("bad prime list" if total == -1 else "table set exceeds 2^32 bytes")
    out = np.zeros(max(total, 1), np.uint8)
    offs = np.zeros(max(len(pr), 1), np.uint32)
    lib().co_build_set(_ptr(pr), len(pr), _ptr(out), _ptr(offs))
    return out[:total].tobytes(), offs[: len(pr)].copy()


def q_bounds(p):
    lo, hi = C.c_uint64(), C.c_uint64()
    lib().co_q_bounds(p, C.byref(lo), C.byref(hi))
    return lo.value, hi.value


REGION, TRIANGLE = 0, 1


def sieve(tables: bytes, primes, offsets, p_lo, p_hi, mode, q_start=0, surv_cap=1 << 22):
    """Returns dict(pairs_tested, survivors, hist (np.uint64[n]), row_rmax
    (np.uint32[rows]), survivor_pairs (np.uint64[k,2]))."""
    t = np.frombuffer(tables, np.uint8) if len(tables) else np.zeros(1, np.uint8)
    pr = np.ascontiguousarray(primes, dtype=np.uint32)
    of = np.ascontiguousarray(offsets, dtype=np.uint32)
    n = len(pr)
    hist = np.zeros(max(n, 1), np.uint64)
    rows = max(p_hi - p_lo + 1, 0)
    rr = np.zeros(max(rows, 1), np.uint32)
    spq = np.zeros((max(surv_cap, 1), 2), np.uint64)
    pt, sv, ns = C.c_uint64(), C.c_uint64(), C.c_uint64()
    lib().co_sieve(_ptr(t), _ptr(pr), _ptr(of), n, p_lo, q_start, p_hi, mode, C.byref(pt),
                   C.byref(sv), _ptr(hist), _ptr(rr), _ptr(spq), surv_cap, C.byref(ns))
    return dict(pairs_tested=pt.value, survivors=sv.value, hist=hist[:n], row_rmax=rr[:rows],
                survivor_pairs=spq[: min(ns.value, surv_cap)])
