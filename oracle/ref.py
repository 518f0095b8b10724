"""ctypes front-end for oracle/_ref/libcuboid_ref.so -- the UNMODIFIED reference
headers (/root/reference/proj/include/cuboid/*.hpp) compiled by oracle/Makefile.

TEST INFRASTRUCTURE ONLY: imported by tests/, __graft_entry__.smoke() and the
CPU legs of bench.py (cpu_baseline, --impl reference). The product package
never imports anything under oracle/.
"""
from __future__ import annotations

import ctypes as C
import os
from dataclasses import dataclass, field

_HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.path.join(_HERE, "_ref", "libcuboid_ref.so")

_u64p = C.POINTER(C.c_uint64)
_u32p = C.POINTER(C.c_uint32)
_i32p = C.POINTER(C.c_int32)
_u8p = C.POINTER(C.c_uint8)

_lib = None


def available() -> bool:
    return os.path.exists(LIB_PATH)


def lib():
    global _lib
    if _lib is None:
        if not available():
            raise FileNotFoundError(
                f"{LIB_PATH} missing: run `make -C oracle` (needs /root/reference)")
        L = C.CDLL(LIB_PATH)
        L.cref_last_error.restype = C.c_char_p
        L.cref_set_build.restype = C.c_void_p
        L.cref_set_build.argtypes = [_u32p, C.c_uint32]
        L.cref_set_load.restype = C.c_void_p
        L.cref_set_load.argtypes = [C.c_char_p, C.c_size_t, C.c_char_p, C.c_size_t]
        L.cref_set_free.argtypes = [C.c_void_p]
        L.cref_set_tables_size.restype = C.c_uint64
        L.cref_set_tables_size.argtypes = [C.c_void_p]
        L.cref_set_export.restype = C.c_uint32
        L.cref_set_export.argtypes = [C.c_void_p, C.c_void_p, C.c_void_p, C.c_void_p]
        L.cref_serialize_index.restype = C.c_int64
        L.cref_serialize_index.argtypes = [C.c_void_p, C.c_void_p, C.c_uint64]
        L.cref_is_unsolvable.argtypes = [C.c_void_p, C.c_uint64, C.c_uint64, C.c_uint64]
        L.cref_build_table.argtypes = [C.c_uint32, C.c_void_p]
        L.cref_build_table_oracle.argtypes = [C.c_uint32, C.c_void_p]
        L.cref_eval_q_mod.restype = C.c_int64
        L.cref_eval_q_mod.argtypes = [C.c_uint32] * 4
        L.cref_q_bounds.argtypes = [C.c_uint64, _u64p, _u64p]
        L.cref_verify_pair.argtypes = [C.c_void_p, C.c_uint64, C.c_uint64, C.c_int, _i32p, _u32p,
                                       C.c_char_p, C.c_uint64]
        L.cref_scan.argtypes = [C.c_void_p, C.c_uint64, C.c_uint64, C.c_uint64, C.c_int, C.c_uint64,
                                C.c_int, C.c_int, _u64p, _u64p, _u64p, _u64p, _u32p, C.c_uint64,
                                _u64p, _u64p, _i32p, C.c_uint64, _u64p, _u64p, _u64p,
                                C.POINTER(C.c_int), C.POINTER(C.c_double)]
        L.cref_scan_mt.argtypes = [C.c_void_p, C.c_uint64, C.c_uint64, C.c_int, C.c_int, _u64p, _u64p,
                                   _u64p, _u64p, _u32p, C.c_uint64, _u64p, C.POINTER(C.c_double)]
        L.cref_triangle.argtypes = [C.c_void_p, C.c_uint64, C.c_uint64, C.c_int, C.c_int, _u64p,
                                    _u64p, _u64p, _u64p, _u32p, C.c_uint64, _u64p, _u64p, _i32p,
                                    C.c_uint64, _u64p, C.POINTER(C.c_double)]
        L.cref_verify_small_region.argtypes = [C.c_void_p, _u64p]
        L.cref_classify.argtypes = [C.c_void_p, C.c_void_p, C.c_uint64, C.c_int, C.c_void_p]
        L.cref_build_tables.argtypes = [C.c_void_p, C.c_uint32, C.c_int, C.c_int, C.c_void_p,
                                        C.c_void_p, C.POINTER(C.c_double)]
        _lib = L
    return _lib


class RefError(RuntimeError):
    def __init__(self, code, msg):
        super().__init__(f"reference error {code}: {msg}")
        self.code = code


def _check(rc):
    if rc != 0:
        raise RefError(rc, lib().cref_last_error().decode())


def _arr(ctype, n, init=None):
    a = (ctype * max(n, 1))()
    if init is not None:
        for i, v in enumerate(init):
            a[i] = v
    return a


class RefSet:
    """The reference SieveSet (sievetable.hpp:155-227)."""

    def __init__(self, handle):
        if not handle:
            raise RefError(-1, lib().cref_last_error().decode())
        self.h = handle
        n = lib().cref_set_export(self.h, None, None, None)
        pr = _arr(C.c_uint32, n)
        off = _arr(C.c_uint32, n)
        lib().cref_set_export(self.h, None, pr, off)
        self.primes = [pr[i] for i in range(n)]
        self.offsets = [off[i] for i in range(n)]

    @classmethod
    def build(cls, primes):
        primes = list(primes)
        return cls(lib().cref_set_build(_arr(C.c_uint32, len(primes), primes), len(primes)))

    @classmethod
    def load(cls, tables: bytes, index: bytes):
        return cls(lib().cref_set_load(tables, len(tables), index, len(index)))

    def __del__(self):
        if getattr(self, "h", None) and _lib is not None:
            _lib.cref_set_free(self.h)
            self.h = None

    def tables(self) -> bytes:
        n = lib().cref_set_tables_size(self.h)
        buf = C.create_string_buffer(max(int(n), 1))
        lib().cref_set_export(self.h, buf, None, None)
        return buf.raw[: int(n)]

    def index_bytes(self) -> bytes:
        n = lib().cref_serialize_index(self.h, None, 0)
        if n < 0:
            raise RefError(-1, lib().cref_last_error().decode())
        buf = C.create_string_buffer(int(n))
        lib().cref_serialize_index(self.h, buf, n)
        return buf.raw

    def is_unsolvable(self, rank, p, q) -> bool:
        rc = lib().cref_is_unsolvable(self.h, rank, p, q)
        if rc < 0:
            raise IndexError(lib().cref_last_error().decode())
        return bool(rc)


def build_table(r: int) -> bytes:
    buf = C.create_string_buffer((r * r + 7) // 8)
    _check(lib().cref_build_table(r, buf))
    return buf.raw


def build_table_oracle(r: int) -> bytes:
    buf = C.create_string_buffer((r * r + 7) // 8)
    _check(lib().cref_build_table_oracle(r, buf))
    return buf.raw


def eval_q_mod(p, q, t, r) -> int:
    v = lib().cref_eval_q_mod(p, q, t, r)
    if v < 0:
        raise ValueError(lib().cref_last_error().decode())
    return v


def q_bounds(p):
    lo, hi = C.c_uint64(), C.c_uint64()
    _check(lib().cref_q_bounds(p, C.byref(lo), C.byref(hi)))
    return lo.value, hi.value


VERDICT_KINDS = ("SievedOut", "NoIntegerRoot", "RootFailsInequalities", "CuboidCandidate")


def verify_pair(rset, p, q, bypass):
    kind, prime = C.c_int32(), C.c_uint32()
    tbuf = C.create_string_buffer(4096)
    _check(lib().cref_verify_pair(rset.h if rset else None, p, q, int(bypass), C.byref(kind),
                                  C.byref(prime), tbuf, 4096))
    return VERDICT_KINDS[kind.value], prime.value, int(tbuf.value.decode() or 0)


@dataclass
class RefStats:
    pairs_tested: int = 0
    survivors: int = 0
    hist_by_rank: list = field(default_factory=list)
    block_r_max: dict = field(default_factory=dict)
    survivor_pairs: list = field(default_factory=list)  # [(p, q, kind)]
    resume_p: int = 0
    resume_q: int = 0
    stopped: bool = False
    elapsed_s: float = 0.0

    def kill_histogram(self, primes):
        return {primes[k]: c for k, c in enumerate(self.hist_by_rank) if c}


def _stats_bufs(nprimes, block_cap):
    return dict(pt=C.c_uint64(), sv=C.c_uint64(), hist=_arr(C.c_uint64, nprimes),
                blocks=_arr(C.c_uint64, block_cap), rmax=_arr(C.c_uint32, block_cap),
                nb=C.c_uint64())


def _fill(st, b, nprimes):
    st.pairs_tested = b["pt"].value
    st.survivors = b["sv"].value
    st.hist_by_rank = [b["hist"][k] for k in range(nprimes)]
    st.block_r_max = {b["blocks"][i]: b["rmax"][i] for i in range(b["nb"].value)}
    return st


def scan(rset, p, q, p_end, small_p=False, batch_pairs=0, stop_preset=False, with_sink=True,
         surv_cap=1 << 20):
    """Reference scan() (engine.hpp:195-295). Raises RefError(code) on ScanRejected."""
    n = len(rset.primes)
    block_cap = max(16, (p_end // 100) - (p // 100) + 2)
    b = _stats_bufs(n, block_cap)
    spq = _arr(C.c_uint64, 2 * surv_cap)
    skind = _arr(C.c_int32, surv_cap)
    ns, rp, rq, stopped, el = C.c_uint64(), C.c_uint64(), C.c_uint64(), C.c_int(), C.c_double()
    _check(lib().cref_scan(rset.h, p, q, p_end, int(small_p), batch_pairs, int(stop_preset),
                           int(with_sink), C.byref(b["pt"]), C.byref(b["sv"]), b["hist"], b["blocks"],
                           b["rmax"], block_cap, C.byref(b["nb"]), spq, skind, surv_cap, C.byref(ns),
                           C.byref(rp), C.byref(rq), C.byref(stopped), C.byref(el)))
    st = _fill(RefStats(), b, n)
    st.survivor_pairs = [(spq[2 * i], spq[2 * i + 1], VERDICT_KINDS[skind[i]])
                         for i in range(min(ns.value, surv_cap))]
    st.resume_p, st.resume_q, st.stopped, st.elapsed_s = rp.value, rq.value, bool(stopped.value), el.value
    return st


def scan_mt(rset, p_lo, p_hi, nthreads, small_p=False):
    n = len(rset.primes)
    block_cap = (p_hi // 100) - (p_lo // 100) + 2
    b = _stats_bufs(n, block_cap)
    el = C.c_double()
    _check(lib().cref_scan_mt(rset.h, p_lo, p_hi, int(small_p), nthreads, C.byref(b["pt"]),
                              C.byref(b["sv"]), b["hist"], b["blocks"], b["rmax"], block_cap,
                              C.byref(b["nb"]), C.byref(el)))
    st = _fill(RefStats(), b, n)
    st.elapsed_s = el.value
    return st


def triangle(rset, p_lo, p_hi, nthreads=1, with_sink=True, surv_cap=1 << 22):
    """TRIANGLE sieve over rows [p_lo, p_hi] through SieveSet::is_unsolvable."""
    n = len(rset.primes)
    block_cap = (p_hi // 100) - (p_lo // 100) + 2
    b = _stats_bufs(n, block_cap)
    cap = surv_cap if with_sink else 0
    spq = _arr(C.c_uint64, 2 * cap)
    skind = _arr(C.c_int32, cap)
    ns, el = C.c_uint64(), C.c_double()
    _check(lib().cref_triangle(rset.h, p_lo, p_hi, nthreads, int(with_sink), C.byref(b["pt"]),
                               C.byref(b["sv"]), b["hist"], b["blocks"], b["rmax"], block_cap,
                               C.byref(b["nb"]), spq, skind, cap, C.byref(ns), C.byref(el)))
    st = _fill(RefStats(), b, n)
    st.survivor_pairs = [(spq[2 * i], spq[2 * i + 1], VERDICT_KINDS[skind[i]])
                         for i in range(min(ns.value, cap))]
    st.elapsed_s = el.value
    return st


def verify_small_region(rset):
    out = _arr(C.c_uint64, 6)
    _check(lib().cref_verify_small_region(rset.h, out))
    keys = ("pairs", "sieved_out", "survivors", "no_integer_root", "root_fails", "candidates")
    return {k: out[i] for i, k in enumerate(keys)}


def classify(rset, pq, nthreads=1):
    """First-killer rank per (p, q) row of the (n, 2) uint64 array pq (-1 =
    survivor) through SieveSet::is_unsolvable in rank order."""
    import numpy as np
    pq = np.ascontiguousarray(pq, dtype=np.uint64)
    out = np.empty(len(pq), np.int32)
    _check(lib().cref_classify(rset.h, pq.ctypes.data, len(pq), nthreads, out.ctypes.data))
    return out


def build_tables(primes, oracle=False, nthreads=1):
    """The reference builders (build_table / build_table_oracle) over `primes`
    into one SieveSet-layout byte string; returns (bytes, elapsed seconds)."""
    import numpy as np
    P = np.ascontiguousarray(primes, dtype=np.uint32)
    sizes = (P.astype(np.uint64) ** 2 + 7) // 8
    offs = np.zeros(len(P), np.uint64)
    offs[1:] = np.cumsum(sizes)[:-1]
    out = np.zeros(int(sizes.sum()), np.uint8)
    el = C.c_double()
    _check(lib().cref_build_tables(P.ctypes.data, len(P), int(oracle), nthreads, offs.ctypes.data,
                                   out.ctypes.data, C.byref(el)))
    return out.tobytes(), el.value
