"""Per-GPU handle over the C ABI: a resident table set plus sieve launches.

numpy arrays in, numpy arrays out. One Device per GPU (one process per GPU);
all work is enqueued on the Device's stream.
"""
from __future__ import annotations

import ctypes as C
from dataclasses import dataclass

import numpy as np

from . import _native as N


def _ptr(a):
    return None if a is None else a.ctypes.data_as(C.c_void_p)


@dataclass
class SieveResult:
    """Device results of one sieve launch (cuboid_gpu.h cgpu_sieve_results)."""
    pairs_tested: int
    survivors: int
    hist: np.ndarray         # uint64[n primes], first-killer counts by rank
    block_lo: int            # p_lo // 100
    block_rmax: np.ndarray   # uint32[p_hi//100 - p_lo//100 + 1]; 0 = block not in shard
    survivor_pairs: np.ndarray  # uint64[k, 2], ascending (p, q)


class Device:
    def __init__(self, device: int = 0, stream: int | None = None):
        self._ctx = C.c_void_p()
        N.check(N.lib().cgpu_create(int(device), C.c_void_p(stream) if stream else None,
                                    C.byref(self._ctx)))
        self.device = device
        self.primes = np.zeros(0, np.uint32)
        self.offsets = np.zeros(0, np.uint32)
        self.total_bytes = 0
        self._last = None

    def close(self):
        if self._ctx:
            N.lib().cgpu_destroy(self._ctx)
            self._ctx = C.c_void_p()

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass

    def set_stream(self, stream: int | None):
        N.check(N.lib().cgpu_set_stream(self._ctx, C.c_void_p(stream) if stream else None))

    def synchronize(self):
        N.check(N.lib().cgpu_synchronize(self._ctx))

    # ---- tables --------------------------------------------------------------
    @staticmethod
    def layout(primes):
        pr = np.ascontiguousarray(primes, dtype=np.uint32)
        offs = np.zeros(max(len(pr), 1), np.uint32)
        total = C.c_uint64()
        N.check(N.lib().cgpu_table_layout(_ptr(pr), len(pr), _ptr(offs), C.byref(total)))
        return offs[: len(pr)], total.value

    def build(self, primes, algorithm=N.BUILD_PRODUCTION, download=True):
        """Build the set on the device (SieveSet::build). Returns (bytes|None, evals)."""
        pr = np.ascontiguousarray(primes, dtype=np.uint32)
        offs, total = self.layout(pr)
        out = np.zeros(max(total, 1), np.uint8) if download else None
        ev = C.c_uint64()
        N.check(N.lib().cgpu_tables_build(self._ctx, _ptr(pr), len(pr), int(algorithm), _ptr(out),
                                          None, C.byref(ev)))
        self.primes, self.offsets, self.total_bytes = pr.copy(), offs, total
        return (out[:total].tobytes() if download else None), ev.value

    def load(self, primes, tables: bytes):
        """Upload reference-format packed tables (load_sieve)."""
        pr = np.ascontiguousarray(primes, dtype=np.uint32)
        buf = np.frombuffer(tables, np.uint8) if len(tables) else np.zeros(1, np.uint8)
        N.check(N.lib().cgpu_tables_load(self._ctx, _ptr(pr), len(pr), _ptr(buf), len(tables)))
        self.primes = pr.copy()
        self.offsets, self.total_bytes = self.layout(pr)

    def load_dev(self, primes, d_ptr: int, nbytes: int, async_: bool = False):
        """Upload packed tables that already sit in device memory on this GPU
        (e.g. all-gathered by parallel.load_tables_sharded), on this stream.
        async_: cgpu_tables_load_dev_async (no host wait; verified later by
        load_status / load_status_copy / the next results call)."""
        pr = np.ascontiguousarray(primes, dtype=np.uint32)
        fn = N.lib().cgpu_tables_load_dev_async if async_ else N.lib().cgpu_tables_load_dev
        N.check(fn(self._ctx, _ptr(pr), len(pr), C.c_void_p(d_ptr), int(nbytes)))
        self.primes = pr.copy()
        self.offsets, self.total_bytes = self.layout(pr)

    def load_host_async(self, primes, h_ptr: int, nbytes: int):
        """cgpu_tables_load_async from host memory at h_ptr (pinned for a truly
        asynchronous copy; it must stay valid until the stream has read it)."""
        pr = np.ascontiguousarray(primes, dtype=np.uint32)
        N.check(N.lib().cgpu_tables_load_async(self._ctx, _ptr(pr), len(pr), C.c_void_p(h_ptr), int(nbytes)))
        self.primes = pr.copy()
        self.offsets, self.total_bytes = self.layout(pr)

    def load_status(self):
        """Verify the last asynchronous load (waits; raises on a deferred error)."""
        N.check(N.lib().cgpu_load_status(self._ctx))

    def load_status_copy(self, dst_ptr: int):
        """Enqueue a copy of the load-status word (u32, 0 = ok) to dst_ptr."""
        N.check(N.lib().cgpu_load_status_copy(self._ctx, C.c_void_p(dst_ptr)))

    def save_files(self, tables_path: str, index_path: str):
        """save_sieve_files of the resident set (sievetable.hpp:334-339)."""
        N.check(N.lib().cgpu_tables_save_files(self._ctx, tables_path.encode(), index_path.encode()))

    def load_files(self, tables_path: str, index_path: str):
        """load_sieve_files onto the device (sievetable.hpp:341-346)."""
        N.check(N.lib().cgpu_tables_load_files(self._ctx, tables_path.encode(), index_path.encode()))
        with open(index_path, "rb") as f:
            self.primes = np.array(parse_index(f.read())[0], np.uint32)
        self.offsets, self.total_bytes = self.layout(self.primes)

    def download(self) -> bytes:
        out = np.zeros(max(self.total_bytes, 1), np.uint8)
        N.check(N.lib().cgpu_tables_download(self._ctx, _ptr(out), self.total_bytes))
        return out[: self.total_bytes].tobytes()

    def killable(self) -> np.ndarray:
        n = C.c_uint32()
        k = np.zeros(max(len(self.primes), 1), np.uint8)
        N.check(N.lib().cgpu_tables_info(self._ctx, C.byref(n), _ptr(k)))
        return k[: n.value].astype(bool)

    # ---- sieve ---------------------------------------------------------------
    def sieve_launch(self, p_lo, p_hi, mode=N.TRIANGLE, q_start=0, shard=(1, 0), surv_cap=1 << 20):
        G, g = shard
        N.check(N.lib().cgpu_sieve_launch(self._ctx, int(p_lo), int(q_start), int(p_hi), int(mode),
                                          int(G), int(g), int(surv_cap)))
        self._last = (int(p_lo), int(p_hi), int(surv_cap))

    def sieve_results(self, want_survivors=True) -> SieveResult:
        p_lo, p_hi, cap = self._last
        n = len(self.primes)
        counts = np.zeros(2, np.uint64)
        hist = np.zeros(max(n, 1), np.uint64)
        nb = p_hi // 100 - p_lo // 100 + 1 if p_hi >= p_lo else 0
        brm = np.zeros(max(nb, 1), np.uint32)
        spq = np.zeros((max(cap, 1), 2), np.uint64) if want_survivors else None
        rc = N.lib().cgpu_sieve_results(self._ctx, _ptr(counts), _ptr(hist), _ptr(brm), nb,
                                        _ptr(spq), cap if want_survivors else 0)
        if rc not in (N.OK, N.ERR_CAPACITY):
            N.check(rc)
        surv = int(counts[1])
        k = min(surv, cap) if want_survivors else 0
        res = SieveResult(int(counts[0]), surv, hist[:n], p_lo // 100, brm[:nb],
                          spq[:k] if want_survivors else np.zeros((0, 2), np.uint64))
        if rc == N.ERR_CAPACITY:
            err = N.CudaSieveError(rc, f"{surv} survivors exceed the buffer of {cap}")
            err.survivors = surv
            raise err
        return res

    def sieve(self, p_lo, p_hi, mode=N.TRIANGLE, q_start=0, shard=(1, 0), surv_cap=1 << 20):
        self.sieve_launch(p_lo, p_hi, mode, q_start, shard, surv_cap)
        return self.sieve_results()

    def timings_ms(self):
        t = (C.c_float * 3)()
        N.check(N.lib().cgpu_last_timings(self._ctx, t))
        return {"plan": t[0], "sieve": t[1], "total": t[2]}

    def sieve_kernel(self) -> str:
        """The kernel the last sieve launch ran ("k_wsieve" or "k_sieve")."""
        return N.lib().cgpu_last_sieve_kernel(self._ctx).decode()

    def launch_count(self) -> int:
        n = C.c_uint32()
        N.check(N.lib().cgpu_last_launch_count(self._ctx, C.byref(n)))
        return n.value

    def classify(self, pq) -> np.ndarray:
        """First-killer rank per (p, q) (-1 = survives every table)."""
        a = np.ascontiguousarray(pq, dtype=np.uint64).reshape(-1, 2)
        out = np.zeros(max(len(a), 1), np.int32)
        N.check(N.lib().cgpu_classify(self._ctx, _ptr(a), len(a), _ptr(out)))
        return out[: len(a)]


def serialize_index(primes) -> bytes:
    """CUPQ v1 index bytes (serialize_index, sievetable.hpp:231-252). Host-only."""
    pr = np.ascontiguousarray(primes, dtype=np.uint32)
    n = C.c_uint64()
    N.check(N.lib().cgpu_index_serialize(_ptr(pr), len(pr), None, 0, C.byref(n)))
    out = np.zeros(n.value, np.uint8)
    N.check(N.lib().cgpu_index_serialize(_ptr(pr), len(pr), _ptr(out), n.value, C.byref(n)))
    return out.tobytes()


def parse_index(index: bytes):
    """Validates like load_sieve (sievetable.hpp:254-292); returns (primes,
    tables stream length). Raises CudaSieveError(ERR_FORMAT) on a bad index."""
    buf = np.frombuffer(index, np.uint8) if len(index) else np.zeros(1, np.uint8)
    n, total = C.c_uint32(), C.c_uint64()
    N.check(N.lib().cgpu_index_parse(_ptr(buf), len(index), None, 0, C.byref(n), C.byref(total)))
    pr = np.zeros(max(n.value, 1), np.uint32)
    N.check(N.lib().cgpu_index_parse(_ptr(buf), len(index), _ptr(pr), n.value, C.byref(n),
                                     C.byref(total)))
    return [int(x) for x in pr[: n.value]], total.value


def q_bounds(p: int):
    lo, hi = C.c_uint64(), C.c_uint64()
    N.check(N.lib().cgpu_q_bounds(int(p), C.byref(lo), C.byref(hi)))
    return lo.value, hi.value
