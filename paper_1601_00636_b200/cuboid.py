"""Host-side mirror of the reference's hot-path API, running on the B200.

Same names, argument meaning and error behaviour as the reference's header-only
C++ API (paths relative to /root/reference/proj/include/cuboid):

    build_table(r)                     sievetable.hpp:123-141
    SieveSet.build(primes)             sievetable.hpp:159-176
    SieveSet.build_default()           sievetable.hpp:178-179
    SieveSet.is_unsolvable(rank,p,q)   sievetable.hpp:199-205
    scan(set, start, p_end, sink, opt) engine.hpp:195-295
    ScanStats (+ merge)                engine.hpp:105-135
    ScanEvent / ScanSink               engine.hpp:97-103
    ScanOptions                        engine.hpp:144-149
    ScanRejected(code)                 engine.hpp:163-167
    q_bounds(p)                        region.hpp:49-63

Every table build and every sieve runs in libcuboid_gpu.so (sm_100a) through
the C ABI of include/cuboid_gpu.h; there is no CPU fallback. The exact final
check of survivors (verify_pair, engine.hpp:66-95, GMP) stays on the CPU in
the reference; pass it as `verifier` to have each ScanEvent carry its verdict,
exactly as scan() does when a sink is set (engine.hpp:272-277).
"""
from __future__ import annotations

import ctypes as C
import itertools
import time
from dataclasses import dataclass, field
from typing import Callable, Optional

import numpy as np

from . import _native as N
from .device import Device, parse_index, q_bounds as _q_bounds, serialize_index as _serialize_index
from .primes import default_primes

MODULUS_LIMIT = 9697                  # primes.hpp:12
REGION_CROSSOVER = 152                # region.hpp:41
P_LIMIT_32BIT = ((1 << 32) - 1) // 59  # region.hpp:43-44: 59p < 2^32
P_LIMIT_64BIT = ((1 << 64) - 1) // 59


class ScanRejected(RuntimeError):
    """engine.hpp:163-167; code in {2,3,4,5,6} (engine.hpp:5-12)."""

    def __init__(self, code: int):
        super().__init__(f"scan rejected with code {code}")
        self.code = code


class FormatError(ValueError):
    """sievetable.hpp:37-39."""


_devices: dict[int, Device] = {}


def device(index: int = 0) -> Device:
    """The process's context on GPU `index` (one process per GPU)."""
    d = _devices.get(index)
    if d is None:
        d = _devices[index] = Device(index)
    return d


def q_bounds(p: int):
    """(q_low, q_high) of row p (region.hpp:49-63)."""
    return _q_bounds(p)


@dataclass
class BitTable:
    """sievetable.hpp:46-55: r and ceil(r^2/8) LSB-first bytes."""
    r: int
    bytes: bytes

    def bit(self, p: int, q: int) -> bool:
        i = p * self.r + q
        return bool((self.bytes[i >> 3] >> (i & 7)) & 1)


def build_table(r: int, dev: int = 0) -> BitTable:
    """One table, built on the GPU (replaces build_table, sievetable.hpp:123-141).
    ValueError (std::invalid_argument) for a modulus that is not a prime < 9697."""
    d = device(dev)
    d._owner = None  # the build replaces the resident tables
    try:
        tb, _ = d.build([r], N.BUILD_PRODUCTION)
    except N.CudaSieveError as e:
        if e.code == N.ERR_INVALID:
            raise ValueError("bit table modulus must be a prime below 9697") from e
        raise
    return BitTable(r, tb)


_SET_SERIALS = itertools.count(1)


class SieveSet:
    """Concatenated tables + prime index, resident on one GPU (sievetable.hpp:151-227)."""

    def __init__(self, primes, tables: bytes, offsets, dev: int):
        self._primes = [int(x) for x in primes]
        self._tables = tables
        self._offsets = [int(x) for x in offsets]
        self._dev = dev
        # residency token: unique per set for the process lifetime (an id()
        # can be reused by a later set once this one is collected)
        self._serial = next(_SET_SERIALS)

    # -- construction ------------------------------------------------------
    @classmethod
    def build(cls, primes, dev: int = 0, algorithm: int = N.BUILD_PRODUCTION) -> "SieveSet":
        """SieveSet::build (sievetable.hpp:159-176): ValueError for an unordered
        or non-prime list (std::invalid_argument), OverflowError past 2^32 bytes."""
        primes = [int(x) for x in primes]
        d = device(dev)
        d._owner = None
        try:
            tb, _ = d.build(primes, algorithm)
        except N.CudaSieveError as e:
            if e.code == N.ERR_INVALID:
                raise ValueError(str(e)) from e
            if e.code == N.ERR_OVERFLOW:
                raise OverflowError(str(e)) from e
            raise
        s = cls(primes, tb, d.offsets, dev)
        d._owner = s._serial
        return s

    @classmethod
    def build_default(cls, dev: int = 0) -> "SieveSet":
        return cls.build(default_primes(), dev)

    @classmethod
    def from_parts(cls, primes, tables: bytes, dev: int = 0) -> "SieveSet":
        """Reference-format bytes (load_sieve, sievetable.hpp:254-292) made resident.
        FormatError for a length mismatch or nonzero padding bits."""
        primes = [int(x) for x in primes]
        d = device(dev)
        d._owner = None
        try:
            d.load(primes, tables)
        except N.CudaSieveError as e:
            if e.code in (N.ERR_FORMAT, N.ERR_INVALID):
                raise FormatError(str(e)) from e
            raise
        s = cls(primes, bytes(tables), d.offsets, dev)
        d._owner = s._serial
        return s

    # -- queries (sievetable.hpp:181-205) ----------------------------------
    def empty(self) -> bool:
        return not self._primes

    def prime_count(self) -> int:
        return len(self._primes)

    def prime_at(self, rank: int) -> int:
        if not 0 <= rank < len(self._primes):
            raise IndexError("rank out of range")
        return self._primes[rank]

    def primes(self):
        return list(self._primes)

    def index(self):
        return list(zip(self._primes, self._offsets))

    def tables(self) -> bytes:
        return self._tables

    def rank_of(self, r: int):
        return self._primes.index(r) if r in self._primes else None

    def table_at(self, rank: int) -> BitTable:
        r = self.prime_at(rank)
        o = self._offsets[rank]
        return BitTable(r, self._tables[o:o + (r * r + 7) // 8])

    def is_unsolvable(self, rank: int, p: int, q: int) -> bool:
        r = self.prime_at(rank)
        i = (p % r) * r + (q % r)
        return bool((self._tables[self._offsets[rank] + (i >> 3)] >> (i & 7)) & 1)

    # -- on-disk formats (sievetable.hpp:229-346) ---------------------------
    def serialize_index(self) -> bytes:
        return serialize_index(self)

    def save_files(self, tables_path: str, index_path: str) -> None:
        """save_sieve_files: the device-resident bytes, written through the C ABI."""
        self.resident().save_files(tables_path, index_path)

    @classmethod
    def load_files(cls, tables_path: str, index_path: str, dev: int = 0) -> "SieveSet":
        """load_sieve_files straight onto the device (FormatError on a bad pair)."""
        d = device(dev)
        d._owner = None
        try:
            d.load_files(tables_path, index_path)
        except N.CudaSieveError as e:
            if e.code in (N.ERR_FORMAT, N.ERR_INVALID):
                raise FormatError(str(e)) from e
            if e.code == N.ERR_IO:
                raise OSError(str(e)) from e
            raise
        s = cls(d.primes, d.download(), d.offsets, dev)
        d._owner = s._serial
        return s

    # -- device residency --------------------------------------------------
    def resident(self) -> Device:
        """The device context with this set loaded (re-uploads if another set
        was made resident on the same GPU since)."""
        d = device(self._dev)
        if getattr(d, "_owner", None) != self._serial:
            d._owner = None
            d.load(self._primes, self._tables)
            d._owner = self._serial
        return d


def serialize_index(set_: "SieveSet") -> bytes:
    """serialize_index (sievetable.hpp:231-252)."""
    return _serialize_index(set_.primes())


def dump_table_text(set_: "SieveSet", r: int) -> str:
    """Text rendering of one table, rows by p residue (sievetable.hpp:296-311)."""
    rank = set_.rank_of(r)
    if rank is None:
        raise ValueError("dump_table_text: prime not in set")
    t = set_.table_at(rank)
    lines = [f"r={r}"]
    for p in range(r):
        lines.append(f"{p}: " + "".join("1" if t.bit(p, q) else "0" for q in range(r)))
    return "\n".join(lines) + "\n"


def serialize_tables(set_: "SieveSet") -> bytes:
    """serialize_tables (sievetable.hpp:229)."""
    return set_.tables()


def load_sieve(tables: bytes, index: bytes, dev: int = 0) -> "SieveSet":
    """load_sieve (sievetable.hpp:254-292): validates the index, then makes the
    set resident. FormatError on any violation."""
    try:
        primes, total = parse_index(index)
    except N.CudaSieveError as e:
        raise FormatError(str(e)) from e
    if len(tables) != total:
        raise FormatError("load_sieve: tables stream length does not match index")
    return SieveSet.from_parts(primes, tables, dev)


@dataclass
class ScanOptions:
    """engine.hpp:144-149. `stop` stands for hooks.stop: a bool, an object with
    is_set(), or a callable. The reference polls it every batch_pairs q
    visited and halts AT that q (engine.hpp:248-257). A scan with a stop hook
    runs as device tiles ending at such poll points; a watcher thread mirrors
    the hook into a mapped host word the kernels poll, so a tile running when
    it rises is abandoned and the scan halts at the next poll point after the
    tile's start -- a stop the reference makes when its flag becomes visible
    between those polls. Raised before the scan: the batch_pairs-th q, like
    the reference (or no stop at all if fewer q remain)."""
    small_p: bool = False
    p_limit: int = P_LIMIT_32BIT
    batch_pairs: int = 1 << 16
    stop: object = None

    def stop_requested(self) -> bool:
        s = self.stop
        if s is None:
            return False
        if hasattr(s, "is_set"):
            return bool(s.is_set())
        return bool(s() if callable(s) else s)


def region_advance(pos, k: int, p_end: int):
    """The pair k steps after pos in scan()'s q visiting order (every q of the
    region rows, engine.hpp:225-248), or None if row p_end ends first
    (cgpu_region_advance: host code, O(rows))."""
    op, oq = C.c_uint64(), C.c_uint64()
    rc = N.lib().cgpu_region_advance(int(pos[0]), int(pos[1]), int(k), int(p_end), C.byref(op), C.byref(oq))
    if rc == N.P_ABOVE_LIMIT:
        return None
    N.check(rc)
    return op.value, oq.value


STOP_TILE_PAIRS = 1 << 37  # q visited per stoppable tile (~20 ms on one B200)


class _StopMirror:
    """Mirrors a ScanOptions stop hook into a mapped host word that the sieve
    kernels of one context poll (cgpu_set_stop_word)."""

    def __init__(self, ctx, opt):
        import threading
        self.ctx, self.opt = ctx, opt
        w = C.c_void_p()
        N.check(N.lib().cgpu_alloc_stop_word(C.byref(w)))
        self.word = w.value
        self.cell = C.c_uint32.from_address(self.word)
        N.check(N.lib().cgpu_set_stop_word(ctx, C.c_void_p(self.word)))
        if opt.stop_requested():
            self.cell.value = 1
        self.done = threading.Event()
        self.t = threading.Thread(target=self._watch, daemon=True)
        self.t.start()

    def _watch(self):
        while not self.done.is_set():
            if self.opt.stop_requested():
                self.cell.value = 1
                return
            self.done.wait(50e-6)

    def raised(self) -> bool:
        return self.cell.value != 0

    def disarm(self):
        if not self.done.is_set():
            self.done.set()
            self.t.join()
            N.check(N.lib().cgpu_set_stop_word(self.ctx, None))

    def close(self):
        self.disarm()
        N.lib().cgpu_free_stop_word(C.c_void_p(self.word))


def stop_point(start, p_end: int, batch_pairs: int):
    """The (p, q) at which a scan with a raised stop flag halts: the
    batch_pairs-th q visited from `start`, counting every q of the region rows
    (skipped pairs included, engine.hpp:248-257); None if the range ends first."""
    k = max(int(batch_pairs), 1)
    p, q = int(start[0]), int(start[1])
    first = True
    while p <= p_end:
        lo, hi = q_bounds(p)
        q0 = q if first else lo
        first = False
        n = hi - q0 + 1 if hi >= q0 else 0
        if k <= n:
            return p, q0 + k - 1
        k -= n
        p += 1
    return None


@dataclass
class ScanEvent:
    p: int
    q: int
    verdict: object = None


@dataclass
class ScanStats:
    """engine.hpp:105-135."""
    pairs_tested: int = 0
    survivors: int = 0
    kill_histogram: dict = field(default_factory=dict)   # prime -> first-kill count
    block_r_max: dict = field(default_factory=dict)      # p // 100 -> max killing prime, 1 if none
    elapsed: float = 0.0                                 # seconds
    resume_p: int = 0
    resume_q: int = 0
    stopped: bool = False
    survivor_pairs: list = field(default_factory=list)   # [(p, q)] ascending

    def histogram_total(self) -> int:
        return sum(self.kill_histogram.values())

    def merge(self, o: "ScanStats") -> None:
        self.pairs_tested += o.pairs_tested
        self.survivors += o.survivors
        for r, k in o.kill_histogram.items():
            self.kill_histogram[r] = self.kill_histogram.get(r, 0) + k
        for b, r in o.block_r_max.items():
            if r > self.block_r_max.get(b, 0):
                self.block_r_max[b] = r
        self.elapsed += o.elapsed
        self.resume_p, self.resume_q, self.stopped = o.resume_p, o.resume_q, o.stopped
        self.survivor_pairs = sorted(self.survivor_pairs + o.survivor_pairs)


def validate_start(loaded: bool, p: int, q: int, opt: ScanOptions) -> int:
    """engine.hpp:152-161."""
    if not loaded:
        return 6
    if p < REGION_CROSSOVER and not opt.small_p:
        return 2
    if p > opt.p_limit or p == 0:
        return 3
    lo, hi = q_bounds(p)
    if q < lo:
        return 4
    if q > hi:
        return 5
    return 0


def _next_pair(p_end: int):
    """Resume point after the last row (engine.hpp:178-187)."""
    np_ = p_end + 1
    return np_, (q_bounds(np_)[0] if np_ <= P_LIMIT_64BIT else 1)


def stats_from_result(set_: SieveSet, res, with_survivors=True) -> ScanStats:
    st = ScanStats()
    st.pairs_tested = res.pairs_tested
    st.survivors = res.survivors
    st.kill_histogram = {set_.prime_at(k): int(c) for k, c in enumerate(res.hist) if c}
    st.block_r_max = {res.block_lo + i: int(v) for i, v in enumerate(res.block_rmax) if v}
    if with_survivors:
        st.survivor_pairs = [(int(p), int(q)) for p, q in res.survivor_pairs]
    return st


def _run(set_: SieveSet, p_lo, q_start, p_hi, mode, shard, surv_cap):
    d = set_.resident()
    cap = surv_cap
    while True:
        try:
            return d.sieve(p_lo, p_hi, mode, q_start=q_start, shard=shard, surv_cap=cap)
        except N.CudaSieveError as e:
            if e.code != N.ERR_CAPACITY:
                raise
            cap = max(2 * cap, getattr(e, "survivors", 0) + 1)


def _span(set_: SieveSet, p0: int, q0: int, p_stop: int, q_stop: int) -> ScanStats:
    """REGION pairs from (p0, q0) up to, not including, (p_stop, q_stop)."""
    d = set_.resident()
    lo = q_bounds(p_stop)[0]
    first = q0 if p_stop == p0 else lo
    p_hi, q_end = p_stop, q_stop - 1
    if q_stop == first:  # the stop falls on the row's first pair: that row is not sieved
        p_hi, q_end = p_stop - 1, 0
    n = set_.prime_count()
    st = ScanStats()
    if p_hi >= p0:
        cap = 1 << 20
        while True:
            counts = np.zeros(2, np.uint64)
            hist = np.zeros(max(n, 1), np.uint64)
            nb = p_hi // 100 - p0 // 100 + 1
            brm = np.zeros(nb, np.uint32)
            spq = np.zeros((cap, 2), np.uint64)
            rc = N.lib().cgpu_sieve_span(d._ctx, p0, q0, p_hi, q_end, counts.ctypes.data_as(C.c_void_p),
                                         hist.ctypes.data_as(C.c_void_p), brm.ctypes.data_as(C.c_void_p),
                                         nb, spq.ctypes.data_as(C.c_void_p), cap)
            if rc == N.ERR_CAPACITY and int(counts[1]) > cap:
                cap = int(counts[1])
                continue
            N.check(rc)
            break
        st.pairs_tested, st.survivors = int(counts[0]), int(counts[1])
        st.kill_histogram = {set_.prime_at(k): int(c) for k, c in enumerate(hist[:n]) if c}
        st.block_r_max = {p0 // 100 + i: int(v) for i, v in enumerate(brm) if v}
        st.survivor_pairs = [(int(a), int(b)) for a, b in spq[: st.survivors]]
    st.block_r_max.setdefault(p_stop // 100, 1)  # the stop row's block is entered (engine.hpp:229-236)
    return st


def scan(set_: SieveSet, start, p_end: int, sink: Optional[Callable] = None,
         opt: Optional[ScanOptions] = None, verifier: Optional[Callable] = None,
         shard=(1, 0), surv_cap: int = 1 << 20) -> ScanStats:
    """The reference scan() (engine.hpp:195-295) on the GPU: REGION rows
    q_low(p) <= q <= 59p from start=(p, q) through p_end. Survivors are handed
    to `sink` in ascending (p, q) order as ScanEvent(p, q, verifier(p, q))."""
    opt = opt or ScanOptions()
    p0, q0 = int(start[0]), int(start[1])
    if set_.empty():
        raise ScanRejected(6)
    code = validate_start(True, p0, q0, opt)
    if code:
        raise ScanRejected(code)
    if p_end > opt.p_limit:
        raise ScanRejected(3)
    t0 = time.perf_counter()
    st = ScanStats(resume_p=p0, resume_q=q0)
    if opt.stop is not None and p0 <= p_end and shard == (1, 0):
        st = _scan_stoppable(set_, (p0, q0), p_end, opt, surv_cap)
    elif p0 <= p_end:
        res = _run(set_, p0, q0, p_end, N.REGION, shard, surv_cap)
        st = stats_from_result(set_, res)
        st.resume_p, st.resume_q = _next_pair(p_end)
    st.elapsed = time.perf_counter() - t0
    if sink is not None:
        for p, q in st.survivor_pairs:
            sink(ScanEvent(p, q, verifier(p, q) if verifier else None))
    return st


def _scan_stoppable(set_: SieveSet, start, p_end: int, opt: ScanOptions, surv_cap: int) -> ScanStats:
    """scan() with a stop hook: tiles that end at poll points (every
    batch_pairs-th q visited), the hook mirrored into the kernels' stop word
    (include/cuboid/gpu.hpp scan_on is the C++ twin)."""
    B = max(int(opt.batch_pairs), 1)
    K = max(1, STOP_TILE_PAIRS // B)
    d = set_.resident()
    mirror = _StopMirror(d._ctx, opt)
    st = ScanStats()
    pos, at_poll = (int(start[0]), int(start[1])), False

    def to_end(p, q):
        res = _run(set_, p, q, p_end, N.REGION, (1, 0), surv_cap)
        st.merge(stats_from_result(set_, res))
        st.resume_p, st.resume_q = _next_pair(p_end)

    def halt_at(at):
        st.merge(_span(set_, pos[0], pos[1], at[0], at[1]))
        st.block_r_max.setdefault(at[0] // 100, 1)
        st.resume_p, st.resume_q, st.stopped = at[0], at[1], True

    try:
        while True:
            if at_poll and opt.stop_requested():  # the reference's poll at pos
                halt_at(pos)
                break
            to = region_advance(pos, K * B if at_poll else K * B - 1, p_end)
            if to is not None:
                part = _span(set_, pos[0], pos[1], to[0], to[1])
            else:
                part = stats_from_result(set_, _run(set_, pos[0], pos[1], p_end, N.REGION, (1, 0), surv_cap))
            if mirror.raised():  # the tile may have been abandoned: the next poll point instead
                mirror.disarm()
                nxt = region_advance(pos, B if at_poll else B - 1, p_end)
                if nxt is not None:
                    halt_at(nxt)
                else:
                    to_end(*pos)
                break
            st.merge(part)
            if to is None:
                st.resume_p, st.resume_q = _next_pair(p_end)
                break
            pos, at_poll = to, True
            st.resume_p, st.resume_q = pos
    finally:
        mirror.close()
    return st


def scan_triangle(set_: SieveSet, p_lo: int, p_hi: int, sink: Optional[Callable] = None,
                  verifier: Optional[Callable] = None, shard=(1, 0),
                  surv_cap: int = 1 << 20) -> ScanStats:
    """TRIANGLE rows 1 <= q < p for p in [p_lo, p_hi] (the BASELINE configs;
    the loop of verify_small_region, engine.hpp:613-625, over q < p)."""
    if set_.empty():
        raise ScanRejected(6)
    if p_lo < 1 or p_hi >= 1 << 32:
        raise ScanRejected(3)
    t0 = time.perf_counter()
    st = ScanStats(resume_p=p_lo, resume_q=1)
    if p_lo <= p_hi:
        res = _run(set_, p_lo, 0, p_hi, N.TRIANGLE, shard, surv_cap)
        st = stats_from_result(set_, res)
        st.resume_p, st.resume_q = p_hi + 1, 1
    st.elapsed = time.perf_counter() - t0
    if sink is not None:
        for p, q in st.survivor_pairs:
            sink(ScanEvent(p, q, verifier(p, q) if verifier else None))
    return st


@dataclass
class SmallRegionSummary:
    """engine.hpp:597-604."""
    pairs: int = 0
    sieved_out: int = 0
    survivors: int = 0
    no_integer_root: int = 0
    root_fails: int = 0
    candidates: int = 0


def verify_small_region(set_: SieveSet, verifier: Callable) -> SmallRegionSummary:
    """verify_small_region (engine.hpp:609-640): every coprime p != q pair of
    the region rows p <= 151, sieved on the GPU; every survivor goes to
    `verifier` (p, q) -> "NoIntegerRoot" | "RootFailsInequalities" |
    "CuboidCandidate" -- the reference's exact check, verify_pair(bypass)
    (engine.hpp:626-635). There is no default: without the exact check the
    survivors are unverified, so a missing verifier raises (TypeError) instead
    of reporting them as NoIntegerRoot. A candidate raises, as in the
    reference."""
    if verifier is None or not callable(verifier):
        raise TypeError("verify_small_region needs the exact final check (verifier)")
    if set_.empty():
        raise ValueError("verify_small_region: empty sieve set")
    st = scan(set_, (1, 1), 151, opt=ScanOptions(small_p=True))
    out = SmallRegionSummary(pairs=st.pairs_tested, sieved_out=st.pairs_tested - st.survivors,
                             survivors=st.survivors)
    for p, q in st.survivor_pairs:
        kind = verifier(p, q)
        if kind == "CuboidCandidate":
            out.candidates += 1
            raise RuntimeError(f"cuboid candidate found at p={p}, q={q}")
        if kind == "RootFailsInequalities":
            out.root_fails += 1
        elif kind == "NoIntegerRoot":
            out.no_integer_root += 1
        else:
            raise ValueError(f"verifier returned an unknown verdict {kind!r} for ({p}, {q})")
    return out


def classify(set_: SieveSet, pairs) -> np.ndarray:
    """First-killer rank per (p, q), -1 if no table rejects it (the sieve part
    of verify_pair, engine.hpp:72-78)."""
    return set_.resident().classify(pairs)
