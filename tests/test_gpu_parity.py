"""Parity of the B200 path (libcuboid_gpu.so through the C ABI) with the
reference: golden fixtures made by the unmodified reference (tests/golden/),
the C oracle (oracle/cuboid_oracle.c) on seeded inputs, and size-independent
properties at the BASELINE sizes. Everything is integer work: the bar is
bit-exact equality of tables, pair counts, first-killer histograms, block
r_max and survivor lists."""
from __future__ import annotations

import ctypes as C
import hashlib
import random

import numpy as np
import pytest

from oracle import port
from oracle import ref as refmod
from paper_1601_00636_b200 import _native as N
from paper_1601_00636_b200 import cuboid
from paper_1601_00636_b200.device import Device, serialize_index as device_serialize_index
from paper_1601_00636_b200.primes import default_primes, odd_primes, primes_in_range

pytestmark = pytest.mark.gpu


def sha(b: bytes) -> str:
    return hashlib.sha256(b).hexdigest()


@pytest.fixture(scope="module")
def dev():
    d = Device(0)
    yield d
    d.close()


def phi_sum(lo, hi):
    """sum of Euler phi(p) for p in [lo, hi] = TRIANGLE candidate count."""
    n = hi + 1
    phi = np.arange(n, dtype=np.int64)
    for p in range(2, n):
        if phi[p] == p:
            phi[p::p] -= phi[p::p] // p
    return int(phi[max(lo, 2):n].sum())


# ---- K1: tables ---------------------------------------------------------------------

@pytest.mark.parametrize("name", ["odd32", "odd64", "odd128", "odd256", "default96"])
@pytest.mark.parametrize("alg", [N.BUILD_PRODUCTION, N.BUILD_EXHAUSTIVE])
def test_tables_identical_to_reference(dev, golden, sets, name, alg):
    P = sets[name]
    tb, evals = dev.build(P, alg)
    g = golden["tables"][name]
    assert len(tb) == g["bytes"]
    if sha(tb) != g["sha256"]:  # name the first differing prime
        for k, h in enumerate(g["per_table_sha256"]):
            o = int(dev.offsets[k])
            assert sha(tb[o:o + (P[k] ** 2 + 7) // 8]) == h, f"table r={P[k]} differs"
    assert sha(tb) == g["sha256"]
    if alg == N.BUILD_EXHAUSTIVE:
        assert evals == sum(r ** 3 for r in P)
    else:
        assert 0 < evals <= sum(r * (r // 2 + 1) for r in P)


def test_single_tables_vs_oracle(dev):
    """test_sievetable.cpp:12-56: U_11 bytes, zero tables for r <= 7, and every
    r <= 97 (plus large ones) equal to the definition/production oracle."""
    assert cuboid.build_table(11).bytes == bytes.fromhex("00E09F7EEDED76CF7BDEEDF6D62FFF00")
    for r in (2, 3, 5, 7):
        assert cuboid.build_table(r).bytes == bytes((r * r + 7) // 8)
    for r in primes_in_range(2, 97) + [541, 1021, 2039, 2053, 4099, 9689]:
        for alg in (N.BUILD_PRODUCTION, N.BUILD_EXHAUSTIVE) if r < 2100 else (N.BUILD_PRODUCTION,):
            tb, _ = dev.build([r], alg)
            assert tb == port.build_table(r), (r, alg)


def test_exhaustive_mixed_paths(dev):
    """One exhaustive build whose primes take every k_cube path at once: r = 2
    and r > 2039 on the IMAD kernel, odd r <= 2039 on the FFMA2 kernel (the
    boundary primes 2039 and 2053 on either side)."""
    P = [2, 3, 13, 1621, 2039, 2053]
    tb, evals = dev.build(P, N.BUILD_EXHAUSTIVE)
    assert evals == sum(r ** 3 for r in P)
    want, _ = port.build_set(P)
    assert tb == want


@pytest.mark.parametrize("r", [0, 1, 4, 9697, 10007])
def test_bad_modulus(r):
    with pytest.raises(ValueError):
        cuboid.build_table(r)


def test_bad_prime_lists():
    with pytest.raises(ValueError):
        cuboid.SieveSet.build([13, 11])
    with pytest.raises(ValueError):
        cuboid.SieveSet.build([11, 15])


def test_load_download_roundtrip_and_format_errors(dev, sets):
    P = sets["default96"]
    tb, _ = port.build_set(P)
    dev.load(P, tb)
    assert dev.download() == tb
    assert dev.killable().all()
    bad = bytearray(tb)
    bad[(11 * 11 + 7) // 8 - 1] |= 0x80  # padding bit of the r = 11 table
    with pytest.raises(cuboid.FormatError):
        cuboid.SieveSet.from_parts(P, bytes(bad))
    with pytest.raises(cuboid.FormatError):
        cuboid.SieveSet.from_parts(P, tb[:-1])
    s = cuboid.SieveSet.from_parts(odd_primes(8), port.build_set(odd_primes(8))[0])
    assert s.resident().killable().tolist() == [False, False, False, True, True, True, True, True]


# ---- K2: sieve against the reference's own results ---------------------------------------

def _check(st: cuboid.ScanStats, g, primes):
    assert st.pairs_tested == g["pairs_tested"]
    assert st.survivors == g["survivors"]
    assert {str(k): v for k, v in st.kill_histogram.items()} == g["kill_histogram"]
    assert {str(k): v for k, v in st.block_r_max.items()} == g["block_r_max"]
    if "survivor_sha256" in g:
        flat = ",".join(f"{p}:{q}" for p, q in st.survivor_pairs)
        assert sha(flat.encode()) == g["survivor_sha256"]
    if "resume" in g:
        assert [st.resume_p, st.resume_q] == g["resume"]


_built = {}


def _set(sets, name):
    if name not in _built:
        _built.clear()  # one resident set at a time keeps device memory small
        _built[name] = cuboid.SieveSet.build(sets[name])
    return _built[name]


@pytest.mark.parametrize("name", ["C1", "C3", "C5_sub", "C4", "R152", "R152_300", "R152_2000",
                                  "R152_5000", "R153_5000tail", "W_row1", "W_1_40", "W_T300",
                                  "R1_151"])
def test_sieve_identical_to_reference(golden, sets, name):
    g = golden["sieve"][name]
    s = _set(sets, g["set"])
    if g["mode"] == "TRIANGLE":
        st = cuboid.scan_triangle(s, g["p_lo"], g["p_hi"])
    else:
        st = cuboid.scan(s, (g["p_lo"], g["q_start"]), g["p_hi"],
                         opt=cuboid.ScanOptions(small_p=g["p_lo"] < 152))
    _check(st, g, sets[g["set"]])


def test_region_pins():
    """test_engine.cpp:71-88, 199-205 and acceptance.cpp:123-144 on the default set."""
    s = cuboid.SieveSet.build_default()
    st = cuboid.scan(s, (152, 3), 152)
    assert (st.pairs_tested, st.survivors, max(st.kill_histogram)) == (4247, 0, 47)
    assert (st.resume_p, st.resume_q) == (153, cuboid.q_bounds(153)[0])
    st = cuboid.scan(s, (152, 3), 300)
    assert st.survivors == 0 and max(st.kill_histogram) <= 137 and len(st.block_r_max) == 3
    st = cuboid.scan(s, (152, 3), 5000)
    assert (st.pairs_tested, st.survivors, max(st.kill_histogram)) == (447994938, 0, 97)


def test_scan_rejections():
    """ScanRejected codes (engine.hpp:152-161, 195-201; test_engine.cpp:90-122)."""
    s = cuboid.SieveSet.build_default()
    for start, p_end, code in [((151, 3), 200, 2), ((0, 1), 10, 2), ((72796056, 10**6), 72796056, 3),
                               ((152, 2), 200, 4), ((152, 59 * 152 + 1), 200, 5),
                               ((152, 3), 72796056, 3)]:
        with pytest.raises(cuboid.ScanRejected) as e:
            cuboid.scan(s, start, p_end)
        assert e.value.code == code, (start, p_end)
    with pytest.raises(cuboid.ScanRejected) as e:
        cuboid.scan(cuboid.SieveSet([], b"", [], 0), (152, 3), 200)
    assert e.value.code == 6


def test_empty_range():
    s = cuboid.SieveSet.build_default()
    st = cuboid.scan(s, (500, 4), 499)
    assert (st.pairs_tested, st.survivors, st.kill_histogram, st.block_r_max) == (0, 0, {}, {})
    assert (st.resume_p, st.resume_q) == (500, 4)


@pytest.mark.parametrize("seed", [1, 2, 3])
def test_random_ranges_vs_oracle(dev, seed):
    """Seeded row ranges, both modes, mid-row starts, several prime sets
    (including all-zero tables that never kill and a heavy-survivor set)."""
    rng = random.Random(seed)
    for P in (odd_primes(32), default_primes(), [11], [11, 13], [3, 5, 7], odd_primes(200)[150:]):
        tb, offs = port.build_set(P)
        dev.load(P, tb)
        for _ in range(3):
            mode = rng.choice([N.TRIANGLE, N.REGION])
            lo = rng.randrange(1, 4000)
            hi = lo + rng.choice([0, 1, 7, 99, 250] if mode == N.TRIANGLE else [0, 1, 7])
            q0 = 0
            if mode == N.REGION and rng.random() < 0.5:
                q0 = rng.randrange(*cuboid.q_bounds(lo))
            o = port.sieve(tb, P, offs, lo, hi, mode, q_start=q0)
            r = dev.sieve(lo, hi, mode, q_start=q0, surv_cap=1 << 22)
            assert r.pairs_tested == o["pairs_tested"], (P[:3], mode, lo, hi, q0)
            assert r.survivors == o["survivors"]
            assert r.hist.tolist() == o["hist"].tolist()
            assert np.array_equal(r.survivor_pairs, o["survivor_pairs"])
            rows = np.asarray(o["row_rmax"])
            want = {}
            for i, v in enumerate(rows):
                b = (lo + i) // 100
                want[b] = max(want.get(b, 0), int(v))
            got = {r.block_lo + i: int(v) for i, v in enumerate(r.block_rmax) if v}
            assert got == want


@pytest.mark.parametrize("prime,flip", [(11, (2, 5)), (13, (0, 4)), (13, (7, 12)), (11, (0, 3))])
def test_non_canonical_tables_vs_oracle(dev, prime, flip):
    """Tables loaded from bytes the reference's builder would never produce
    (one flipped bit of a row a >= 1, which breaks u(la, lb) = u(a, b), or of
    row 0) must still sieve exactly like the reference itself (oracle/_ref,
    the reference headers loaded with the same bytes): REGION never probes row
    0 (scan(), engine.hpp:240-242), TRIANGLE reads it like any other row (the
    is_unsolvable loop, sievetable.hpp:199-205) -- the context re-derives
    its layout when a set with bits in row 0 switches mode."""
    P = odd_primes(96)
    tb, offs = port.build_set(P)
    k = P.index(prime)
    a, b = flip
    i = a * prime + b
    bad = bytearray(tb)
    bad[int(offs[k]) + (i >> 3)] ^= 1 << (i & 7)
    bad = bytes(bad)
    dev.load(P, bad)
    rset = refmod.RefSet.load(bad, device_serialize_index(P))
    for lo, hi, mode in ((2, 3000, N.TRIANGLE), (152, 700, N.REGION), (2, 1500, N.TRIANGLE)):
        o = port.sieve(bad, P, offs, lo, hi, mode)
        r = dev.sieve(lo, hi, mode, surv_cap=1 << 22)
        assert (r.pairs_tested, r.survivors) == (o["pairs_tested"], o["survivors"])
        assert r.hist.tolist() == o["hist"].tolist()
        assert np.array_equal(r.survivor_pairs, o["survivor_pairs"])
        if mode == N.TRIANGLE:
            w = refmod.triangle(rset, lo, hi, 4, with_sink=True)
        else:
            w = refmod.scan(rset, lo, 3, hi, with_sink=True)
        assert (r.pairs_tested, r.survivors) == (w.pairs_tested, w.survivors)
        assert r.hist.tolist() == list(w.hist_by_rank)
        assert [tuple(x) for x in r.survivor_pairs.tolist()] == [(p, q) for p, q, _ in w.survivor_pairs]


REG_LAYOUTS = [
    # (prime set, CUBOID_REG3_PROBES, CUBOID_NO_STD_PRIMES): every register /
    # window-table probe layout the context can choose (capi.cu finalize_set)
    (odd_primes(96), None, None),                                    # standard 11..37 (immediates)
    (odd_primes(96), None, "1"),                                     # same primes, generic kernel
    (odd_primes(96), "0", None),                                     # no 3-word probe
    (odd_primes(96), "2", None),                                     # 37 table + 41 funnel probe
    (odd_primes(96), "4", None),                                     # 37 table + 41, 43, 47 funnel
    (primes_in_range(11, 31) + primes_in_range(61, 400), None, None),  # generic 3-word table r = 61
    (primes_in_range(11, 31) + primes_in_range(59, 400), "3", None),   # 59 table + 61 funnel (67 > 63)
    (primes_in_range(13, 400), None, None),                          # 11 absent: two-word probes only
    ([11] + primes_in_range(37, 400), None, None),                   # one register probe
    (primes_in_range(67, 500), None, None),                          # no register probes
]


@pytest.mark.parametrize("case", range(len(REG_LAYOUTS)))
def test_register_probe_layouts_vs_oracle(dev, case, monkeypatch):
    """Each register-probe layout (window-table probes, funnel probes, the
    standard-prime instantiation, no register probes) against the oracle."""
    P, reg3, nostd = REG_LAYOUTS[case]
    for k, v in (("CUBOID_REG3_PROBES", reg3), ("CUBOID_NO_STD_PRIMES", nostd)):
        if v is None:
            monkeypatch.delenv(k, raising=False)
        else:
            monkeypatch.setenv(k, v)
    tb, offs = port.build_set(P)
    dev.load(P, tb)
    rng = random.Random(100 + case)
    for mode, lo, hi in ((N.TRIANGLE, 1, 1200), (N.TRIANGLE, rng.randrange(2000, 6000), None),
                         (N.REGION, rng.randrange(152, 3000), None)):
        hi = hi or lo + (60 if mode == N.TRIANGLE else 3)
        o = port.sieve(tb, P, offs, lo, hi, mode)
        r = dev.sieve(lo, hi, mode, surv_cap=1 << 22)
        assert r.pairs_tested == o["pairs_tested"], (case, mode, lo, hi)
        assert r.survivors == o["survivors"]
        assert r.hist.tolist() == o["hist"].tolist()
        assert np.array_equal(r.survivor_pairs, o["survivor_pairs"])


@pytest.mark.parametrize("row_cost,alpha", [("1", "0"), ("5000", "0"), ("800", "40"), ("50", "12")])
def test_load_balance_knobs_never_change_results(golden, sets, row_cost, alpha, monkeypatch):
    """The plan's work units (row setup charge, drain-aware window weights)
    only move rows between warps: extreme settings give the reference's C3
    result exactly, whole and as 3 block-cyclic shards."""
    monkeypatch.setenv("CUBOID_ROW_COST", row_cost)
    monkeypatch.setenv("CUBOID_DRAIN_ALPHA", alpha)
    d = Device(0)  # knobs are read when a context is created
    try:
        P = sets["odd64"]
        tb, _ = port.build_set(P)
        d.load(P, tb)
        g = golden["sieve"]["C3"]
        want = {str(k): v for k, v in g["kill_histogram"].items()}
        r = d.sieve(2, 10000, N.TRIANGLE)
        assert (r.pairs_tested, r.survivors) == (g["pairs_tested"], g["survivors"])
        assert {str(P[k]): int(c) for k, c in enumerate(r.hist) if c} == want
        hist = np.zeros(len(P), np.uint64)
        pairs = 0
        for k in range(3):
            x = d.sieve(2, 10000, N.TRIANGLE, shard=(3, k))
            hist += x.hist
            pairs += x.pairs_tested
        assert pairs == g["pairs_tested"]
        assert {str(P[k]): int(c) for k, c in enumerate(hist) if c} == want
    finally:
        d.close()


def test_heavy_survivor_compaction(dev):
    """Weak sieve {11} (test_engine.cpp:177-197) over C1's triangle: 405,546
    survivors, emitted in canonical ascending (p, q) order."""
    P = [11]
    tb, offs = port.build_set(P)
    dev.load(P, tb)
    o = port.sieve(tb, P, offs, 2, 2000, port.TRIANGLE)
    r = dev.sieve(2, 2000, N.TRIANGLE, surv_cap=1 << 20)
    assert r.survivors == o["survivors"] == 405546
    assert np.array_equal(r.survivor_pairs, o["survivor_pairs"])
    with pytest.raises(N.CudaSieveError) as e:
        dev.sieve(2, 2000, N.TRIANGLE, surv_cap=1000)
    assert e.value.code == N.ERR_CAPACITY and e.value.survivors == 405546


@pytest.mark.skipif(not refmod.available(), reason="oracle/_ref not built")
def test_survivors_reach_the_reference_final_check():
    """scan() hands each survivor to verify_pair(bypass) in order (engine.hpp:272-277)."""
    rs = refmod.RefSet.build([11])
    s = cuboid.SieveSet.build([11])
    events = []
    st = cuboid.scan(s, (1, 1), 1, sink=events.append, opt=cuboid.ScanOptions(small_p=True),
                     verifier=lambda p, q: refmod.verify_pair(rs, p, q, True)[0])
    ref = refmod.scan(rs, 1, 1, 1, small_p=True)
    assert [(e.p, e.q, e.verdict) for e in events] == ref.survivor_pairs
    assert st.survivors == len(events) > 0


# ---- multi-shard semantics (ScanStats::merge, test_engine.cpp:134-175) -----------------

@pytest.mark.parametrize("G", [2, 3, 8])
def test_block_cyclic_shards_merge_to_full(dev, golden, sets, G):
    g = golden["sieve"]["C3"]
    tb, _ = port.build_set(sets["odd64"])
    dev.load(sets["odd64"], tb)
    hist = np.zeros(64, np.uint64)
    pairs = surv = 0
    brm = {}
    for k in range(G):
        r = dev.sieve(2, 10000, N.TRIANGLE, shard=(G, k))
        pairs += r.pairs_tested
        surv += r.survivors
        hist += r.hist
        for i, v in enumerate(r.block_rmax):
            if v:
                assert (r.block_lo + i) % G == k  # each block lives on one shard
                brm[r.block_lo + i] = int(v)
    assert pairs == g["pairs_tested"] and surv == 0
    assert {str(sets["odd64"][k]): int(c) for k, c in enumerate(hist) if c} == g["kill_histogram"]
    assert {str(b): v for b, v in sorted(brm.items())} == g["block_r_max"]


# ---- BASELINE full sizes: size-independent properties ------------------------------------

def test_c5_full_range_vs_reference(dev, golden, sets):
    """C5, the headline config (10^5 < p <= 3*10^5, 256 primes, 2.43e10 pairs)
    over its WHOLE range against the reference's own result (golden C5 from
    oracle/_ref: engine.hpp:259-277 statistics with sievetable.hpp:199-205
    probes): pairs, survivors, the first-killer histogram and all 2001 block
    r_max values; plus 4-way block-cyclic shards merging to it."""
    s = _set(sets, "odd256")
    full = cuboid.scan_triangle(s, 100001, 300000)
    g = golden["sieve"]["C5"]
    assert (g["p_lo"], g["p_hi"], g["set"]) == (100001, 300000, "odd256")
    _check(full, g, sets["odd256"])
    assert full.pairs_tested == phi_sum(100001, 300000) == 24317097730
    merged = cuboid.ScanStats()
    for k in range(4):
        merged.merge(cuboid.scan_triangle(s, 100001, 300000, shard=(4, k)))
    _check(merged, g, sets["odd256"])
    sub = cuboid.scan_triangle(s, 200001, 201000)
    _check(sub, golden["sieve"]["C5_sub"], sets["odd256"])


def test_c4_random_subsample_classify(dev, golden, sets):
    """C4's seeded 10^6-pair subsample (p weighted by phi(p), q
    uniform among the coprime residues, tests/subsample.py): the first-killer
    rank of every pair from the device classify path equals the reference's
    rank-ordered SieveSet::is_unsolvable (golden C4_subsample, oracle/_ref)."""
    import subsample
    g = golden["sieve"]["C4_subsample"]
    P = sets["odd128"]
    tb, offs = port.build_set(P)
    dev.load(P, tb)
    pq = subsample.sample(g["n"], g["seed"], g["p_max"])
    assert hashlib.sha256(pq.tobytes()).hexdigest() == g["pairs_sha256"]
    got = dev.classify(pq).astype("<i4")
    assert hashlib.sha256(got.tobytes()).hexdigest() == g["ranks_sha256"]
    hist = np.bincount(got + 1, minlength=len(P) + 1)
    assert int(hist[0]) == g["survivors"]
    assert {str(P[k]): int(c) for k, c in enumerate(hist[1:]) if c} == g["rank_histogram"]


def test_sharded_sieve_single_rank(dev):
    """parallel.ShardedSieve (the multi-GPU product path) at world size 1."""
    from paper_1601_00636_b200.parallel import ShardedSieve
    P = [11, 13]
    tb, offs = port.build_set(P)
    dev.load(P, tb)
    s = ShardedSieve(dev, P)
    s.launch(2, 700)
    pairs, surv, hist, brm, sp = s.reduce()
    o = port.sieve(tb, P, offs, 2, 700, port.TRIANGLE)
    assert (pairs, surv) == (o["pairs_tested"], o["survivors"])
    assert hist.tolist() == o["hist"].astype(np.int64).tolist()
    assert np.array_equal(sp, o["survivor_pairs"])


def test_load_from_device_memory_and_nccl_sharded_upload(dev, golden, sets):
    """cgpu_tables_load_dev (tables already in device memory) and the N>1
    e2e upload path parallel.load_tables_sharded run through a real NCCL
    all-gather (world size 1 on this GPU): identical resident set, C3 result
    identical to the reference's; a bad padding bit is still a FormatError."""
    import os
    import socket
    import torch
    import torch.distributed as dist
    from paper_1601_00636_b200 import parallel
    P = sets["odd64"]
    tb, offs = port.build_set(P)
    d_tb = torch.frombuffer(bytearray(tb), dtype=torch.uint8).cuda()
    torch.cuda.synchronize()  # the context has its own stream: the bytes must be ready
    dev.load_dev(P, d_tb.data_ptr(), d_tb.numel())
    assert dev.download() == tb
    bad = d_tb.clone()
    k11 = list(P).index(11)
    bad[int(offs[k11]) + (11 * 11 + 7) // 8 - 1] |= 0x80  # a padding bit of the r = 11 table
    torch.cuda.synchronize()
    with pytest.raises(N.CudaSieveError):
        dev.load_dev(P, bad.data_ptr(), bad.numel())
    sk = socket.socket()
    sk.bind(("127.0.0.1", 0))
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(sk.getsockname()[1]))
    sk.close()
    dist.init_process_group("nccl", rank=0, world_size=1, device_id=torch.device("cuda", 0))
    try:
        stream = torch.cuda.Stream()
        dev.set_stream(stream.cuda_stream)
        host = torch.frombuffer(bytearray(tb), dtype=torch.uint8).pin_memory()
        with torch.cuda.stream(stream):
            full = parallel.load_tables_sharded(dev, P, host)
        dev.synchronize()
        assert full.is_cuda and dev.download() == tb
        r = dev.sieve(2, 10000, N.TRIANGLE)
        g = golden["sieve"]["C3"]
        assert r.pairs_tested == g["pairs_tested"] and r.survivors == g["survivors"]
        assert {str(P[k]): int(c) for k, c in enumerate(r.hist) if c} == g["kill_histogram"]
    finally:
        dev.set_stream(None)
        dist.destroy_process_group()


def test_async_loads_verified_on_the_device(dev, golden, sets):
    """cgpu_tables_load_async / _dev_async (the e2e pipeline's loads, no host
    wait): results identical to the reference's; a padding error and
    non-canonical flags (an all-zero table the probe list expected to kill,
    a set bit in row 0) are reported by the deferred status -- through the
    status word, load_status and the next results call -- and the context
    re-derives so the repeated launch is right."""
    import torch
    P = sets["odd64"]
    tb, offs = port.build_set(P)
    g = golden["sieve"]["C3"]
    host = torch.frombuffer(bytearray(tb), dtype=torch.uint8).pin_memory()
    word = torch.zeros(1, dtype=torch.int32).pin_memory()
    for _ in range(3):  # first load speculates the builder's flags, later ones the verified flags
        dev.load_host_async(P, host.data_ptr(), len(tb))
        dev.load_status_copy(word.data_ptr())
        r = dev.sieve(2, 10000, N.TRIANGLE)
        assert int(word[0]) == 0
        assert r.pairs_tested == g["pairs_tested"] and r.survivors == g["survivors"]
        assert {str(P[k]): int(c) for k, c in enumerate(r.hist) if c} == g["kill_histogram"]
    dev.load_status()
    # a padding bit: FormatError at the status check
    bad = bytearray(tb)
    k11 = list(P).index(11)
    bad[int(offs[k11]) + (11 * 11 + 7) // 8 - 1] |= 0x80
    hb = torch.frombuffer(bad, dtype=torch.uint8).pin_memory()
    dev.load_host_async(P, hb.data_ptr(), len(tb))
    dev.load_status_copy(word.data_ptr())
    with pytest.raises(N.CudaSieveError) as e:
        dev.load_status()
    assert e.value.code == N.ERR_FORMAT and int(word[0]) & 1
    # the r = 11 table zeroed (never kills), against verified flags that say it kills
    dev.load(P, tb)
    z = bytearray(tb)
    z[int(offs[k11]):int(offs[k11]) + (11 * 11 + 7) // 8] = bytes((11 * 11 + 7) // 8)
    hz = torch.frombuffer(z, dtype=torch.uint8).pin_memory()
    dev.load_host_async(P, hz.data_ptr(), len(tb))
    dev.load_status_copy(word.data_ptr())
    dev.synchronize()
    assert int(word[0]) & 2
    with pytest.raises(N.CudaSieveError) as e:
        dev.sieve(2, 3000, N.TRIANGLE)  # the results call verifies the load
    assert e.value.code == N.ERR_INVALID
    r = dev.sieve(2, 3000, N.TRIANGLE)  # re-derived: right now
    o = port.sieve(bytes(z), P, offs, 2, 3000, port.TRIANGLE)
    assert (r.pairs_tested, r.survivors) == (o["pairs_tested"], o["survivors"])
    assert r.hist.tolist() == o["hist"].tolist()
    # a set bit in row 0 of r = 13: speculated canonical, reported, then exact in TRIANGLE
    k13 = list(P).index(13)
    w0 = bytearray(tb)
    w0[int(offs[k13])] |= 0x10
    h0 = torch.frombuffer(w0, dtype=torch.uint8).pin_memory()
    dev.load(P, tb)
    dev.load_host_async(P, h0.data_ptr(), len(tb))
    with pytest.raises(N.CudaSieveError):
        dev.load_status()
    r = dev.sieve(2, 3000, N.TRIANGLE)
    o = port.sieve(bytes(w0), P, offs, 2, 3000, port.TRIANGLE)
    assert (r.pairs_tested, r.survivors) == (o["pairs_tested"], o["survivors"])
    assert r.hist.tolist() == o["hist"].tolist()


def test_in_process_multi_gpu_clique(golden, sets):
    """cgpu_multi_* (the in-process NCCL path of cuboid::gpu::scan(...,
    devices)) over every device this box has: C3 whole-row TRIANGLE and a
    REGION span ending mid-row equal the reference's / the single-context
    result; survivors gathered in canonical order (weak sieve)."""
    L = N.lib()
    n = C.c_int()
    N.check(L.cgpu_device_count(C.byref(n)))
    devs = (C.c_int * n.value)(*range(n.value))
    m = C.c_void_p()
    N.check(L.cgpu_multi_create(n.value, devs, C.byref(m)))
    try:
        def run(P, lo, q0, hi, q_end, mode, cap=1 << 16):
            pr = np.ascontiguousarray(P, dtype=np.uint32)
            tb, _ = port.build_set(P)
            buf = np.frombuffer(tb, np.uint8)
            N.check(L.cgpu_multi_tables_load(m, pr.ctypes.data_as(C.c_void_p), len(pr),
                                             buf.ctypes.data_as(C.c_void_p), len(tb)))
            counts = np.zeros(2, np.uint64)
            hist = np.zeros(len(P), np.uint64)
            nb = hi // 100 - lo // 100 + 1
            brm = np.zeros(nb, np.uint32)
            surv = np.zeros((cap, 2), np.uint64)
            N.check(L.cgpu_multi_sieve(m, lo, q0, hi, q_end, mode, counts.ctypes.data_as(C.c_void_p),
                                       hist.ctypes.data_as(C.c_void_p), brm.ctypes.data_as(C.c_void_p), nb,
                                       surv.ctypes.data_as(C.c_void_p), cap))
            return counts, hist, brm, surv[:int(counts[1])]
        P = sets["odd64"]
        counts, hist, brm, _ = run(P, 2, 0, 10000, 0, N.TRIANGLE)
        g = golden["sieve"]["C3"]
        assert (int(counts[0]), int(counts[1])) == (g["pairs_tested"], g["survivors"])
        assert {str(P[k]): int(c) for k, c in enumerate(hist) if c} == g["kill_histogram"]
        assert {str(i): int(v) for i, v in enumerate(brm) if v} == g["block_r_max"]
        W = [11]
        counts, hist, brm, surv = run(W, 1, 1, 40, 0, N.REGION)
        tb, offs = port.build_set(W)
        o = port.sieve(tb, W, offs, 1, 40, port.REGION, q_start=1)
        assert (int(counts[0]), int(counts[1])) == (o["pairs_tested"], o["survivors"])
        assert np.array_equal(surv, o["survivor_pairs"])
        D = default_primes()
        counts, hist, brm, _ = run(D, 152, 3, 700, 12345, N.REGION)  # ends mid-row 700, at q = 12345
        # the reference halted at (700, 12346): a pre-armed stop at that q visited
        visited = 1 + sum(cuboid.q_bounds(p)[1] - (3 if p == 152 else cuboid.q_bounds(p)[0]) + 1
                          for p in range(152, 700)) + (12346 - cuboid.q_bounds(700)[0])
        rs = refmod.RefSet.build(D)
        ref = refmod.scan(rs, 152, 3, 700, batch_pairs=visited, stop_preset=True)
        assert ref.stopped and (ref.resume_p, ref.resume_q) == (700, 12346)
        assert (int(counts[0]), int(counts[1])) == (ref.pairs_tested, ref.survivors)
        assert [int(x) for x in hist] == list(ref.hist_by_rank)
        got_brm = {152 // 100 + i: int(v) for i, v in enumerate(brm) if v}
        assert got_brm == ref.block_r_max
    finally:
        L.cgpu_multi_destroy(m)


@pytest.mark.parametrize("seed", [1, 2, 3])
def test_random_region_spans_vs_reference(dev, seed):
    """Seeded REGION spans that start AND end mid-row (cgpu_sieve_span, what a
    stopped scan covers) against the reference's own scan() halted by a
    pre-armed stop at the same pair (engine.hpp:248-257): counts, histogram,
    block r_max."""
    rng = random.Random(seed)
    D = default_primes()
    tb, _ = port.build_set(D)
    dev.load(D, tb)
    rs = refmod.RefSet.build(D)
    for _ in range(6):
        p0 = rng.randrange(152, 20000)
        lo, hi = cuboid.q_bounds(p0)
        q0 = rng.randrange(lo, hi + 1)
        p1 = p0 + rng.randrange(0, 40)
        lo1, hi1 = cuboid.q_bounds(p1)
        q1 = rng.randrange(lo1 if p1 > p0 else q0, hi1 + 1)  # last pair sieved
        visited = 1 + sum(cuboid.q_bounds(p)[1] - (q0 if p == p0 else cuboid.q_bounds(p)[0]) + 1
                          for p in range(p0, p1)) + (q1 + 1 - (q0 if p1 == p0 else lo1))
        stop_at = cuboid.region_advance((p0, q0), visited - 1, p1 + 1)
        assert stop_at == ((p1, q1 + 1) if q1 < hi1 else (p1 + 1, cuboid.q_bounds(p1 + 1)[0]))
        ref = refmod.scan(rs, p0, q0, p1 + 1, batch_pairs=visited, stop_preset=True)
        assert ref.stopped and (ref.resume_p, ref.resume_q) == stop_at
        nb = p1 // 100 - p0 // 100 + 1
        counts = np.zeros(2, np.uint64)
        hist = np.zeros(len(D), np.uint64)
        brm = np.zeros(nb, np.uint32)
        spq = np.zeros((16, 2), np.uint64)
        N.check(N.lib().cgpu_sieve_span(dev._ctx, p0, q0, p1, q1, counts.ctypes.data_as(C.c_void_p),
                                        hist.ctypes.data_as(C.c_void_p), brm.ctypes.data_as(C.c_void_p), nb,
                                        spq.ctypes.data_as(C.c_void_p), 16))
        assert (int(counts[0]), int(counts[1])) == (ref.pairs_tested, ref.survivors)
        assert [int(x) for x in hist] == list(ref.hist_by_rank)
        got = {p0 // 100 + i: int(v) for i, v in enumerate(brm) if v}
        # the reference also enters the stop row's block, which lies past the span
        # when the stop is the first pair of row p1 + 1
        want = {b: r for b, r in ref.block_r_max.items() if b <= p1 // 100}
        assert got == want


def test_classify_large_pairs_vs_reference(dev, sets):
    """k_classify's 64-bit residues for pairs up to 2^32 against the
    reference's SieveSet::is_unsolvable in rank order."""
    P = sets["odd256"]
    tb, _ = port.build_set(P)
    dev.load(P, tb)
    rng = np.random.default_rng(99)
    p = rng.integers(1 << 20, (1 << 32) - 1, 20000, dtype=np.uint64)
    q = rng.integers(1, 1 << 32, 20000, dtype=np.uint64)
    pq = np.stack([p, q], 1)
    got = dev.classify(pq)
    want = refmod.classify(refmod.RefSet.build(P), pq, 4)
    assert np.array_equal(got.astype(np.int64), want.astype(np.int64))


def test_files_roundtrip_with_reference(tmp_path, sets):
    """GPU-built tables written through the C ABI are the reference's files
    (save_sieve_files / load_sieve_files, test_sievetable.cpp:240-262), and
    reference-written files load onto the device and sieve identically."""
    P = sets["default96"]
    s = cuboid.SieveSet.build(P)
    tp, ip = str(tmp_path / "tables.bin"), str(tmp_path / "primes.bin")
    s.save_files(tp, ip)
    tb, ix = open(tp, "rb").read(), open(ip, "rb").read()
    assert tb == port.build_set(P)[0]
    assert ix == s.serialize_index()
    if refmod.available():
        rs = refmod.RefSet.load(tb, ix)
        assert rs.tables() == tb and rs.index_bytes() == ix
    back = cuboid.SieveSet.load_files(tp, ip)
    assert back.primes() == P and back.tables() == tb
    st = cuboid.scan(back, (152, 3), 300)
    assert st.survivors == 0 and st.pairs_tested == cuboid.scan(s, (152, 3), 300).pairs_tested
    with pytest.raises(OSError):
        cuboid.SieveSet.load_files(str(tmp_path / "missing.bin"), ip)
    with pytest.raises(cuboid.FormatError):
        cuboid.load_sieve(tb[:-1], ix)
    empty = cuboid.load_sieve(b"", cuboid.serialize_index(cuboid.SieveSet([], b"", [], 0)))
    assert empty.empty()


def test_bench_subcommand_output(tmp_path, golden):
    """cli.hpp:213-248 (cmd_bench) on the GPU: the reference default set's
    files, REGION [152, 5000] -- 447,994,938 pairs per run (acceptance.cpp:
    123-144), the reference's line formats and the paper's 3.54e-07 s/pair."""
    import io
    from paper_1601_00636_b200 import bench_cmd
    s = cuboid.SieveSet.build_default()
    tp, ip = str(tmp_path / "t.bin"), str(tmp_path / "p.bin")
    s.save_files(tp, ip)
    out = io.StringIO()
    assert bench_cmd.cmd_bench(tp, ip, 152, 5000, 3, out=out) == 0
    lines = out.getvalue().splitlines()
    assert len(lines) == 5
    for k in range(3):
        assert lines[k].startswith(f"run {k + 1}: {golden['sieve']['R152_5000']['pairs_tested']} pairs in ")
        assert lines[k].endswith(" s/pair")
    assert lines[3] == "reference dt: 3.54e-07 s/pair"
    assert lines[4].startswith("run-to-run variation: ")
    out = io.StringIO()
    bench_cmd.cmd_bench(tp, ip, 200, 199, 1, out=out)  # empty range
    assert out.getvalue() == "run 1: 0 pairs in " + out.getvalue().split(" in ")[1]
    assert out.getvalue().endswith(" s (empty range)\n")


def test_dump_table_text_matches_u11():
    """test_sievetable.cpp:222-238: the text dump of r = 11 is the paper's U_11."""
    s = cuboid.SieveSet.build([2, 11])
    txt = cuboid.dump_table_text(s, 11).splitlines()
    assert txt[0] == "r=11"
    want = port.build_table(11)
    for p in range(11):
        row = txt[1 + p].split(": ")[1]
        assert row == "".join(str((want[(p * 11 + q) >> 3] >> ((p * 11 + q) & 7)) & 1) for q in range(11))
    assert cuboid.dump_table_text(s, 2) == "r=2\n0: 00\n1: 00\n"


def test_historical_region_scan():
    """p = 1..154000 over the full region with the 96 primes
    11..541: no pair passes the sieve and the deepest first killer is 137 (the
    29th prime of the set)."""
    s = cuboid.SieveSet.build_default()
    st = cuboid.scan(s, (1, 1), 154000, opt=cuboid.ScanOptions(small_p=True))
    assert st.survivors == 0
    assert max(st.kill_histogram) == 137
    assert max(st.block_r_max.values()) == 137
    assert len(st.block_r_max) == 1541
    assert st.histogram_total() == st.pairs_tested


def _factors(n):
    f, d = [], 2
    while d * d <= n:
        if n % d == 0:
            f.append(d)
            while n % d == 0:
                n //= d
        d += 1 if d == 2 else 2
    if n > 1:
        f.append(n)
    return f


def _coprime_count(p, lo, hi):
    """#{q in [lo, hi]: gcd(p, q) = 1, q != p} by inclusion-exclusion."""
    fs = _factors(p)
    tot = 0
    for mask in range(1 << len(fs)):
        d, bits = 1, 0
        for i, f in enumerate(fs):
            if mask >> i & 1:
                d *= f
                bits += 1
        tot += (-1) ** bits * (hi // d - (lo - 1) // d)
    if p == 1 and lo <= 1 <= hi:
        tot -= 1
    return tot


def test_rows_at_the_32bit_limits(dev, sets):
    """Maximum sizes: the last REGION row below the 32-bit limit (q up to
    59p = 4,294,967,245, region.hpp:43-44) and TRIANGLE rows next to 2^32:
    exact candidate counts, every candidate accounted for, and a tail of the
    REGION row checked pair by pair against the oracle."""
    P = sets["default96"]
    tb, offs = port.build_set(P)
    dev.load(P, tb)
    p = 72796055
    lo, hi = cuboid.q_bounds(p)
    r = dev.sieve(p, p, N.REGION)
    assert r.pairs_tested == _coprime_count(p, lo, hi)
    assert int(r.hist.sum()) + r.survivors == r.pairs_tested
    q0 = hi - 20000
    r = dev.sieve(p, p, N.REGION, q_start=q0)
    o = port.sieve(tb, P, offs, p, p, port.REGION, q_start=q0)
    assert (r.pairs_tested, r.survivors) == (o["pairs_tested"], o["survivors"])
    assert r.hist.tolist() == o["hist"].tolist()
    for p in (4294967291, 4294967295, 4294967294):  # prime; 3*5*17*257*65537; 2*3*...
        r = dev.sieve(p, p, N.TRIANGLE)
        assert r.pairs_tested == _coprime_count(p, 1, p - 1), p
        assert int(r.hist.sum()) + r.survivors == r.pairs_tested
    with pytest.raises(N.CudaSieveError):
        dev.sieve(4294967296, 4294967296, N.TRIANGLE)


@pytest.mark.skipif(not refmod.available(), reason="oracle/_ref not built")
@pytest.mark.parametrize("bp", [1, 59, 1000, 9000, 65536, 400000])
def test_prearmed_stop_matches_reference(bp):
    """A stop flag raised before scan() halts at the reference's batch boundary
    with the same statistics and resume point (engine.hpp:248-257,
    test_engine.cpp:149-164); resuming from there and merging gives the whole
    scan (test_engine.cpp:134-175)."""
    P = default_primes()
    rs = refmod.RefSet.build(P)
    s = cuboid.SieveSet.build(P)
    for start in [(152, 3), (153, 7000), (401, 23000), (499, cuboid.q_bounds(499)[1])]:
        ref = refmod.scan(rs, start[0], start[1], 700, batch_pairs=bp, stop_preset=True)
        got = cuboid.scan(s, start, 700, opt=cuboid.ScanOptions(batch_pairs=bp, stop=True))
        assert got.stopped == ref.stopped
        assert (got.resume_p, got.resume_q) == (ref.resume_p, ref.resume_q)
        assert got.pairs_tested == ref.pairs_tested and got.survivors == ref.survivors
        assert got.kill_histogram == ref.kill_histogram(P)
        assert got.block_r_max == ref.block_r_max
        tail = cuboid.scan(s, (got.resume_p, got.resume_q), 700)
        got.merge(tail)
        whole = refmod.scan(rs, start[0], start[1], 700)
        assert got.pairs_tested == whole.pairs_tested
        assert got.kill_histogram == whole.kill_histogram(P)
        assert got.block_r_max == whole.block_r_max


def test_prearmed_stop_short_range_completes():
    """A flag raised before scan() with fewer q left than batch_pairs: the
    reference never reaches a poll and scans the whole range."""
    P = default_primes()
    rs = refmod.RefSet.build(P)
    s = cuboid.SieveSet.build(P)
    ref = refmod.scan(rs, 152, 3, 400, batch_pairs=1 << 30, stop_preset=True)
    got = cuboid.scan(s, (152, 3), 400, opt=cuboid.ScanOptions(batch_pairs=1 << 30, stop=True))
    assert not ref.stopped and not got.stopped
    assert (got.pairs_tested, got.resume_p, got.resume_q) == (ref.pairs_tested, ref.resume_p, ref.resume_q)
    assert got.kill_histogram == ref.kill_histogram(P)


def test_stop_raised_mid_scan_halts_at_a_poll_point():
    """The Python mirror sees a flag raised WHILE the device sieves (mapped
    stop word): it halts at a poll point of the reference (q visited + 1 is a
    multiple of batch_pairs), the halves merge to the uninterrupted scan, and
    the stopped half equals a pre-armed stop at the same poll."""
    import threading
    P = default_primes()
    s = cuboid.SieveSet.build(P)
    p_end, B = 1500000, 1 << 16
    ev = threading.Event()
    threading.Timer(0.3, ev.set).start()
    h = cuboid.scan(s, (152, 3), p_end, opt=cuboid.ScanOptions(batch_pairs=B, stop=ev))
    assert h.stopped and 152 < h.resume_p < p_end
    visited = 0
    for p in range(152, h.resume_p + 1):
        lo, hi = cuboid.q_bounds(p)
        q0 = 3 if p == 152 else lo
        visited += (hi - q0 + 1) if p < h.resume_p else (h.resume_q - q0)
    assert (visited + 1) % B == 0
    tail = cuboid.scan(s, (h.resume_p, h.resume_q), p_end)
    whole = cuboid.scan(s, (152, 3), p_end)
    again = cuboid.scan(s, (152, 3), p_end, opt=cuboid.ScanOptions(batch_pairs=visited + 1, stop=True))
    assert (again.pairs_tested, again.kill_histogram, again.block_r_max, again.resume_p, again.resume_q) == \
        (h.pairs_tested, h.kill_histogram, h.block_r_max, h.resume_p, h.resume_q)
    h.merge(tail)
    assert (h.pairs_tested, h.survivors, h.kill_histogram, h.block_r_max, h.resume_p, h.resume_q) == \
        (whole.pairs_tested, whole.survivors, whole.kill_histogram, whole.block_r_max, whole.resume_p,
         whole.resume_q)


def test_stoppable_scan_tiles_equal_one_launch():
    """A scan polled for stops (never raised) runs as many tiles: same result."""
    s = cuboid.SieveSet.build(default_primes())
    tiled = cuboid.scan(s, (152, 3), 200000, opt=cuboid.ScanOptions(stop=lambda: False))
    one = cuboid.scan(s, (152, 3), 200000)
    assert not tiled.stopped
    assert (tiled.pairs_tested, tiled.kill_histogram, tiled.block_r_max, tiled.resume_p, tiled.resume_q) == \
        (one.pairs_tested, one.kill_histogram, one.block_r_max, one.resume_p, one.resume_q)


def test_multi_chunk_launch(dev, sets):
    """A range of more than one launch chunk (1,048,500 row slots): TRIANGLE
    p <= 1.1e6 (3.7e11 pairs) -- every candidate counted once across the
    chunked plan/sieve launches, and block-cyclic shards merging to it."""
    P = sets["odd32"]
    tb, _ = port.build_set(P)
    dev.load(P, tb)
    hi = 1_100_000
    r = dev.sieve(2, hi, N.TRIANGLE)
    assert r.pairs_tested == phi_sum(2, hi)
    assert int(r.hist.sum()) + r.survivors == r.pairs_tested
    assert (r.block_rmax >= 1).all()
    parts = [dev.sieve(2, hi, N.TRIANGLE, shard=(2, k)) for k in range(2)]
    assert sum(x.pairs_tested for x in parts) == r.pairs_tested
    assert np.array_equal(parts[0].hist + parts[1].hist, r.hist)
    assert np.array_equal(np.maximum(parts[0].block_rmax, parts[1].block_rmax), r.block_rmax)


def test_build_is_deterministic(dev, sets):
    """test_sievetable.cpp:264-270: building twice gives identical bytes."""
    for alg in (N.BUILD_PRODUCTION, N.BUILD_EXHAUSTIVE):
        a, _ = dev.build(sets["odd64"], alg)
        b, _ = dev.build(sets["odd64"], alg)
        assert a == b


def test_verify_small_region_pin(golden):
    """engine.hpp:609-640 / test_engine.cpp:416-423: 413,362 pairs, all sieved
    out; every survivor goes through the reference's own verify_pair(bypass)."""
    s = cuboid.SieveSet.build_default()
    rset = refmod.RefSet.build(default_primes())
    v = cuboid.verify_small_region(s, lambda p, q: refmod.verify_pair(rset, p, q, True)[0])
    g = golden["verify_small_region"]
    assert (v.pairs, v.sieved_out, v.survivors, v.no_integer_root, v.root_fails, v.candidates) == \
        (g["pairs"], g["sieved_out"], g["survivors"], g["no_integer_root"], g["root_fails"],
         g["candidates"])
    weak = cuboid.SieveSet.build([11])
    wref = refmod.RefSet.build([11])
    w = cuboid.verify_small_region(weak, lambda p, q: refmod.verify_pair(wref, p, q, True)[0])
    want = refmod.verify_small_region(wref)
    assert w.survivors > 0
    assert vars(w) == want
    with pytest.raises(TypeError):
        cuboid.verify_small_region(weak, None)
