"""Pins the CPU oracle (oracle/cuboid_oracle.c, the plain-C restatement) to the
reference: its own known-answer tests (proj/tests/*.cpp) and the golden
fixtures generated from the unmodified reference headers (tests/golden/,
oracle/_ref). CPU only; nothing here needs a GPU.
"""
from __future__ import annotations

import hashlib
import random

import numpy as np
import pytest

from oracle import port
from oracle import ref as refmod
from paper_1601_00636_b200.primes import default_primes, is_prime, odd_primes, primes_in_range

needs_ref_early = pytest.mark.skipif(not refmod.available(), reason="oracle/_ref not built")

# proj/tests/test_sievetable.cpp:12-37 -- the 11x11 matrix U_11 of the paper's
# Table 2.5 (rows p~, columns q~) and its 16 packed bytes (PAPER.md (2.6)).
U11_BYTES = bytes.fromhex("00E09F7EEDED76CF7BDEEDF6D62FFF00")


def sha(b: bytes) -> str:
    return hashlib.sha256(b).hexdigest()


# ---- tables ---------------------------------------------------------------------

def test_r11_golden_bytes(golden):
    """test_sievetable.cpp:12-37 (kU11 / paper (2.6))."""
    assert port.build_table(11) == U11_BYTES
    assert golden["tables"]["r11_bytes"] == U11_BYTES.hex()
    got, _ = port.build_table_oracle(11)
    assert got == U11_BYTES


@pytest.mark.parametrize("r", [2, 3, 5, 7])
def test_tiny_primes_all_zero(r):
    """test_sievetable.cpp:39-47."""
    assert port.build_table(r) == bytes((r * r + 7) // 8)


def test_builder_matches_definition_up_to_97():
    """test_sievetable.cpp:49-56 / acceptance.cpp:83-90: production == oracle."""
    for r in primes_in_range(2, 97):
        prod = port.build_table(r)
        brute, _ = port.build_table_oracle(r)
        assert prod == brute, r


@pytest.mark.parametrize("r", [0, 1, 4, 9, 9697, 9699, 10007])
def test_bad_moduli_rejected(r):
    """test_sievetable.cpp:58-64, 272-277."""
    with pytest.raises(ValueError):
        port.build_table(r)


def test_zero_margins_and_symmetry():
    """test_sievetable.cpp:66-90: row 0 and column 0 solvable; u(p,q) = u(q,p)
    and u(p,q) = u(-p,q) (Q is even in p and q)."""
    for r in (11, 13, 97, 541):
        tb = port.build_table(r)
        bit = lambda a, b: (tb[(a * r + b) >> 3] >> ((a * r + b) & 7)) & 1
        for a in range(r):
            assert bit(0, a) == 0 and bit(a, 0) == 0
        rng = random.Random(r)
        for _ in range(500):
            a, b = rng.randrange(r), rng.randrange(r)
            assert bit(a, b) == bit(b, a) == bit((r - a) % r, b)


def test_projective_scaling():
    """test_sievetable.cpp:92-102: u(lp, lq) = u(p, q) for l != 0 mod r."""
    rng = random.Random(99)
    for r in (11, 31, 101, 1021):
        tb = port.build_table(r)
        bit = lambda a, b: (tb[(a * r + b) >> 3] >> ((a * r + b) & 7)) & 1
        for _ in range(300):
            a, b, l = rng.randrange(r), rng.randrange(r), rng.randrange(1, r)
            assert bit(a, b) == bit(a * l % r, b * l % r)


@pytest.mark.parametrize("name", ["odd32", "odd64", "default96", "odd128"])
def test_sets_match_reference_golden(golden, sets, name):
    """Byte-identical concatenated sets vs the reference's SieveSet::build."""
    tb, offs = port.build_set(sets[name])
    g = golden["tables"][name]
    assert len(tb) == g["bytes"]
    assert sha(tb) == g["sha256"]


def test_default_set_sizes(sets):
    """test_sievetable.cpp:131-141, test_cli.cpp:60-64: 96 primes, 1,048,164
    table bytes; r = 541 occupies 36,586 bytes."""
    tb, offs = port.build_set(sets["default96"])
    assert len(sets["default96"]) == 96
    assert len(tb) == 1048164
    assert len(tb) - offs[-1] == 36586


@pytest.mark.slow
def test_odd256_matches_reference_golden(golden, sets):
    tb, _ = port.build_set(sets["odd256"])
    assert sha(tb) == golden["tables"]["odd256"]["sha256"]


def test_set_validation():
    with pytest.raises(ValueError):
        port.build_set([13, 11])
    with pytest.raises(ValueError):
        port.build_set([11, 15])


# ---- modular arithmetic ------------------------------------------------------------

def _q_exact(p, q, t):
    """Q_pq(t) (modpoly.hpp:3-11, PAPER.md): degree 10, even in t."""
    s = t * t
    c4 = (2 * q * q + p * p) * (3 * q * q - 2 * p * p)
    c3 = q**8 + 10 * p**2 * q**6 + 4 * p**4 * q**4 - 14 * p**6 * q**2 + p**8
    c2 = -p**2 * q**2 * (q**8 - 14 * p**2 * q**6 + 4 * p**4 * q**4 + 10 * p**6 * q**2 + p**8)
    c1 = -p**6 * q**6 * (q**2 + 2 * p**2) * (3 * p**2 - 2 * q**2)
    c0 = -p**10 * q**10
    return (((((s + c4) * s + c3) * s + c2) * s + c1) * s) + c0


def test_mod_examples_and_validation():
    """test_modpoly.cpp:49-64."""
    assert port.eval_q_mod(0, 5, 0, 11) == 0
    assert port.eval_q_mod(1, 1, 1, 7) == 0
    assert port.eval_q_mod(1, 0, 1, 11) == 0
    for args in [(1, 1, 1, 4), (1, 1, 1, 9697), (1, 1, 1, 10007), (11, 1, 1, 11), (1, 12, 1, 11),
                 (1, 1, 13, 11)]:
        assert port.eval_q_mod(*args) == -1


def test_mod_matches_exact_small():
    """test_modpoly.cpp:66-89: mod r evaluation of the residues == exact value mod r."""
    for r in primes_in_range(2, 97):
        for p in range(1, 50, 3):
            for q in range(1, 50, 4):
                for t in range(0, 50, 7):
                    assert port.eval_q_mod(p % r, q % r, t % r, r) == _q_exact(p, q, t) % r


def test_mod_matches_exact_random():
    """acceptance.cpp:220-242 (10^4 random samples, seed 160401)."""
    rng = random.Random(160401)
    rs = primes_in_range(2, 9689)
    for _ in range(10000):
        r = rng.choice(rs)
        p, q, t = rng.randrange(r), rng.randrange(r), rng.randrange(r)
        assert port.eval_q_mod(p, q, t, r) == _q_exact(p, q, t) % r


def test_evenness():
    """test_modpoly.cpp:91-107, including r = 9689."""
    rng = random.Random(20160401)
    for r in (11, 541, 9689):
        for _ in range(200):
            p, q, t = rng.randrange(r), rng.randrange(r), rng.randrange(r)
            assert port.eval_q_mod(p, q, t, r) == port.eval_q_mod(p, q, (r - t) % r, r)


# ---- region bounds ------------------------------------------------------------------

def test_q_bounds():
    """region.hpp:49-63 (test_region.cpp): q_high = 59p; q_low = least q with
    9q^3 >= p above the 152 crossover, ceil(p/59) below it."""
    assert port.q_bounds(1) == (1, 59)
    assert port.q_bounds(151) == (3, 59 * 151)
    assert port.q_bounds(152) == (3, 59 * 152)
    rng = random.Random(424242)
    for _ in range(2000):
        p = rng.randrange(152, 1 << 40)
        lo, hi = port.q_bounds(p)
        assert hi == 59 * p and 9 * lo**3 >= p and (lo == 1 or 9 * (lo - 1) ** 3 < p)


# ---- sieve --------------------------------------------------------------------------

def _hist_by_prime(primes, hist):
    return {str(primes[k]): int(c) for k, c in enumerate(hist) if c}


def _block_rmax(p_lo, row_rmax):
    out = {}
    for i, v in enumerate(row_rmax):
        b = (p_lo + i) // 100
        out[b] = max(out.get(b, 0), int(v))
    return {str(b): v for b, v in sorted(out.items())}


def _check_sieve(golden, sets, name):
    g = golden["sieve"][name]
    P = sets[g["set"]]
    tb, offs = port.build_set(P)
    mode = port.TRIANGLE if g["mode"] == "TRIANGLE" else port.REGION
    o = port.sieve(tb, P, offs, g["p_lo"], g["p_hi"], mode, q_start=g.get("q_start", 0))
    assert o["pairs_tested"] == g["pairs_tested"]
    assert o["survivors"] == g["survivors"]
    assert _hist_by_prime(P, o["hist"]) == g["kill_histogram"]
    assert _block_rmax(g["p_lo"], o["row_rmax"]) == g["block_r_max"]
    if "survivor_sha256" in g:
        flat = ",".join(f"{p}:{q}" for p, q in o["survivor_pairs"].tolist())
        assert sha(flat.encode()) == g["survivor_sha256"]
    return o


@pytest.mark.parametrize("name", ["C1", "R152", "R152_300", "R153_5000tail", "W_row1", "W_1_40",
                                  "W_T300", "R1_151"])
def test_sieve_matches_reference_golden(golden, sets, name):
    _check_sieve(golden, sets, name)


def test_row_152_pin(golden, sets):
    """test_engine.cpp:71-88: row p=152 -> 4,247 pairs, 0 survivors, max killer 47."""
    g = golden["sieve"]["R152"]
    assert g["pairs_tested"] == 4247 and g["survivors"] == 0
    assert max(int(k) for k in g["kill_histogram"]) == 47
    assert g["resume"] == [153, port.q_bounds(153)[0]]


def test_region_5000_pin(golden):
    """acceptance.cpp:123-144: [152,5000] -> 447,994,938 pairs, 0 survivors, max 97."""
    g = golden["sieve"]["R152_5000"]
    assert g["pairs_tested"] == 447994938 and g["survivors"] == 0
    assert max(int(k) for k in g["kill_histogram"]) == 97


def test_config_pins(golden):
    """SURVEY.md 8(c) survey-derived goldens, regenerated from the reference."""
    s = golden["sieve"]
    assert s["C1"]["pairs_tested"] == 1216587 and s["C1"]["survivors"] == 0
    assert s["C3"]["pairs_tested"] == 30397485
    assert s["C4"]["pairs_tested"] == 3039650753 and s["C4"]["survivors"] == 0
    assert s["C5_sub"]["pairs_tested"] == 121858132


def test_c5_golden_is_the_full_headline_range(golden):
    """The headline config's reference result covers all of C5: 2.43e10 pairs
    (sum phi(p)), 0 survivors, one r_max per p/100 block."""
    g = golden["sieve"]["C5"]
    assert (g["p_lo"], g["p_hi"], g["mode"], g["set"]) == (100001, 300000, "TRIANGLE", "odd256")
    assert g["pairs_tested"] == 24317097730 and g["survivors"] == 0
    assert sum(g["kill_histogram"].values()) == g["pairs_tested"]
    assert len(g["block_r_max"]) == 300000 // 100 - 100001 // 100 + 1


def test_c4_subsample_sampler_and_ranks(golden):
    """The phi-weighted coprime sampler (tests/subsample.py) reproduces the
    golden's pairs, and a numpy restatement of is_unsolvable's rank-ordered
    probe (sievetable.hpp:199-205) over the C oracle's tables reproduces the
    reference's first-killer ranks (oracle/_ref, golden C4_subsample)."""
    import math

    import subsample
    g = golden["sieve"]["C4_subsample"]
    pq = subsample.sample(g["n"], g["seed"], g["p_max"])
    assert hashlib.sha256(pq.tobytes()).hexdigest() == g["pairs_sha256"]
    p, q = pq[:, 0], pq[:, 1]
    assert bool(np.all((q >= 1) & (q < p))) and bool(np.all(np.gcd(p, q) == 1))
    assert all(math.gcd(int(a), int(b)) == 1 for a, b in pq[:100])
    P = odd_primes(128)
    tb, offs = port.build_set(P)
    buf = np.frombuffer(tb, np.uint8)
    ranks = np.full(len(p), -1, np.int32)
    for k, r in enumerate(P):
        i = (p % r) * r + (q % r)
        hit = ((buf[offs[k] + (i >> 3)] >> (i & 7).astype(np.uint8)) & 1).astype(bool)
        ranks[(ranks < 0) & hit] = k
    assert hashlib.sha256(ranks.astype("<i4").tobytes()).hexdigest() == g["ranks_sha256"]


@needs_ref_early
def test_c4_subsample_ref_classify_spot(golden):
    """The golden's ranks come from SieveSet::is_unsolvable: spot-check 2000
    pairs through the reference library directly."""
    import subsample
    g = golden["sieve"]["C4_subsample"]
    pq = subsample.sample(g["n"], g["seed"], g["p_max"])[:2000]
    rs = refmod.RefSet.build(odd_primes(128))
    got = refmod.classify(rs, pq, 2)
    for (a, b), k in zip(pq[:50].tolist(), got[:50].tolist()):
        want = next((j for j in range(128) if rs.is_unsolvable(j, a, b)), -1)
        assert k == want


def test_small_region_pin(golden):
    """test_engine.cpp:416-423: verify_small_region visits 413,362 pairs."""
    assert golden["verify_small_region"]["pairs"] == 413362
    assert golden["verify_small_region"]["candidates"] == 0


# ---- against the reference library itself (oracle/_ref), when built here ---------------

needs_ref = pytest.mark.skipif(not refmod.available(), reason="oracle/_ref not built")


@needs_ref
def test_port_vs_ref_tables_and_eval():
    rng = random.Random(7)
    for r in (11, 101, 541, 1021, 1621, 9689):
        assert port.build_table(r) == refmod.build_table(r)
    for _ in range(2000):
        r = rng.choice(primes_in_range(2, 9689))
        p, q, t = rng.randrange(r), rng.randrange(r), rng.randrange(r)
        assert port.eval_q_mod(p, q, t, r) == refmod.eval_q_mod(p, q, t, r)


@needs_ref
def test_port_vs_ref_sieve_random_rows():
    """Seeded random row ranges in both modes, two prime sets."""
    rng = random.Random(13)
    for P in (odd_primes(32), default_primes()):
        rs = refmod.RefSet.build(P)
        tb, offs = port.build_set(P)
        assert tb == rs.tables()
        for _ in range(4):
            lo = rng.randrange(152, 3000)
            hi = lo + rng.randrange(0, 8)
            st = refmod.triangle(rs, lo, hi, 1)
            o = port.sieve(tb, P, offs, lo, hi, port.TRIANGLE)
            assert (o["pairs_tested"], o["survivors"]) == (st.pairs_tested, st.survivors)
            assert [int(x) for x in o["hist"]] == list(st.hist_by_rank)
            q0 = rng.randrange(*port.q_bounds(lo))
            st = refmod.scan(rs, lo, q0, hi)
            o = port.sieve(tb, P, offs, lo, hi, port.REGION, q_start=q0)
            assert (o["pairs_tested"], o["survivors"]) == (st.pairs_tested, st.survivors)
            assert [int(x) for x in o["hist"]] == list(st.hist_by_rank)


@needs_ref
def test_ref_verify_pair_pins():
    """test_engine.cpp:51-59: (152, 3) is sieved out by 11."""
    rs = refmod.RefSet.build(default_primes())
    kind, prime, _ = refmod.verify_pair(rs, 152, 3, False)
    assert kind == "SievedOut" and prime == 11


def test_is_prime_helper():
    assert [n for n in range(30) if is_prime(n)] == [2, 3, 5, 7, 11, 13, 17, 19, 23, 29]
    assert odd_primes(4) == [3, 5, 7, 11]
    assert default_primes()[0] == 11 and default_primes()[-1] == 541
    assert len(odd_primes(256)) == 256 and odd_primes(256)[-1] == 1621
