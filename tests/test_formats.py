"""On-disk formats: the CUPQ v1 index and the tables
stream (sievetable.hpp:229-346, proj/README.md "File formats"), through the
C ABI's host-only entry points. The pins are the reference's
(test_sievetable.cpp:131-262) and the index hashes of the reference's own
serialize_index (tests/golden). CPU only."""
from __future__ import annotations

import hashlib

import pytest

from oracle import port
from paper_1601_00636_b200 import _native as N
from paper_1601_00636_b200.device import parse_index, serialize_index
from paper_1601_00636_b200.primes import default_primes

HDR, REC = 9, 6


def sha(b):
    return hashlib.sha256(b).hexdigest()


@pytest.mark.parametrize("name", ["odd32", "odd64", "odd128", "odd256", "default96"])
def test_index_bytes_identical_to_reference(golden, sets, name):
    ix = serialize_index(sets[name])
    g = golden["tables"][name]
    assert len(ix) == g["index_bytes"]
    assert sha(ix) == g["index_sha256"]
    primes, total = parse_index(ix)
    assert primes == sets[name] and total == g["bytes"]


def test_default_index_size():
    """test_sievetable.cpp:131-141: 585 B = 9-byte header + 96 records."""
    assert len(serialize_index(default_primes())) == 585


def test_empty_set_header_only_index():
    ix = serialize_index([])
    assert ix == b"CUPQ\x01\x00\x00\x00\x00"
    assert parse_index(ix) == ([], 0)


def _fmt_error(ix):
    with pytest.raises(N.CudaSieveError) as e:
        parse_index(ix)
    assert e.value.code == N.ERR_FORMAT


def test_corrupt_index_rejected():
    """test_sievetable.cpp:164-209."""
    ix = bytearray(serialize_index([11, 13]))
    _fmt_error(bytes(ix[:-1]))                     # truncated
    _fmt_error(bytes(ix[:5]))                      # shorter than the header
    b = bytearray(ix); b[0] ^= 0xFF; _fmt_error(bytes(b))        # bad magic
    b = bytearray(ix); b[4] = 9; _fmt_error(bytes(b))            # bad version
    b = bytearray(ix); b[HDR] = 12; _fmt_error(bytes(b))         # 11 -> 12, not prime
    b = bytearray(ix); b[HDR + REC + 2] ^= 1; _fmt_error(bytes(b))  # offset mismatch
    sw = bytearray(ix)                                            # non-monotone primes
    sw[HDR:HDR + REC], sw[HDR + REC:HDR + 2 * REC] = ix[HDR + REC:HDR + 2 * REC], ix[HDR:HDR + REC]
    _fmt_error(bytes(sw))
    b = bytearray(ix); b[HDR] = 0xF7; b[HDR + 1] = 0x25; _fmt_error(bytes(b))  # 9719: prime >= 9697
    b = bytearray(ix); b[5] = 3; _fmt_error(bytes(b))            # record count mismatch


def test_index_roundtrip_random_lists():
    import random
    rng = random.Random(7)
    allp = [p for p in range(2, 9697) if port.lib().co_is_prime(p)]
    for _ in range(20):
        P = sorted(rng.sample(allp, rng.randrange(1, 60)))
        primes, total = parse_index(serialize_index(P))
        assert primes == P and total == sum((r * r + 7) // 8 for r in P)


def test_serialize_rejects_bad_lists():
    for P in ([13, 11], [11, 15], [9697]):
        with pytest.raises(N.CudaSieveError):
            serialize_index(P)


def test_is_unsolvable_examples():
    """test_sievetable.cpp:212-220, through the Python mirror's host accessor
    (no device needed to read a set's bytes)."""
    from paper_1601_00636_b200 import cuboid
    tb, offs = port.build_set([11])
    s = cuboid.SieveSet([11], tb, offs, 0)
    assert s.is_unsolvable(0, 1, 2)
    assert not s.is_unsolvable(0, 12, 21)   # residues (1, 10)
    assert not s.is_unsolvable(0, 22, 7)    # residue row 0
    assert s.is_unsolvable(0, 12, 13)       # residues (1, 2)
    with pytest.raises(IndexError):
        s.is_unsolvable(3, 1, 2)
    assert s.prime_count() == 1 and s.prime_at(0) == 11 and s.rank_of(11) == 0 and s.rank_of(13) is None
    assert s.table_at(0).bytes == tb
    assert cuboid.dump_table_text(s, 11).splitlines()[0] == "r=11"
