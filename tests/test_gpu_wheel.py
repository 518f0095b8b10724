"""The sieve parity cases once more with the wheel sieve (k_wsieve) forced on
every standard-set launch, short rows included (CUBOID_WHEEL=2; by default only
launches of long rows take it), and with it switched off (CUBOID_WHEEL=0: the
window sieve k_sieve everywhere) -- the knob is read when a context is
created, so each setting runs in its own interpreter."""
from __future__ import annotations

import os
import subprocess
import sys

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
CASES = ("sieve_identical or region_pins or random_ranges or non_canonical or register_probe_layouts or "
         "heavy_survivor or block_cyclic or c4_random_subsample or random_region_spans or "
         "rows_at_the_32bit_limits or prearmed_stop or stoppable_scan_tiles or multi_chunk or "
         "verify_small_region_pin or c5_full_range")


@pytest.mark.gpu
@pytest.mark.parametrize("mode", ["2", "0"])
def test_sieve_parity_cases_with_the_wheel_forced_and_off(mode):
    env = dict(os.environ, CUBOID_WHEEL=mode)
    r = subprocess.run([sys.executable, "-m", "pytest", os.path.join(ROOT, "tests", "test_gpu_parity.py"),
                        "-m", "gpu", "-q", "-x", "-k", CASES, "-p", "no:cacheprovider"],
                       env=env, cwd=ROOT, capture_output=True, text=True, timeout=1500)
    assert r.returncode == 0, r.stdout[-3000:] + r.stderr[-2000:]
    assert " passed" in r.stdout


@pytest.mark.gpu
def test_wheel_rows_divisible_by_the_wheel_primes_and_large_factors():
    """Rows the wheel treats specially, against the C oracle: p divisible by 11, 13, 17 and by
    their products (whole residue classes stay alive, class 0 is dropped), rows whose cofactor is a
    prime above 37681 (the two-candidate mask path), rows shorter than one class period, and
    REGION rows starting and ending mid-row."""
    code = r'''
import sys, os
sys.path.insert(0, os.environ["ROOT"])
import numpy as np
from oracle import port
from paper_1601_00636_b200 import _native as N
from paper_1601_00636_b200.device import Device
from paper_1601_00636_b200.primes import odd_primes
P = odd_primes(96)
tb, offs = port.build_set(P)
dev = Device(0)
dev.load(P, tb)
cases = [(N.TRIANGLE, 2431 * 41, 2431 * 41, 0), (N.TRIANGLE, 187 * 531, 187 * 531 + 2, 0),
         (N.TRIANGLE, 2 * 37693, 2 * 37693, 0), (N.TRIANGLE, 3 * 77801, 3 * 77801 + 1, 0),
         (N.TRIANGLE, 143 * 1009, 143 * 1009, 0), (N.TRIANGLE, 1, 40, 0), (N.TRIANGLE, 2400, 2440, 0),
         (N.REGION, 2431, 2432, 0), (N.REGION, 4862, 4862, 1000), (N.REGION, 7 * 5477, 7 * 5477, 0),
         (N.TRIANGLE, 3 * 5 * 7 * 19 * 23, 3 * 5 * 7 * 19 * 23, 0), (N.TRIANGLE, 221 * 997, 221 * 997, 0)]
for mode, lo, hi, q0 in cases:
    o = port.sieve(tb, P, offs, lo, hi, mode, q_start=q0)
    r = dev.sieve(lo, hi, mode, q_start=q0, surv_cap=1 << 22)
    assert r.pairs_tested == o["pairs_tested"], (mode, lo, hi, q0)
    assert r.survivors == o["survivors"], (mode, lo, hi)
    assert r.hist.tolist() == o["hist"].tolist(), (mode, lo, hi)
    assert np.array_equal(r.survivor_pairs, o["survivor_pairs"])
    rows = np.asarray(o["row_rmax"])
    want = {}
    for i, v in enumerate(rows):
        want[(lo + i) // 100] = max(want.get((lo + i) // 100, 0), int(v))
    assert {r.block_lo + i: int(v) for i, v in enumerate(r.block_rmax) if v} == want
# a set that ends at 37: no deep probes at all, every q alive after the window loop survives
P2 = odd_primes(11)
assert P2[-1] == 37
tb2, offs2 = port.build_set(P2)
dev.load(P2, tb2)
for mode, lo, hi in ((N.TRIANGLE, 2, 2600), (N.REGION, 152, 330)):
    o = port.sieve(tb2, P2, offs2, lo, hi, mode)
    r = dev.sieve(lo, hi, mode, surv_cap=1 << 22)
    assert dev.sieve_kernel() == "k_wsieve"
    assert (r.pairs_tested, r.survivors) == (o["pairs_tested"], o["survivors"]) and r.survivors > 100
    assert r.hist.tolist() == o["hist"].tolist()
    assert np.array_equal(r.survivor_pairs, o["survivor_pairs"])
print("wheel rows ok", len(cases))
'''
    env = dict(os.environ, CUBOID_WHEEL="2", ROOT=ROOT)
    r = subprocess.run([sys.executable, "-c", code], env=env, capture_output=True, text=True, timeout=900)
    assert r.returncode == 0, r.stdout[-2000:] + r.stderr[-3000:]
    assert "wheel rows ok" in r.stdout
