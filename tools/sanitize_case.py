"""Small end-to-end exercise of every device entry point, for
compute-sanitizer (memcheck / racecheck / synccheck / initcheck, one tool per
run). Checks results against the C oracle so a silent corruption also fails."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402

from oracle import port  # noqa: E402
from paper_1601_00636_b200 import _native as N  # noqa: E402
from paper_1601_00636_b200.device import Device  # noqa: E402
from paper_1601_00636_b200.primes import default_primes, odd_primes  # noqa: E402

dev = Device(0)
for P in ([11], [11, 13], odd_primes(40), default_primes()[:30]):
    want, offs = port.build_set(P)
    for alg in (N.BUILD_PRODUCTION, N.BUILD_EXHAUSTIVE):
        got, _ = dev.build(P, alg)
        assert got == want, (P[:3], alg)
    for (lo, hi, mode, q0) in [(2, 600, N.TRIANGLE, 0), (1, 3, N.REGION, 0), (152, 160, N.REGION, 5),
                               (301, 301, N.TRIANGLE, 0)]:
        r = dev.sieve(lo, hi, mode, q_start=q0, surv_cap=1 << 20)
        o = port.sieve(want, P, offs, lo, hi, mode, q_start=q0)
        assert r.pairs_tested == o["pairs_tested"] and r.survivors == o["survivors"]
        assert np.array_equal(r.hist, o["hist"]) and np.array_equal(r.survivor_pairs, o["survivor_pairs"])
        r2 = dev.sieve(lo, hi, mode, q_start=q0, shard=(3, 1), surv_cap=1 << 20)
    pq = np.array([[p, q] for p in range(2, 60) for q in range(1, p)], np.uint64)
    dev.classify(pq)
dev.load(odd_primes(12), port.build_set(odd_primes(12))[0])
dev.sieve(2, 300, N.TRIANGLE)
dev.close()
# the wheel sieve k_wsieve forced on every standard-set launch (the knob is read at context creation)
os.environ["CUBOID_WHEEL"] = "2"
dev = Device(0)
for P in (odd_primes(40), odd_primes(11)):
    want, offs = port.build_set(P)
    dev.load(P, want)
    for (lo, hi, mode, q0) in [(2, 700, N.TRIANGLE, 0), (2431, 2433, N.TRIANGLE, 0), (152, 158, N.REGION, 5),
                               (187 * 13, 187 * 13, N.REGION, 0), (1, 3, N.REGION, 0)]:
        r = dev.sieve(lo, hi, mode, q_start=q0, surv_cap=1 << 20)
        assert dev.sieve_kernel() == "k_wsieve"
        o = port.sieve(want, P, offs, lo, hi, mode, q_start=q0)
        assert r.pairs_tested == o["pairs_tested"] and r.survivors == o["survivors"]
        assert np.array_equal(r.hist, o["hist"]) and np.array_equal(r.survivor_pairs, o["survivor_pairs"])
        dev.sieve(lo, hi, mode, q_start=q0, shard=(3, 1), surv_cap=1 << 20)
print("sanitize case ok")
