"""Scratch GPU check: parity of tables + sieve against the oracles, rough timings."""
import sys, time, os
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
from paper_1601_00636_b200 import device as D, _native as N, odd_primes, default_primes
from oracle import port, ref

dev = D.Device(0)
for k in (32, 64, 128, 256):
    P = odd_primes(k)
    want, _ = port.build_set(P)
    for alg in (N.BUILD_PRODUCTION, N.BUILD_EXHAUSTIVE):
        t = time.time(); got, ev = dev.build(P, alg); dt = time.time() - t
        print(f"tables k={k} alg={alg} equal={got == want} evals={ev} wall={dt*1e3:.1f}ms", flush=True)

P = odd_primes(32)
t, o = port.build_set(P)
dev.load(P, t)
r = dev.sieve(2, 2000, N.TRIANGLE)
print("C1", r.pairs_tested, r.survivors, {P[k]: int(c) for k, c in enumerate(r.hist) if c}, r.block_rmax[:5])
o1 = port.sieve(t, P, o, 2, 2000, port.TRIANGLE)
print("C1 oracle", o1["pairs_tested"], np.array_equal(o1["hist"], r.hist))

DP = default_primes()
t, o = port.build_set(DP)
dev.load(DP, t)
for (a, b) in [(152, 152), (152, 2000), (152, 5000)]:
    r = dev.sieve(a, b, N.REGION, q_start=3 if a == 152 else 0)
    print("REGION", a, b, r.pairs_tested, r.survivors, max((DP[k] for k, c in enumerate(r.hist) if c), default=0), dev.timings_ms())

W = [11]
t, o = port.build_set(W)
dev.load(W, t)
r = dev.sieve(1, 1, N.REGION)
print("weak", r.survivors, r.survivor_pairs[:5].tolist())
r = dev.sieve(2, 2000, N.TRIANGLE)
o1 = port.sieve(t, W, o, 2, 2000, port.TRIANGLE)
print("weak C1", r.survivors, o1["survivors"], np.array_equal(r.survivor_pairs, o1["survivor_pairs"]), np.array_equal(o1["hist"], r.hist))

P = odd_primes(128)
dev.build(P, N.BUILD_PRODUCTION, download=False)
for it in range(3):
    r = dev.sieve(2, 100000, N.TRIANGLE)
    print("C4", r.pairs_tested, r.survivors, dev.timings_ms(), "pairs/s", r.pairs_tested / (dev.timings_ms()["sieve"] * 1e-3))
P = odd_primes(256)
dev.build(P, N.BUILD_PRODUCTION, download=False)
for it in range(2):
    r = dev.sieve(100001, 300000, N.TRIANGLE)
    print("C5", r.pairs_tested, r.survivors, dev.timings_ms(), "pairs/s", r.pairs_tested / (dev.timings_ms()["sieve"] * 1e-3))
