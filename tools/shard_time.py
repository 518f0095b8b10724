"""Per-shard sieve time vs the full C5 launch (strong-scaling check on one GPU):
for G = 2, 4, 8 the slowest block-cyclic shard's plan+sieve time against
full/G, plus small launches that expose the fixed per-launch cost."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_1601_00636_b200 import device as D, _native as N, odd_primes  # noqa: E402

dev = D.Device(0)
dev.build(odd_primes(256), N.BUILD_PRODUCTION, download=False)


def best(lo, hi, shard=(1, 0), k=3):
    ts = []
    for _ in range(k):
        r = dev.sieve(lo, hi, N.TRIANGLE, shard=shard)
        ts.append(dev.timings_ms())
    return min(ts, key=lambda t: t["total"]), r.pairs_tested


full, fp = best(100001, 300000, k=4)
print("full", full, fp)
for lo, hi in ((100001, 100010), (100001, 101000), (100001, 125000), (275001, 300000)):
    t, n = best(lo, hi)
    print(f"range {lo}-{hi}: {t} pairs {n} rate {n / t['sieve'] / 1e9:.3g} Gpairs/ms")
for G in (2, 4, 8):
    worst = 0
    for g in range(G):
        t, n = best(100001, 300000, (G, g))
        worst = max(worst, t["total"])
        if G == 8:
            print("  shard", g, t, n)
    print(G, "worst shard total ms", worst, "ideal", full["total"] / G, "eff", full["total"] / G / worst)
