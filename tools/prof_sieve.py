"""Small driver for ncu: one table build + a few sieve launches of a config."""
import sys, os
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_1601_00636_b200 import device as D, _native as N, odd_primes
cfg = sys.argv[1] if len(sys.argv) > 1 else "C5"
k, lo, hi = {"C4": (128, 2, 100000), "C5": (256, 100001, 300000), "C3": (64, 2, 10000)}[cfg]
dev = D.Device(0)
dev.build(odd_primes(k), N.BUILD_PRODUCTION, download=False)
for _ in range(int(sys.argv[2]) if len(sys.argv) > 2 else 2):
    r = dev.sieve(lo, hi, N.TRIANGLE)
    print(cfg, r.pairs_tested, dev.timings_ms(), flush=True)
