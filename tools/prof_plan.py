"""Small driver for ncu: k_plan (+ k_sieve) of one 8-way C5 shard."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_1601_00636_b200 import device as D, _native as N, odd_primes  # noqa: E402

dev = D.Device(0)
dev.build(odd_primes(256), N.BUILD_PRODUCTION, download=False)
for _ in range(3):
    dev.sieve(100001, 300000, N.TRIANGLE, shard=(8, 2))
    print(dev.timings_ms(), flush=True)
