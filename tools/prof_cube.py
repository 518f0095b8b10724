"""Small driver for ncu: the exhaustive table build (BASELINE config 2), twice."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_1601_00636_b200 import device as D, _native as N, odd_primes  # noqa: E402

dev = D.Device(0)
for _ in range(2):
    dev.build(odd_primes(256), N.BUILD_EXHAUSTIVE, download=False)
    print("C2", dev.timings_ms(), flush=True)
