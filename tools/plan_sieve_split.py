import sys, os
sys.path.insert(0, os.getcwd())
from paper_1601_00636_b200 import device as D, _native as N, odd_primes
dev = D.Device(0)
for k, lo, hi in ((256, 100001, 300000), (128, 2, 100000)):
    dev.build(odd_primes(k), N.BUILD_PRODUCTION, download=False)
    ts = []
    for _ in range(5):
        dev.sieve(lo, hi, N.TRIANGLE)
        ts.append(dev.timings_ms())
    print(os.environ.get("CUBOID_GPU_LIB", "default"), k, min(t["plan"] for t in ts[1:]), min(t["sieve"] for t in ts[1:]))
