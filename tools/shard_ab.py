"""A/B of sieve libraries on the strong-scaling shapes: per library (CUBOID_GPU_LIB),
the full C5 launch, the slowest of the 8 block-cyclic C5 shards, and C4."""
import json
import os
import subprocess
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
CHILD = r'''
import sys, os, json
sys.path.insert(0, os.environ["ROOT"])
from paper_1601_00636_b200 import device as D, _native as N, odd_primes
dev = D.Device(0)
def best(lo, hi, shard=(1, 0), k=3):
    t = []
    for _ in range(k):
        dev.sieve(lo, hi, N.TRIANGLE, shard=shard)
        t.append(dev.timings_ms()["total"])
    return min(t)
dev.build(odd_primes(256), N.BUILD_PRODUCTION, download=False)
full = best(100001, 300000, k=4)
worst8 = max(best(100001, 300000, (8, g)) for g in range(8))
worst4 = max(best(100001, 300000, (4, g)) for g in range(4))
dev.build(odd_primes(128), N.BUILD_PRODUCTION, download=False)
c4 = best(2, 100000, k=4)
print(json.dumps({"C5": full, "C5_shard4_worst": worst4, "eff4": full / 4 / worst4,
                  "C5_shard8_worst": worst8, "eff8": full / 8 / worst8, "C4": c4}))
'''
KNOBS = ("CUBOID_DRAIN_ALPHA", "CUBOID_POOL_FRAC", "CUBOID_POOL_DIV", "CUBOID_ROW_COST")
for spec in sys.argv[1].split(","):  # LIB[@ALPHA[@POOL_FRAC[@POOL_DIV[@ROW_COST]]]] (empty = default)
    lib, *knobs = spec.split("@")
    env = dict(os.environ, ROOT=ROOT)
    for name, v in zip(KNOBS, knobs):
        if v:
            env[name] = v
    if lib != "default":
        env["CUBOID_GPU_LIB"] = os.path.join(ROOT, lib)
    r = subprocess.run([sys.executable, "-c", CHILD], env=env, capture_output=True, text=True)
    print(spec, r.stdout.strip() if r.returncode == 0 else r.stderr[-400:], flush=True)
