"""A/B timing of sieve variants on one GPU: libraries (CUBOID_GPU_LIB) x
row-cost charges (CUBOID_ROW_COST) x workloads. Prints min sieve-kernel ms."""
import itertools
import json
import os
import subprocess
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
CHILD = r'''
import sys, os, json
sys.path.insert(0, os.environ["ROOT"])
from paper_1601_00636_b200 import device as D, _native as N, odd_primes
cfg = {"C3": (64, 2, 10000), "C4": (128, 2, 100000), "C5": (256, 100001, 300000),
       "T50k": (256, 2, 50000), "T150k": (256, 50001, 150000), "T200k": (256, 100001, 200000),
       "R5k": (96, 152, 5000)}
dev = D.Device(0)
out = {}
for name in sys.argv[1].split(","):
    k, lo, hi = cfg[name]
    dev.build(odd_primes(k), N.BUILD_PRODUCTION, download=False)
    t = []
    mode = N.REGION if name.startswith("R") else N.TRIANGLE
    for _ in range(5):
        r = dev.sieve(lo, hi, mode)
        t.append(dev.timings_ms()["sieve"])
    out[name] = (min(t[1:]), r.pairs_tested)
print(json.dumps(out))
'''


def main():
    libs = sys.argv[1].split(",")
    costs = sys.argv[2].split(",")
    wls = sys.argv[3] if len(sys.argv) > 3 else "C4,C5"
    regs = sys.argv[4].split(",") if len(sys.argv) > 4 else ["8"]
    reg3 = sys.argv[5].split(",") if len(sys.argv) > 5 else ["4"]
    for lib, cost, nreg, nr3 in itertools.product(libs, costs, regs, reg3):
        env = dict(os.environ, ROOT=ROOT, CUBOID_ROW_COST=cost, CUBOID_MAX_REG_PROBES=nreg,
                   CUBOID_REG3_PROBES=nr3)
        if lib != "default":
            env["CUBOID_GPU_LIB"] = os.path.join(ROOT, lib)
        r = subprocess.run([sys.executable, "-c", CHILD, wls], env=env, capture_output=True, text=True)
        res = json.loads(r.stdout.strip().splitlines()[-1]) if r.returncode == 0 else r.stderr[-500:]
        print(f"lib={lib} row_cost={cost} reg2={nreg} reg3={nr3} {res}", flush=True)


if __name__ == "__main__":
    main()
