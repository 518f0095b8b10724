"""Randomised parity sweep of the device sieve against the C oracle (a tool,
not part of the -m gpu suite): random prime sets (standard 11..37 heads and
generic ones, with and without 3, 5, 7), random TRIANGLE and REGION ranges
with mid-row starts, both loop-variant sets of k_sieve (CUBOID_SHORT_ROWS forced per
context) and the wheel sieve k_wsieve (CUBOID_WHEEL=2), random block-cyclic shards. Prints one line per case and a summary.

    python tools/fuzz_sieve.py [seconds] [seed]
"""
import os
import random
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402

from oracle import port  # noqa: E402  (the checker)
from paper_1601_00636_b200 import _native as N  # noqa: E402
from paper_1601_00636_b200.device import Device  # noqa: E402
from paper_1601_00636_b200.primes import odd_primes, primes_in_range  # noqa: E402


def main():
    budget = float(sys.argv[1]) if len(sys.argv) > 1 else 120.0
    rng = random.Random(int(sys.argv[2]) if len(sys.argv) > 2 else 7)
    devs = {}
    for sr in ("0", "1", "w"):  # "w": the wheel sieve forced on every standard-set launch
        os.environ["CUBOID_SHORT_ROWS"] = "0" if sr == "w" else sr
        os.environ["CUBOID_WHEEL"] = "2" if sr == "w" else "0"
        devs[sr] = Device(0)
    t0, n, bad = time.time(), 0, 0
    while time.time() - t0 < budget:
        kind = rng.choice(["std", "std", "generic", "small"])
        if kind == "std":
            P = odd_primes(rng.choice([32, 64, 96, 128, 200]))
        elif kind == "generic":
            lo = rng.choice([11, 13, 17, 41])
            P = primes_in_range(lo, rng.choice([200, 400, 900]))
        else:
            P = sorted(rng.sample(primes_in_range(11, 300), rng.randrange(1, 6)))
        tb, offs = port.build_set(P)
        sr = rng.choice(["0", "1", "w", "w"])
        dev = devs[sr]
        dev.load(P, tb)
        mode = rng.choice([N.TRIANGLE, N.REGION])
        weak = kind == "small"  # few primes: most pairs survive, keep the ranges small
        if mode == N.TRIANGLE:
            lo = rng.randrange(2, 5000 if weak else 60000)
            hi = lo + rng.randrange(0, 30 if weak else 300)
            q0 = 0
        else:
            lo = rng.randrange(1, 2000 if weak else 20000)
            hi = lo + rng.randrange(0, 3 if weak else 40)
            qlo, qhi = port.q_bounds(lo)
            q0 = rng.choice([0, rng.randrange(qlo, qhi + 1)])
        G = rng.choice([1, 1, 2, 3])
        g = rng.randrange(G)
        r = dev.sieve(lo, hi, mode, q_start=q0, shard=(G, g), surv_cap=1 << 22)
        rows = [(max(lo, 100 * b), min(hi, 100 * b + 99)) for b in range(lo // 100, hi // 100 + 1) if b % G == g]
        pairs = surv = 0
        hist = np.zeros(len(P), np.int64)
        sp = []
        for a, z in rows:
            o = port.sieve(tb, P, offs, a, z, mode, q_start=q0 if a == lo else 0)
            pairs += o["pairs_tested"]
            surv += o["survivors"]
            hist += o["hist"].astype(np.int64)
            sp.extend(map(tuple, o["survivor_pairs"].tolist()))
        ok = (r.pairs_tested == pairs and r.survivors == surv and r.hist.astype(np.int64).tolist() == hist.tolist()
              and [tuple(x) for x in r.survivor_pairs.tolist()] == sp)
        n += 1
        bad += not ok
        print(f"{'ok ' if ok else 'BAD'} {kind:7s} short={sr} mode={'T' if mode else 'R'} "
              f"p={lo}..{hi} q0={q0} shard={G}/{g} primes={len(P)} pairs={pairs}", flush=True)
    print(f"summary: {n} cases, {bad} mismatches, {time.time() - t0:.0f} s")
    return 1 if bad else 0


if __name__ == "__main__":
    sys.exit(main())
