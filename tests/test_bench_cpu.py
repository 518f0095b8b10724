"""bench.py's host logic on the CPU: the `--gpus N` self-launch (N ranks
through torch.distributed.run, gloo here) and the parity flag, which compares
a step's result with the reference's full-range golden statistics."""
from __future__ import annotations

import json
import os
import subprocess
import sys

import numpy as np
import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import bench  # noqa: E402
from paper_1601_00636_b200.primes import odd_primes  # noqa: E402


def test_gpus_flag_self_launches_ranks():
    """`python bench.py --gpus 2` with WORLD_SIZE unset starts 2 ranks itself
    (the driver's form, BENCH_r01.cmd); rank 0 reports the world it saw."""
    env = {k: v for k, v in os.environ.items() if k not in ("WORLD_SIZE", "RANK", "LOCAL_RANK")}
    out = subprocess.run([sys.executable, os.path.join(ROOT, "bench.py"), "--gpus", "2", "--backend", "gloo",
                          "--launch-check"], capture_output=True, text=True, timeout=300, env=env, cwd=ROOT)
    assert out.returncode == 0, out.stderr[-2000:]
    lines = [json.loads(ln) for ln in out.stdout.splitlines() if ln.startswith("{")]
    assert len(lines) == 1
    assert lines[0]["n_gpus"] == 2 and lines[0]["ranks_seen"] == 2 and lines[0]["backend"] == "gloo"
    assert "launching 2 ranks" in out.stderr


@pytest.fixture(scope="module")
def c5_golden():
    g = json.load(open(os.path.join(ROOT, "tests", "golden", "golden.json")))["sieve"]["C5"]
    P = odd_primes(256)
    hist = np.zeros(256, np.int64)
    for k, r in enumerate(P):
        hist[k] = g["kill_histogram"].get(str(r), 0)
    wl = bench.WORKLOADS["C5"]
    blk0 = wl["p_lo"] // 100
    brm = np.zeros(wl["p_hi"] // 100 - blk0 + 1, np.int64)
    for b, v in g["block_r_max"].items():
        brm[int(b) - blk0] = v
    return g, P, hist, brm, wl


def test_parity_flag_accepts_the_reference_result(c5_golden):
    g, P, hist, brm, wl = c5_golden
    r = bench.golden_parity("C5", P, g["pairs_tested"], g["survivors"], hist, brm, wl)
    assert r["ok"] and all(r["checks"].values())


@pytest.mark.parametrize("what", ["hist", "brm", "pairs"])
def test_parity_flag_rejects_any_difference(c5_golden, what):
    """A result that keeps pairs == sum(hist) + survivors (what round 1 checked)
    but moves one kill between primes, or one block's r_max, is a mismatch."""
    g, P, hist, brm, wl = c5_golden
    hist, brm, pairs = hist.copy(), brm.copy(), g["pairs_tested"]
    if what == "hist":
        hist[0] -= 1
        hist[1] += 1
    elif what == "brm":
        brm[17] = 137
    else:
        pairs += 1
        hist[0] += 1
    r = bench.golden_parity("C5", P, pairs, g["survivors"], hist, brm, wl)
    assert not r["ok"]
