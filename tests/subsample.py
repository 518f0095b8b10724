"""C4's seeded 10^6-pair subsample: p drawn with weight phi(p)
over 2 <= p <= 10^5 (the row's candidate count), q uniform among the
integers in [1, p) coprime to p. Test infrastructure: the golden generator
(tests/golden/make_golden.py C4S, first-killer ranks from oracle/_ref) and the
GPU test draw the same pairs from numpy's PCG64 with the recorded seed.
"""
from __future__ import annotations

import numpy as np

SEED = 20160401  # the reference's seed style (test_modpoly.cpp:100)
N_PAIRS = 10**6
P_MAX = 100000


def totients(n: int) -> np.ndarray:
    """phi(k) for k = 0..n (phi(0) = 0)."""
    phi = np.arange(n + 1, dtype=np.int64)
    for k in range(2, n + 1):
        if phi[k] == k:  # k prime: untouched so far
            phi[k::k] -= phi[k::k] // k
    phi[0] = 0
    return phi


def sample(n: int = N_PAIRS, seed: int = SEED, p_max: int = P_MAX) -> np.ndarray:
    """(n, 2) uint64 array of (p, q): p ~ phi(p) over [2, p_max], q uniform
    among the coprime residues of p in [1, p)."""
    rng = np.random.Generator(np.random.PCG64(seed))
    w = totients(p_max)[2:]
    cdf = np.cumsum(w)
    u = rng.integers(0, int(cdf[-1]), n, dtype=np.int64)
    p = 2 + np.searchsorted(cdf, u, side="right").astype(np.int64)
    q = np.zeros(n, np.int64)
    todo = np.arange(n)
    while len(todo):  # rejection sampling: uniform over [1, p), keep the coprime draws
        cand = rng.integers(1, p[todo], dtype=np.int64)
        ok = np.gcd(cand, p[todo]) == 1
        q[todo[ok]] = cand[ok]
        todo = todo[~ok]
    return np.stack([p, q], 1).astype(np.uint64)
