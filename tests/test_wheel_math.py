"""The arithmetic of the wheel sieve (csrc/sieve.cu k_wsieve, K2w) restated in plain
Python and checked against the C oracle on the CPU: alive classes of q mod 2431, stride-2431
windows with their coprimality masks (both factor paths), the analytic first-kill counts of
11, 13, 17 by inclusion-exclusion, and the constants the kernel relies on. The kernel itself is
checked on the GPU (tests/test_gpu_wheel.py); this file pins the algorithm where no GPU is needed."""
from __future__ import annotations

import math
import random

import numpy as np
import pytest

from oracle import port
from paper_1601_00636_b200.primes import odd_primes

M = 2431            # kWheelM = 11 * 13 * 17
CHUNK = 32 * M      # kWheelChunk
DIV_MUL = 1766750   # kWheelDivMul: floor(x / 2431) = (x * DIV_MUL) >> 32 for x < 2^20
E143, E17 = 1717, 715
MID_MAX = 37681     # kWheelMidMax


def _tables(P):
    tb, offs = port.build_set(P)
    rows = {}
    for k, r in enumerate(P):
        n = (r * r + 7) // 8
        bits = np.unpackbits(np.frombuffer(tb[int(offs[k]):int(offs[k]) + n], np.uint8), bitorder="little")[:r * r]
        rows[r] = bits.reshape(r, r)
    return tb, offs, rows


def _prime_factors(p):
    out, d = [], 2
    while d * d <= p:
        if p % d == 0:
            out.append(d)
            while p % d == 0:
                p //= d
        d += 1
    if p > 1:
        out.append(p)
    return out


def test_constants():
    assert M == 11 * 13 * 17 and E143 % 143 == 1 and E143 % 17 == 0 and E17 % 17 == 1 and E17 % 143 == 0
    assert all((x * DIV_MUL) >> 32 == x // M for x in range(0, 1 << 20, 7))
    assert all((x * DIV_MUL) >> 32 == x // M for x in range(CHUNK - 5000, CHUNK + 5000))
    assert 2 * (MID_MAX - 1) ** 2 < 2 ** 32 and 2 * MID_MAX > 31 * M  # lazy product fits; two multiples at most above
    for n17 in range(1, 18):  # the kernel's division of a class index by the mod-17 list length
        rcp = 65536 // n17 + 1
        assert all((c * rcp) >> 16 == c // n17 for c in range(2432))


def _mask_mid(q0, f):
    """First i with f | q0 + 2431 i is (q0 mod f) g mod f, g = -(2431^-1) mod f, from the two
    small inverse tables ((1 + f k) / 143 with k = (-f^-1) mod 143, likewise 17)."""
    k143 = next(y for y in range(1, 143) if (f % 143 * y) % 143 == 142)
    k17 = next(y for y in range(1, 17) if (f % 17 * y) % 17 == 16)
    i143, i17 = (1 + f * k143) // 143, (1 + f * k17) // 17
    assert (1 + f * k143) % 143 == 0 and (143 * i143) % f == 1 and (17 * i17) % f == 1
    g = f - (i143 * i17) % f
    t = q0 % f + (f if q0 % 3 == 0 else 0)  # a lazy remainder in [0, 2f)
    assert t * g < 2 ** 32
    i0 = (t * g) % f
    pat = sum(1 << i for i in range(0, 32, f)) if f < 32 else 1
    return (pat << i0) & 0xffffffff if i0 < 32 else 0


def _mask_large(q0, f):
    t = q0 % f
    d = f - t if t else 0
    m = 0
    for _ in range(2):
        i = (min(d, CHUNK) * DIV_MUL) >> 32
        if i * M == d and i < 32:
            m |= 1 << i
        d += f
        if d >= 2 ** 32:
            d = CHUNK + 1
    return m


def test_coprimality_masks_of_stride_windows():
    rng = random.Random(5)
    primes = [f for f in range(3, 120000) if all(f % d for d in range(2, int(f ** 0.5) + 1)) and f not in (11, 13, 17)]
    for _ in range(4000):
        f = rng.choice(primes) if rng.random() < 0.8 else rng.choice([3, 5, 7, 19, 23, 29, 31, 37679, 37691, 77801])
        q0 = rng.randrange(1, 2 ** 32 - 31 * M)
        want = sum(1 << i for i in range(32) if (q0 + M * i) % f == 0)
        got = _mask_mid(q0, f) if f < MID_MAX else _mask_large(q0, f)
        assert got == want, (f, q0)


def _wheel_row(rows, P, p, qa, qb):
    """First-kill counts by rank for q in [qa, qb] of row p the way k_wsieve forms them."""
    hist = np.zeros(len(P), np.int64)
    a = {r: p % r for r in (11, 13, 17)}
    alive = {r: [b for b in range(r) if not rows[r][a[r]][b]] for r in (11, 13, 17)}
    facs = [f for f in _prime_factors(p) if f <= qb]
    # S0, S1, S2 by inclusion-exclusion over the squarefree divisors d: q = d t, t in [t0, t1]
    S = [0, 0, 0]
    for sub in range(1 << len(facs)):
        d = math.prod(f for i, f in enumerate(facs) if sub >> i & 1)
        if d > qb:
            continue
        t0, t1 = (qa - 1) // d + 1, qb // d
        if t1 < t0:
            continue
        sign = -1 if bin(sub).count("1") & 1 else 1
        n = t1 - t0 + 1
        B11 = [rho for rho in range(11) if (d * rho) % 11 in alive[11]]
        P143 = [rho for rho in range(143) if (d * rho) % 11 in alive[11] and (d * rho) % 13 in alive[13]]
        c1 = (n // 11) * len(B11) + sum(1 for i in range(n % 11) if (t0 + i) % 11 in B11)
        c2 = (n // 143) * len(P143) + sum(1 for i in range(n % 143) if (t0 + i) % 143 in P143)
        S[0] += sign * n
        S[1] += sign * c1
        S[2] += sign * c2
    # alive classes (class 0 of a wheel prime that divides p holds no coprime q), stride windows
    l143 = [o for o in range(143) if (qa + o) % 11 in alive[11] and (qa + o) % 13 in alive[13]
            and not (a[11] == 0 and (qa + o) % 11 == 0) and not (a[13] == 0 and (qa + o) % 13 == 0)]
    l17 = [o for o in range(17) if (qa + o) % 17 in alive[17] and not (a[17] == 0 and (qa + o) % 17 == 0)]
    S3 = 0
    surv = []
    rank = {r: k for k, r in enumerate(P)}
    for o143 in l143:
        for o17 in l17:
            o = (o143 * E143 + o17 * E17) % M
            q = qa + o
            while q <= qb:
                if math.gcd(p, q) == 1:
                    S3 += 1
                    for r in P[P.index(19):]:
                        if rows[r][p % r][q % r] and p % r:
                            hist[rank[r]] += 1
                            break
                    else:
                        surv.append(q)
                q += M
    hist[rank[11]], hist[rank[13]], hist[rank[17]] = S[0] - S[1], S[1] - S[2], S[2] - S3
    return hist, sorted(surv), S[0]


@pytest.mark.parametrize("mode,p,q_start", [
    (port.TRIANGLE, 2431, 0), (port.TRIANGLE, 187 * 13, 0), (port.TRIANGLE, 1001, 0),
    (port.TRIANGLE, 2 * 3 * 5 * 7 * 11, 0), (port.TRIANGLE, 1619, 0), (port.TRIANGLE, 2048, 0),
    (port.TRIANGLE, 3 * 17 * 19, 0), (port.TRIANGLE, 221, 0), (port.TRIANGLE, 4862, 0), (port.TRIANGLE, 30, 0),
    (port.REGION, 152, 0), (port.REGION, 187, 0), (port.REGION, 221, 3000), (port.REGION, 330, 0),
    (port.REGION, 143, 0)])
def test_wheel_row_equals_the_oracle(mode, p, q_start):
    """One row, the way k_wsieve forms its counts, against the C oracle: rows the wheel primes
    divide (whole classes alive, class 0 dropped), rows shorter than a class period, REGION rows
    (q_low(p) <= q <= 59 p, also from a mid-row start)."""
    P = odd_primes(40)
    tb, offs, rows = _tables(P)
    for r in (3, 5, 7):  # never kill (the device skips them); row 0 never kills in scan()
        assert not rows[r].any()
    if mode == port.TRIANGLE:
        qa, qb = 1, p - 1
    else:
        qa, qb = port.q_bounds(p)
        qa = q_start or qa
    o = port.sieve(tb, P, offs, p, p, mode, q_start=q_start)
    hist, surv, cand = _wheel_row(rows, P, p, qa, qb)
    assert cand == o["pairs_tested"]
    assert hist.tolist() == np.asarray(o["hist"]).tolist()
    assert surv == [int(q) for pp, q in np.asarray(o["survivor_pairs"]).reshape(-1, 2)]
