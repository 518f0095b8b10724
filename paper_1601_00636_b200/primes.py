"""Prime lists used by the reference and the BASELINE configs."""
from __future__ import annotations


def is_prime(n: int) -> bool:
    """Trial division (include/cuboid/primes.hpp:14-21)."""
    if n < 2:
        return False
    if n % 2 == 0:
        return n == 2
    d = 3
    while d * d <= n:
        if n % d == 0:
            return False
        d += 2
    return True


def primes_in_range(lo: int, hi: int) -> list[int]:
    """Primes in [lo, hi], ascending (primes.hpp:24-30)."""
    return [n for n in range(max(lo, 2), hi + 1) if is_prime(n)]


def odd_primes(k: int) -> list[int]:
    """The first k odd primes (3, 5, 7, ...): the BASELINE.json prime lists."""
    out, n = [], 3
    while len(out) < k:
        if is_prime(n):
            out.append(n)
        n += 2
    return out


def default_primes() -> list[int]:
    """The reference default: the 96 primes 11..541 (sievetable.hpp:178-179)."""
    return primes_in_range(11, 541)
