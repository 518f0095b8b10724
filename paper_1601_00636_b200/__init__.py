"""B200-native residue-table builder and (p,q) pair sieve for the
modulo-primes perfect-cuboid search (arXiv 1601.00636).

Product path: libcuboid_gpu.so (sm_100a CUDA, include/cuboid_gpu.h) through
paper_1601_00636_b200.device / .cuboid. There is no CPU fallback.
"""
from . import _native  # noqa: F401
from .primes import default_primes, odd_primes, primes_in_range  # noqa: F401

__all__ = ["default_primes", "odd_primes", "primes_in_range"]
