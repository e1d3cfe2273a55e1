"""Synthetic inputs shared by tests, the bench and the checkers.

SplitMix64 exactly as the reference defines it (proj/include/hmat/core.hpp:128-148),
vectorised with numpy uint64 wrap-around arithmetic.  The draw conventions are
the reference's own:

* points: ``SplitMix64(seed)``, point-major -- ``for i<N: for a<d: coords[a][i] =
  uniform()`` (proj/tests/test_tree.cpp:30-42);
* vectors: ``SplitMix64(seed).symmetric()`` in [-1,1)
  (proj/tools/hmat_cli.cpp:74-79, proj/tests/test_hmatrix.cpp:15-20).

This module only generates inputs; it is imported by the product-facing bench as
well, so it must not (and does not) touch any checker.
"""
from __future__ import annotations

import numpy as np

_GOLDEN = np.uint64(0x9E3779B97F4A7C15)
_M1 = np.uint64(0xBF58476D1CE4E5B9)
_M2 = np.uint64(0x94D049BB133111EB)


def splitmix64_stream(seed: int, count: int, start: int = 0) -> np.ndarray:
    """The ``count`` successive ``next()`` outputs of SplitMix64(seed), skipping ``start``."""
    with np.errstate(over="ignore"):
        k = np.arange(start + 1, start + count + 1, dtype=np.uint64)
        z = np.uint64(seed) + k * _GOLDEN
        z = (z ^ (z >> np.uint64(30))) * _M1
        z = (z ^ (z >> np.uint64(27))) * _M2
        return z ^ (z >> np.uint64(31))


def uniform(seed: int, count: int, start: int = 0) -> np.ndarray:
    """``SplitMix64::uniform()`` -- (next() >> 11) * 2^-53, exact in float64."""
    return (splitmix64_stream(seed, count, start) >> np.uint64(11)).astype(np.float64) * (2.0 ** -53)


def symmetric(seed: int, count: int) -> np.ndarray:
    """``SplitMix64::symmetric()`` -- 2*uniform()-1."""
    return 2.0 * uniform(seed, count) - 1.0


def uniform_points(n: int, d: int, seed: int = 42) -> np.ndarray:
    """SoA coordinates, shape (d, n), point-major draw order."""
    return np.ascontiguousarray(uniform(seed, n * d).reshape(n, d).T)


def axis_major_points(n: int, d: int, seed: int) -> np.ndarray:
    """SoA coordinates drawn axis by axis (proj/tests/test_morton.cpp:25-32)."""
    return np.ascontiguousarray(uniform(seed, n * d).reshape(d, n))


def halton_points(n: int, d: int) -> np.ndarray:
    """First n Halton points, bases = first d primes, index from 1, unscrambled,
    with the reference's exact accumulation order (proj/src/core.cpp:16-26, 104-122)."""
    primes = [2, 3, 5, 7, 11, 13, 17, 19, 23, 29, 31, 37, 41, 43, 47, 53, 59, 61, 67, 71]
    out = np.empty((d, n), dtype=np.float64)
    for a in range(d):
        base = primes[a]
        inv = 1.0 / base
        idx = np.arange(1, n + 1, dtype=np.int64)
        value = np.zeros(n)
        factor = np.full(n, inv)
        while np.any(idx > 0):
            live = idx > 0
            value = np.where(live, value + factor * (idx % base).astype(np.float64), value)
            idx = idx // base
            factor = np.where(live, factor * inv, factor)
        out[a] = value
    return out
