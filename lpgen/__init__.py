"""lpgen — seeded synthetic dense LP inputs shared by the oracle tests and the CUDA path.

This module holds NO arithmetic of the simplex method: it only draws the
inputs (A, b, c) of "randomly generated dense" LPs (§V.B,
"structural properties similar to the ones of [19,33]"; the paper gives no
distribution, so the recipe of SPEC.md:365-380 [generator] is adopted, with
the counter-based generator pinned in SURVEY.md §8(d)):

    draw i (i = 0, 1, 2, ...):  z = seed + (i+1) * 0x9E3779B97F4A7C15  (mod 2^64)
                                z = (z ^ z>>30) * 0xBF58476D1CE4E5B9
                                z = (z ^ z>>27) * 0x94D049BB133111EB
                                z ^= z>>31
    u = (z >> 11) * 2^-53                 in [0, 1), exact
    value = lo + (hi - lo) * u            multiply, then add (two roundings, no FMA)
    order: A row-major (draws 0 .. m*n-1), then b (m draws), then c (n draws)
    A, c: lo = 1, hi = 10      b: lo = n, hi = 2n      sense: maximize

Because the generator is counter-based, any sub-block (a row range, a column
slab) can be drawn independently and bit-identically — which is how each rank
of a column-partitioned solve could draw only its own columns.

Fixtures with closed-form answers (Klee–Minty, diagonal, planted optimum,
tie-heavy integer LPs, textbook examples) live in ``lpgen.fixtures``.
"""
from __future__ import annotations

import numpy as np

GOLDEN = np.uint64(0x9E3779B97F4A7C15)
MIX1 = np.uint64(0xBF58476D1CE4E5B9)
MIX2 = np.uint64(0x94D049BB133111EB)
_TWO_M53 = float(2.0 ** -53)


def splitmix64(seed: int, first: int, count: int) -> np.ndarray:
    """Raw 64-bit outputs for draws first .. first+count-1 (uint64 array)."""
    with np.errstate(over="ignore"):
        i = np.arange(first + 1, first + count + 1, dtype=np.uint64)
        z = np.uint64(seed & 0xFFFFFFFFFFFFFFFF) + i * GOLDEN
        z = (z ^ (z >> np.uint64(30))) * MIX1
        z = (z ^ (z >> np.uint64(27))) * MIX2
        z = z ^ (z >> np.uint64(31))
    return z


def uniform01(seed: int, first: int, count: int) -> np.ndarray:
    """u = (z >> 11) * 2^-53 for draws first .. first+count-1 (float64, exact)."""
    z = splitmix64(seed, first, count)
    return (z >> np.uint64(11)).astype(np.float64) * _TWO_M53


def _scale(u: np.ndarray, lo: float, hi: float) -> np.ndarray:
    # (hi - lo) * u first, then + lo: numpy never contracts to an FMA.
    return np.add(np.multiply(u, float(hi - lo)), float(lo))


def dense_A_rows(m: int, n: int, seed: int, row0: int, row1: int) -> np.ndarray:
    """Rows [row0, row1) of A (row-major draws 0 .. m*n-1)."""
    assert 0 <= row0 <= row1 <= m
    u = uniform01(seed, row0 * n, (row1 - row0) * n)
    return _scale(u, 1.0, 10.0).reshape(row1 - row0, n)


def dense_lp(m: int, n: int, seed: int, *, chunk_rows: int = 2048):
    """(A, b, c) of the dense random LP (m, n, seed); A is C-contiguous float64 (m, n)."""
    if m < 1 or n < 1:
        raise ValueError("m, n must be >= 1")
    A = np.empty((m, n), dtype=np.float64)
    for r0 in range(0, m, chunk_rows):
        r1 = min(m, r0 + chunk_rows)
        A[r0:r1] = dense_A_rows(m, n, seed, r0, r1)
    b = _scale(uniform01(seed, m * n, m), float(n), float(2 * n))
    c = _scale(uniform01(seed, m * n + m, n), 1.0, 10.0)
    return A, b, c


__all__ = ["splitmix64", "uniform01", "dense_A_rows", "dense_lp"]
