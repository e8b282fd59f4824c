"""Structured LP inputs whose answers are known in closed form (test fixtures).

Only inputs are built here; the expected answers are written out in the tests,
each citing where it comes from.  Nothing here performs a simplex step.

* textbook LPs ("classic LP"; Chvátal, *Linear Programming*, ch. 2)
* Klee–Minty cube (Klee & Minty 1972): Dantzig's rule visits all 2^n vertices
* diagonal LPs: A = diag(d) — every pivot is independent
* planted-optimum dense LPs: x*, y* chosen first, b and c built to satisfy
  complementary slackness, so obj = c^T x* = b^T y* by construction
* tie-heavy small-integer LPs (exercise both tie-breaks)
* Beale's cycling example (Beale 1955)
"""
from __future__ import annotations

import numpy as np

from . import uniform01


def classic():
    """max 3x1 + 5x2 s.t. x1 <= 4, 2x2 <= 12, 3x1 + 2x2 <= 18."""
    A = np.array([[1.0, 0.0], [0.0, 2.0], [3.0, 2.0]])
    b = np.array([4.0, 12.0, 18.0])
    c = np.array([3.0, 5.0])
    return A, b, c


def chvatal():
    """Chvátal, Linear Programming (1983), ch. 2: max 5x1+4x2+3x3."""
    A = np.array([[2.0, 3.0, 1.0], [4.0, 1.0, 2.0], [3.0, 4.0, 2.0]])
    b = np.array([5.0, 11.0, 8.0])
    c = np.array([5.0, 4.0, 3.0])
    return A, b, c


def unbounded_1d():
    """max x s.t. -x <= 1."""
    return np.array([[-1.0]]), np.array([1.0]), np.array([1.0])


def beale():
    """Beale (1955): max 3/4 x1 - 150 x2 + 1/50 x3 - 6 x4, cycles under Dantzig."""
    A = np.array([[0.25, -60.0, -1.0 / 25.0, 9.0],
                  [0.5, -90.0, -1.0 / 50.0, 3.0],
                  [0.0, 0.0, 1.0, 0.0]])
    b = np.array([0.0, 0.0, 1.0])
    c = np.array([0.75, -150.0, 1.0 / 50.0, -6.0])
    return A, b, c


def klee_minty(n: int):
    """max sum_j 2^(n-j) x_j  s.t.  2*sum_{j<i} 2^(i-j) x_j + x_i <= 5^i  (1-based i, j).

    All data are exact integers < 2^53 for n <= 20."""
    A = np.zeros((n, n))
    b = np.zeros(n)
    c = np.zeros(n)
    for i in range(1, n + 1):
        for j in range(1, i):
            A[i - 1, j - 1] = 2.0 * 2.0 ** (i - j)
        A[i - 1, i - 1] = 1.0
        b[i - 1] = 5.0 ** i
    for j in range(1, n + 1):
        c[j - 1] = 2.0 ** (n - j)
    return A, b, c


def diagonal(m: int, seed: int):
    """A = diag(d), d_i in {1,2,4} (powers of two keep b_i/d_i exact), integer b, c.

    Costs are distinct so the entering order is unique."""
    rng = np.random.default_rng(seed)
    d = rng.choice([1.0, 2.0, 4.0], size=m)
    b = rng.integers(1, 100, size=m).astype(np.float64)
    c = rng.permutation(np.arange(1, m + 1)).astype(np.float64)
    return np.diag(d), b, c


def tie_heavy(m: int, n: int, seed: int):
    """Small-integer LP: A in {0..3}, b in {0..5}, c in {0..3} — many exact ties."""
    rng = np.random.default_rng(seed)
    A = rng.integers(0, 4, size=(m, n)).astype(np.float64)
    b = rng.integers(0, 6, size=m).astype(np.float64)
    c = rng.integers(0, 4, size=n).astype(np.float64)
    return A, b, c


def planted(m: int, n: int, seed: int, support: int):
    """Dense LP with a planted optimum.

    A ~ U[1,10) (SplitMix64 draws of ``seed``), support sets S (columns) and R
    (rows) with |S| = |R| = support, x*_S, y*_R ~ U[1,2), slack s (s_R = 0,
    else U[1,10)), reduced cost d (d_S = 0, else U[1,10)):
        b = A x* + s,   c = A^T y* - d.
    Then x* is primal feasible, y* dual feasible and complementary, so
    obj* = c^T x* = b^T y*.  Returns (A, b, c, x_star, y_star)."""
    u = uniform01(seed, 0, m * n + 2 * support + m + n)
    A = (u[: m * n] * 9.0 + 1.0).reshape(m, n)
    rng = np.random.default_rng(seed)
    S = np.sort(rng.choice(n, size=support, replace=False))
    R = np.sort(rng.choice(m, size=support, replace=False))
    x = np.zeros(n)
    y = np.zeros(m)
    x[S] = 1.0 + u[m * n: m * n + support]
    y[R] = 1.0 + u[m * n + support: m * n + 2 * support]
    s = 1.0 + 9.0 * u[m * n + 2 * support: m * n + 2 * support + m]
    s[R] = 0.0
    d = 1.0 + 9.0 * u[m * n + 2 * support + m:]
    d[S] = 0.0
    b = A @ x + s
    c = A.T @ y - d
    return A, b, c, x, y


def with_lower_bounds(m: int, n: int, seed: int, frac: float = 0.1, eq: int = 0):
    """The dense generator LP (lpgen.dense_lp) with a fraction `frac` of its rows turned into
    "at least" rows  -a_i x <= -t_i  (b_i < 0: Phase I needs an artificial for each), plus `eq`
    equality constraints a_i x = t_i written as the pair  a_i x <= t_i  (row i, replacing a
    generator row) and  -a_i x <= -t_i  (appended, so its index is higher).  When Phase I pivots
    in such a pair the ratio tie goes to the lower row (reading c4), the "<=" copy leaves, and the
    appended row ends Phase I as  -s_j - s_i + art_j = 0  with its artificial basic at zero: the
    drive-out (reading p4) must pivot it out on column s_i.

    Feasibility by construction: x0 = (1/(20 n)) * ones satisfies every "<=" row (a_i x0 <= 0.5
    < n <= b_i); t_i = a_i x0 / 2 makes x0 strictly feasible for the ">=" rows; the
    equality rows use t_i = a_i x0 (x0 satisfies them)."""
    from . import dense_lp
    A, b, c = dense_lp(m, n, seed)
    rng = np.random.default_rng(seed + 7919)
    rows = np.sort(rng.choice(m, size=max(1, int(round(frac * m))), replace=False))
    x0 = np.full(n, 1.0 / (20.0 * n))
    t = 0.5 * (A[rows] @ x0)
    A = A.copy()
    b = b.copy()
    A[rows] = -A[rows]
    b[rows] = -t
    if eq:
        free = np.setdiff1d(np.arange(m), rows)[:eq]
        te = A[free] @ x0
        b[free] = te
        A = np.vstack([A, -A[free]])
        b = np.concatenate([b, -te])
    return A, b, c
