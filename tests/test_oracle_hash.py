"""Pins for oracle.tableau_hash — the whole-tableau digest that is the only
whole-tableau check at 4000², 8000² and 20000x40000 (VERDICT r1 "parity unpinned:
oracle.tableau_hash").  A digest is only a check if a plausible divergence changes it,
so these tests pin its SENSITIVITY and its INVARIANCES, not its value:

* its mixing function is SplitMix64's finaliser: pinned by the published SplitMix64
  output for seed 0 (0xe220a8397b1dcdaf) and the survey's independently computed raw
  outputs for seed 1 (0x910a2dec89025cc1, 0xbeeb8da1658eec67, ...);
* a one-ulp change of ANY single element changes it (every position of a tableau);
* swapping two unequal elements, permuting two rows, or transposing a square tableau
  changes it (the element index is bound into each term);
* -0.0 and +0.0 hash the same (reading c16: signed zeros never decide anything);
* it does not depend on the chunking used to compute it.
"""
import numpy as np
import pytest

import lpgen
import oracle

G = np.uint64(0x9E3779B97F4A7C15)


def test_mix_is_splitmix64_finaliser():
    with np.errstate(over="ignore"):
        assert int(oracle._mix64(np.uint64(0) + G)) == 0xE220A8397B1DCDAF
        outs = [int(oracle._mix64(np.uint64(1) + np.uint64(i) * G)) for i in (1, 2, 3)]
    assert outs == [0x910A2DEC89025CC1, 0xBEEB8DA1658EEC67, 0xF893A2EEFB32555E]


def small_tableau(seed=3):
    A, b, c = lpgen.dense_lp(12, 17, seed)
    T, _ = oracle.build_tableau(A, b, c)
    T = oracle.pivot(T, 4, 5)                 # a non-trivial, non-integer tableau
    return T


def test_one_ulp_anywhere_changes_hash():
    T = small_tableau()
    h0 = oracle.tableau_hash(T)
    for i in range(T.shape[0]):
        for j in range(T.shape[1]):
            U = T.copy()
            U[i, j] = np.nextafter(U[i, j], np.inf)
            assert oracle.tableau_hash(U) != h0, (i, j)
            U[i, j] = np.nextafter(T[i, j], -np.inf)
            assert oracle.tableau_hash(U) != h0, (i, j)


def test_swaps_permutations_transpose_change_hash():
    T = small_tableau()
    h0 = oracle.tableau_hash(T)
    rng = np.random.default_rng(0)
    for _ in range(200):
        i1, i2 = rng.integers(0, T.shape[0], 2)
        j1, j2 = rng.integers(0, T.shape[1], 2)
        if T[i1, j1] == T[i2, j2]:
            continue
        U = T.copy()
        U[i1, j1], U[i2, j2] = T[i2, j2], T[i1, j1]
        assert oracle.tableau_hash(U) != h0
    U = T.copy()
    U[[2, 7]] = U[[7, 2]]
    assert oracle.tableau_hash(U) != h0
    S = np.arange(36, dtype=np.float64).reshape(6, 6) * 0.37
    assert oracle.tableau_hash(S) != oracle.tableau_hash(np.ascontiguousarray(S.T))


def test_signed_zero_invariance_and_zero_vs_tiny():
    T = small_tableau()
    T[3, 3] = 0.0
    h0 = oracle.tableau_hash(T)
    U = T.copy()
    U[3, 3] = -0.0
    assert oracle.tableau_hash(U) == h0
    U[3, 3] = 5e-324                          # the smallest subnormal is NOT zero
    assert oracle.tableau_hash(U) != h0


@pytest.mark.parametrize("chunk", [1, 3, 7, 256])
def test_chunking_independent(chunk):
    T = small_tableau(5)
    assert oracle.tableau_hash(T, chunk_rows=chunk) == oracle.tableau_hash(T)


def test_shape_bound_into_hash():
    """Same values, different logical width -> different element indices -> different hash."""
    v = np.linspace(1.0, 2.0, 24)
    assert oracle.tableau_hash(v.reshape(4, 6)) == oracle.tableau_hash(v.reshape(4, 6).copy())
    # e = i*W + j is the same for a pure reshape, so equal — the index is the row-major position
    assert oracle.tableau_hash(v.reshape(4, 6)) == oracle.tableau_hash(v.reshape(6, 4))
    w = v.copy()
    w[[0, 23]] = w[[23, 0]]
    assert oracle.tableau_hash(w.reshape(4, 6)) != oracle.tableau_hash(v.reshape(4, 6))
