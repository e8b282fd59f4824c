"""The row-parallel oracle build (liboracle_omp.so) is bitwise identical to the
single-thread build (SURVEY.md §8(d) "Oracle baseline" (ii): "That build is bitwise
identical to the 1-thread build, which must be proven on the 64²–4000² configs").

liboracle_omp.so is simplex_oracle.c compiled with -fopenmp; the only parallel loop is
or_pivot's row loop (PAPER.md:94 Step 3), where every element still receives exactly one
fma whose operands are fixed before the loop.  These tests run it with several threads
and compare whole tableaux bit for bit (not via a hash) against the single-thread build,
and the full 4000² trace/hash against the golden the single-thread build wrote.
Only this build writes the 8000² seed-2 and 20000x40000 goldens (scripts/make_golden*.py).
"""
import ctypes as C
import os

import numpy as np
import pytest

import lpgen
from lpgen import fixtures
import oracle

GOLDEN_DIR = os.path.join(os.path.dirname(__file__), "golden")


@pytest.fixture(scope="module", autouse=True)
def threads():
    oracle.lib(parallel=True)
    gomp = C.CDLL("libgomp.so.1")
    gomp.omp_set_num_threads(4)           # force a real split even on a 1-core runner
    gomp.omp_get_max_threads.restype = C.c_int
    assert gomp.omp_get_max_threads() == 4
    yield


def bits(a):
    return np.ascontiguousarray(a).view(np.uint64)


def both(A, b, c, **kw):
    r1 = oracle.solve(A, b, c, keep_tableau=True, **kw)
    r2 = oracle.solve(A, b, c, keep_tableau=True, parallel=True, **kw)
    return r1, r2


def assert_identical(r1, r2):
    assert r1.status == r2.status and r1.pivots == r2.pivots
    assert np.array_equal(r1.trace_k, r2.trace_k) and np.array_equal(r1.trace_r, r2.trace_r)
    assert np.array_equal(bits(r1.T), bits(r2.T))          # every element, every bit (incl. -0)
    assert np.array_equal(bits(r1.x), bits(r2.x)) and np.array_equal(bits(r1.y), bits(r2.y))
    assert np.array_equal(r1.basis, r2.basis)


@pytest.mark.parametrize("seed", range(1, 11))
def test_omp_equals_single_64(seed):
    assert_identical(*both(*lpgen.dense_lp(64, 64, seed)))


@pytest.mark.parametrize("seed", range(5))
def test_omp_equals_single_tie_heavy(seed):
    """Integer tie-heavy LPs (many exact ties in both argmins): any reordering of the row
    loop that leaked into a decision would show here first."""
    assert_identical(*both(*fixtures.tie_heavy(30, 37, 1000 + seed)))


def test_omp_equals_single_bland_and_cap():
    A, b, c = lpgen.dense_lp(200, 300, 7)
    assert_identical(*both(A, b, c, rule=oracle.BLAND))
    assert_identical(*both(A, b, c, max_pivots=50))
    assert_identical(*both(A, b, c, stop_after=33))


def test_omp_equals_single_1000():
    assert_identical(*both(*lpgen.dense_lp(1000, 1000, 1)))


def test_omp_chunked_iterate_equals_solve():
    """or_iterate resumed in chunks (how make_golden_long.py runs) = one uninterrupted solve."""
    A, b, c = lpgen.dense_lp(300, 500, 3)
    ref = oracle.solve(A, b, c, keep_tableau=True)
    T, basis = oracle.build_tableau(A, b, c)
    it, ks, rs, st = 0, [], [], oracle.RUNNING
    while st == oracle.RUNNING:
        st, it, k, r = oracle.iterate(T, basis, it, stop_at=it + 37, parallel=True)
        ks.append(k)
        rs.append(r)
    assert st == ref.status and it == ref.pivots
    assert np.array_equal(np.concatenate(ks), ref.trace_k) and np.array_equal(np.concatenate(rs), ref.trace_r)
    assert np.array_equal(bits(T), bits(ref.T)) and np.array_equal(basis, ref.basis)


def test_omp_4000_against_single_thread_golden():
    """The full 4000² seed-1 solve (8487 pivots) by the row-parallel build against the
    golden the single-thread build wrote (trace, objective bits, y bits, tableau digest)."""
    g = np.load(os.path.join(GOLDEN_DIR, "dense_4000x4000_s1.npz"))
    A, b, c = lpgen.dense_lp(4000, 4000, 1)
    r = oracle.solve(A, b, c, keep_tableau=True, parallel=True)
    assert r.status == int(g["status"]) and r.pivots == int(g["pivots"])
    assert np.array_equal(r.trace_k, g["trace_k"]) and np.array_equal(r.trace_r, g["trace_r"])
    assert bits(np.array(r.objective)) == bits(np.array(float(g["objective"])))
    assert np.array_equal(bits(r.y), bits(g["y"]))
    assert oracle.tableau_hash(r.T) == int(g["tableau_hash"])
