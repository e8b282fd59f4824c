"""The latency path for small tableaux (k_solve_small): the whole solve in ONE launch of ONE
CTA with the tableau in shared memory (on small LPs communication and
reductions dominate).  Selected automatically (lookahead = 0) when the tableau fits in one
CTA's shared memory, on one column part, without Phase I; stats().path == 1 proves which
path ran.  Bar: bit-identical to the oracle (trace, objective, x, y, whole tableau).
Seeds 1..100 of the 64x64 config are SURVEY.md §8(d)'s seed list for that config.
"""
import json
import os

import numpy as np
import pytest

import lpgen
import oracle
from lpgen import fixtures as F

pytestmark = pytest.mark.gpu

GOLD = json.load(open(os.path.join(os.path.dirname(__file__), "golden", "worked_examples.json")))


@pytest.fixture(scope="module")
def sx(cuda_device):
    import paper_2211_10979_b200 as sx
    return sx


def small_solve(sx, A, b, c, expect_path=1, **kw):
    with sx.Simplex(A, b, c, **kw) as s:
        assert s.stats().path == expect_path
        st = s.solve()
        x, y, obj, piv, st2 = s.solution()
        k, r = s.trace()
        T, _ = s.tableau()
        h = s.tableau_hash()
        assert s.stats().kernel_launches >= 1
    assert st == st2
    return dict(status=st, x=x, y=y, obj=obj, pivots=piv, k=k, r=r, T=T, hash=h)


def assert_same(g, o):
    assert g["status"] == o.status and g["pivots"] == o.pivots
    assert np.array_equal(g["k"], o.trace_k) and np.array_equal(g["r"], o.trace_r)
    assert g["obj"] == o.objective
    assert np.array_equal(g["x"], o.x) and np.array_equal(g["y"], o.y)
    assert np.array_equal(g["T"], o.T)
    assert g["hash"] == oracle.tableau_hash(o.T)


@pytest.mark.parametrize("seed", range(1, 101))
def test_dense_64_seeds(sx, seed):
    A, b, c = lpgen.dense_lp(64, 64, seed)
    assert_same(small_solve(sx, A, b, c), oracle.solve(A, b, c, keep_tableau=True))


def test_dense_64_golden_row(sx):
    """SURVEY.md §8(c) golden row (64, 64, 1): 24 pivots, objective 0x1.c9320127cef55p+6."""
    A, b, c = lpgen.dense_lp(64, 64, 1)
    g = small_solve(sx, A, b, c)
    assert g["pivots"] == 24 and float(g["obj"]).hex() == "0x1.c9320127cef55p+6"


@pytest.mark.parametrize("name", ["classic", "chvatal", "unbounded", "beale", "entering_tie", "ratio_tie",
                                  "zero_iteration"])
def test_worked_examples(sx, name):
    fix = {"classic": F.classic, "chvatal": F.chvatal, "unbounded": F.unbounded_1d, "beale": F.beale}
    if name in fix:
        A, b, c = fix[name]()
    else:
        g = GOLD[name]
        A, b, c = (np.array(g[k], float) for k in ("A", "b", "c"))
    kw = {"max_pivots": 30} if name == "beale" else {}
    assert_same(small_solve(sx, A, b, c, **kw), oracle.solve(A, b, c, keep_tableau=True, **kw))


@pytest.mark.parametrize("seed", range(8))
def test_tie_heavy_both_rules(sx, seed):
    A, b, c = F.tie_heavy(20 + seed, 31 - seed, 700 + seed)
    assert_same(small_solve(sx, A, b, c), oracle.solve(A, b, c, keep_tableau=True))
    assert_same(small_solve(sx, A, b, c, pivot_rule=sx.BLAND),
                oracle.solve(A, b, c, keep_tableau=True, rule=oracle.BLAND))


def test_klee_minty_exact(sx):
    """Klee–Minty n=10: exactly 2^10 - 1 pivots, optimum 5^10 (closed form)."""
    A, b, c = F.klee_minty(10)
    g = small_solve(sx, A, b, c, max_pivots=2000)
    assert g["pivots"] == 1023 and g["obj"] == 5.0 ** 10
    assert_same(g, oracle.solve(A, b, c, keep_tableau=True, max_pivots=2000))


def test_iterate_windows_match_oracle_prefixes(sx):
    """simplex_iterate on the one-launch path: stop exactly at each window end, tableau equal to
    the oracle's prefix run there; termination reported at the start of the next call."""
    A, b, c = lpgen.dense_lp(64, 64, 3)
    o = oracle.solve(A, b, c, keep_tableau=True)
    with sx.Simplex(A, b, c) as s:
        assert s.stats().path == 1
        total = 0
        while True:
            done, st = s.iterate(5)
            total += done
            T, _ = s.tableau()
            ref = oracle.solve(A, b, c, keep_tableau=True, stop_after=total)
            assert np.array_equal(T, ref.T), total
            if st != sx.RUNNING:
                break
        assert total == o.pivots and st == o.status
        assert s.iterate(5) == (0, st)


def test_reset_and_resolve(sx):
    A, b, c = lpgen.dense_lp(40, 50, 8)
    A2, b2, c2 = lpgen.dense_lp(40, 50, 9)
    o1, o2 = oracle.solve(A, b, c), oracle.solve(A2, b2, c2)
    with sx.Simplex(A, b, c) as s:
        assert s.solve() == o1.status and s.solution()[2] == o1.objective
        s.reset(A2, b2, c2)
        assert s.solve() == o2.status and s.solution()[2] == o2.objective
        assert np.array_equal(s.trace()[0], o2.trace_k)


def test_largest_fitting_and_first_not_fitting(sx):
    """100x150 (101 x 251 doubles = 203 KB) runs on the one-CTA path; a tableau beyond one CTA's
    shared memory falls back to the device loop (path 0) — both bit-identical."""
    A, b, c = lpgen.dense_lp(100, 150, 4)
    assert_same(small_solve(sx, A, b, c), oracle.solve(A, b, c, keep_tableau=True))
    A, b, c = lpgen.dense_lp(120, 150, 4)
    assert_same(small_solve(sx, A, b, c, expect_path=0), oracle.solve(A, b, c, keep_tableau=True))


def test_explicit_lookahead_keeps_device_loop(sx):
    """An explicit lookahead (1 or 16) keeps the graph-segment loop even on a tiny tableau, so the
    other kernels stay testable at small sizes."""
    A, b, c = lpgen.dense_lp(64, 64, 5)
    o = oracle.solve(A, b, c, keep_tableau=True)
    for look in (1, 16):
        assert_same(small_solve(sx, A, b, c, expect_path=0, lookahead=look), o)


def test_phase1_and_virtual_ranks_use_device_loop(sx):
    A, b, c = lpgen.dense_lp(30, 40, 6)
    b2 = b.copy()
    b2[3] = -1.0
    with sx.Simplex(A, b2, c) as s:
        assert s.stats().path == 0
    with sx.Simplex(A, b, c, virtual_ranks=2) as s:
        assert s.stats().path == 0
