"""GPU parity of Bland's rule (pivot_rule = 1) against the oracle's
or_solve_rule(rule=BLAND): identical traces and bit-identical tableaux on every path (one
pivot per pass, rank-s look-ahead, column slabs)."""
import os

import numpy as np
import pytest

import lpgen
import oracle
from lpgen import fixtures as F

from test_gpu_parity import GOLDEN_DIR, assert_same, gpu_solve

pytestmark = pytest.mark.gpu

PATHS = [dict(lookahead=1), dict(lookahead=4), dict(lookahead=16), dict(lookahead=16, overlap=False),
         dict(lookahead=32), dict(lookahead=1, virtual_ranks=3)]
PATH_IDS = ["pass1", "look4", "look16", "look16serial", "pair32", "slabs3"]


@pytest.fixture(scope="module")
def sx(cuda_device):
    import paper_2211_10979_b200 as sx
    return sx


def bland(A, b, c, **kw):
    return oracle.solve(A, b, c, rule=oracle.BLAND, keep_tableau=True, **kw)


@pytest.mark.parametrize("path", PATHS, ids=PATH_IDS)
def test_beale_terminates(sx, path):
    A, b, c = F.beale()
    o = bland(A, b, c)
    assert o.status == oracle.OPTIMAL and abs(o.objective - 0.05) < 1e-12
    g = gpu_solve(sx, A, b, c, pivot_rule=sx.BLAND, **path)
    assert_same(g, o)


@pytest.mark.parametrize("path", PATHS, ids=PATH_IDS)
@pytest.mark.parametrize("seed", range(8))
def test_tie_heavy(sx, seed, path):
    rng = np.random.default_rng(100 + seed)
    m, n = int(rng.integers(3, 40)), int(rng.integers(3, 40))
    A, b, c = F.tie_heavy(m, n, 100 + seed)
    A[:, A.sum(axis=0) == 0] = 1.0
    assert_same(gpu_solve(sx, A, b, c, pivot_rule=sx.BLAND, **path), bland(A, b, c))


@pytest.mark.parametrize("path", PATHS, ids=PATH_IDS)
def test_klee_minty_and_dense(sx, path):
    A, b, c = F.klee_minty(8)
    assert_same(gpu_solve(sx, A, b, c, pivot_rule=sx.BLAND, **path), bland(A, b, c))
    A, b, c = lpgen.dense_lp(150, 220, 5)
    assert_same(gpu_solve(sx, A, b, c, pivot_rule=sx.BLAND, **path), bland(A, b, c))


def test_dense_1000_bland(sx):
    A, b, c = lpgen.dense_lp(1000, 1000, 1)
    o = oracle.solve(A, b, c, rule=oracle.BLAND, keep_tableau=True)
    for look in (1, 16):
        with sx.Simplex(A, b, c, pivot_rule=sx.BLAND, lookahead=look) as s:
            st = s.solve()
            x, y, obj, piv, _ = s.solution()
            k, r = s.trace()
            h = s.tableau_hash()
        assert st == o.status and piv == o.pivots and obj == o.objective
        assert np.array_equal(k, o.trace_k) and np.array_equal(r, o.trace_r)
        assert np.array_equal(x, o.x) and h == oracle.tableau_hash(o.T)


def test_rule_validation(sx):
    A, b, c = F.classic()
    with pytest.raises(sx.SimplexError) as e:
        sx.Simplex(A, b, c, pivot_rule=7)
    assert e.value.code == sx.E_ARG


@pytest.mark.parametrize("overlap", [True, False], ids=["pipe", "serial"])
def test_golden_4000_bland(sx, overlap):
    """Bland's rule on the 4000x4000 benchmark LP runs into the 20(m+n) = 160000 cap: the whole
    trace, the objective, x, y and the tableau digest against the oracle's 2-hour single-thread
    run (tests/golden/dense_4000x4000_s1_bland.*, scripts/make_golden.py)."""
    g = np.load(os.path.join(GOLDEN_DIR, "dense_4000x4000_s1_bland.npz"))
    A, b, c = lpgen.dense_lp(4000, 4000, 1)
    with sx.Simplex(A, b, c, pivot_rule=sx.BLAND, overlap=overlap) as s:
        st = s.solve()
        x, y, obj, piv, _ = s.solution()
        k, r = s.trace()
        h = s.tableau_hash()
    assert st == int(g["status"]) == sx.ITERATION_LIMIT and piv == int(g["pivots"]) == 160000
    assert np.array_equal(k, g["trace_k"]) and np.array_equal(r, g["trace_r"])
    assert obj == float(g["objective"]) and np.array_equal(y, g["y"])
    xs = np.zeros(4000)
    xs[g["x_idx"]] = g["x_val"]
    assert np.array_equal(x, xs)
    assert h == int(g["tableau_hash"])
