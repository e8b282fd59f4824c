"""The hybrid CPU lane (options.host_share = θ; SURVEY.md §8(f) NEXT #4 — the paper's own
contribution, §IV: columns split between the CPU cores and the GPU,
per-iteration exchange of candidates, each side pivoting its own columns).  Bar: bit-identical to
the oracle for every θ (trace, objective, x, y, the whole tableau — GPU and host columns — and the
digest): the host lane uses the same c8 arithmetic (IEEE division, one fma per element)."""
import json
import os

import numpy as np
import pytest

import lpgen
import oracle
from lpgen import fixtures as F

pytestmark = pytest.mark.gpu
GOLDEN_DIR = os.path.join(os.path.dirname(__file__), "golden")


@pytest.fixture(scope="module")
def sx(cuda_device):
    import paper_2211_10979_b200 as sx
    return sx


def hybrid_solve(sx, A, b, c, theta, **kw):
    with sx.Simplex(A, b, c, host_share=theta, **kw) as s:
        st0 = s.stats()
        assert st0.path == 2 and st0.host_cols >= 1
        st = s.solve()
        x, y, obj, piv, _ = s.solution()
        k, r = s.trace()
        T, _ = s.tableau()
        h = s.tableau_hash()
    return dict(status=st, x=x, y=y, obj=obj, pivots=piv, k=k, r=r, T=T, hash=h, host_cols=st0.host_cols)


def assert_same(g, o):
    assert g["status"] == o.status and g["pivots"] == o.pivots
    assert np.array_equal(g["k"], o.trace_k) and np.array_equal(g["r"], o.trace_r)
    assert g["obj"] == o.objective
    assert np.array_equal(g["x"], o.x) and np.array_equal(g["y"], o.y)
    assert np.array_equal(g["T"], o.T)
    assert g["hash"] == oracle.tableau_hash(o.T)


@pytest.mark.parametrize("theta", [1e-9, 0.01, 0.05, 0.3, 0.7, 0.999])
def test_dense_theta_sweep(sx, theta):
    A, b, c = lpgen.dense_lp(200, 300, 12)
    assert_same(hybrid_solve(sx, A, b, c, theta), oracle.solve(A, b, c, keep_tableau=True))


@pytest.mark.parametrize("theta", [0.1, 0.5])
@pytest.mark.parametrize("seed", range(4))
def test_tie_heavy_both_rules(sx, theta, seed):
    A, b, c = F.tie_heavy(25 + seed, 33, 900 + seed)
    assert_same(hybrid_solve(sx, A, b, c, theta), oracle.solve(A, b, c, keep_tableau=True))
    assert_same(hybrid_solve(sx, A, b, c, theta, pivot_rule=sx.BLAND),
                oracle.solve(A, b, c, keep_tableau=True, rule=oracle.BLAND))


@pytest.mark.parametrize("name", ["classic", "chvatal", "unbounded", "beale", "klee_minty"])
def test_worked_examples(sx, name):
    A, b, c = {"classic": F.classic, "chvatal": F.chvatal, "unbounded": F.unbounded_1d, "beale": F.beale,
               "klee_minty": lambda: F.klee_minty(8)}[name]()
    kw = {"max_pivots": 30} if name == "beale" else {"max_pivots": 1000} if name == "klee_minty" else {}
    for theta in (0.2, 0.6):
        assert_same(hybrid_solve(sx, A, b, c, theta, **kw), oracle.solve(A, b, c, keep_tableau=True, **kw))


def test_iterate_windows(sx):
    A, b, c = lpgen.dense_lp(150, 220, 5)
    o = oracle.solve(A, b, c, keep_tableau=True)
    with sx.Simplex(A, b, c, host_share=0.25) as s:
        total = 0
        while True:
            done, st = s.iterate(7)
            assert done <= 7
            total += done
            T, _ = s.tableau()
            assert np.array_equal(T, oracle.solve(A, b, c, keep_tableau=True, stop_after=total).T)
            if st != sx.RUNNING:
                break
        assert total == o.pivots and st == o.status
        s.reset(A, b, c)                          # the host lane is rebuilt too
        assert s.solve() == o.status and s.solution()[2] == o.objective


def test_golden_1000(sx):
    g = np.load(os.path.join(GOLDEN_DIR, "dense_1000x1000_s1.npz"))
    A, b, c = lpgen.dense_lp(1000, 1000, 1)
    with sx.Simplex(A, b, c, host_share=0.02) as s:
        st = s.solve()
        x, y, obj, piv, _ = s.solution()
        k, r = s.trace()
        h = s.tableau_hash()
    assert st == int(g["status"]) and piv == int(g["pivots"])
    assert np.array_equal(k, g["trace_k"]) and np.array_equal(r, g["trace_r"])
    assert obj == float(g["objective"]) and np.array_equal(y, g["y"])
    assert h == int(g["tableau_hash"])


def test_options_rejected(sx):
    A, b, c = lpgen.dense_lp(20, 30, 1)
    for kw in (dict(host_share=1.0), dict(host_share=0.1, lookahead=16), dict(host_share=0.1, virtual_ranks=2),
               dict(host_share=0.1, exchange=1)):
        with pytest.raises(sx.SimplexError) as e:
            sx.Simplex(A, b, c, **kw)
        assert e.value.code == sx.E_ARG, kw
    b2 = b.copy()
    b2[0] = -1.0
    with pytest.raises(sx.SimplexError) as e:
        sx.Simplex(A, b2, c, host_share=0.1)
    assert e.value.code == sx.E_ARG
