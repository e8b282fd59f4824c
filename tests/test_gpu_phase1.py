"""GPU parity of the two-phase method (b with negative entries)
against the oracle's or_solve_2phase: identical status, pivot trace (Phase I, drive-out and
Phase II pivots), objective, x and y — bit for bit — on every single-part path."""
import numpy as np
import pytest

import lpgen
import oracle

pytestmark = pytest.mark.gpu

PATHS = [dict(lookahead=1), dict(lookahead=4), dict(lookahead=16), dict(lookahead=16, overlap=False),
         dict(lookahead=32), dict(lookahead=1, virtual_ranks=3), dict(lookahead=16, virtual_ranks=2),
         dict(lookahead=8, virtual_ranks=3, exchange=2)]
PATH_IDS = ["pass1", "look4", "look16", "look16serial", "pair32", "slabs3", "mpart2", "mpart3peer"]


@pytest.fixture(scope="module")
def sx(cuda_device):
    import paper_2211_10979_b200 as sx
    return sx


def gpu(sx, A, b, c, **kw):
    if "virtual_ranks" in kw:                      # at most one part per column (n + m of them)
        kw["virtual_ranks"] = min(kw["virtual_ranks"], A.shape[0] + A.shape[1])
    with sx.Simplex(A, b, c, **kw) as s:
        st = s.solve()
        x, y, obj, piv, _ = s.solution()
        k, r = s.trace()
    return st, x, y, obj, piv, k, r


def check(sx, A, b, c, rule=0, **kw):
    o = oracle.solve_2phase(A, b, c, rule=rule)
    st, x, y, obj, piv, k, r = gpu(sx, A, b, c, pivot_rule=rule, **kw)
    assert st == o.status, (st, o.status)
    assert piv == o.pivots
    assert np.array_equal(k, o.trace_k) and np.array_equal(r, o.trace_r)
    if o.status == oracle.OPTIMAL:
        assert obj == o.objective
        assert np.array_equal(x, o.x) and np.array_equal(y, o.y)
    return o


@pytest.mark.parametrize("path", PATHS, ids=PATH_IDS)
def test_spec_examples(sx, path):
    a = lambda v: np.asarray(v, dtype=float)  # noqa: E731
    o = check(sx, a([[-1.0], [1.0]]), a([-2.0, 4.0]), a([1.0]), **path)
    assert o.status == oracle.OPTIMAL and o.objective == 4.0
    o = check(sx, a([[1.0], [-1.0]]), a([1.0, -3.0]), a([1.0]), **path)
    assert o.status == oracle.INFEASIBLE
    o = check(sx, a([[-1.0]]), a([-1.0]), a([1.0]), **path)
    assert o.status == oracle.UNBOUNDED


def _mixed(seed, count, tie):
    rng = np.random.default_rng(seed)
    out = []
    for _ in range(count):
        m = int(rng.integers(1, 24))
        n = int(rng.integers(1, 30))
        if tie:
            A = rng.integers(-2, 4, size=(m, n)).astype(float)
            b = rng.integers(-1, 8, size=m).astype(float)
        else:
            A = rng.uniform(-3, 10, size=(m, n))
            b = rng.uniform(-n, 2 * n, size=m)
        A = np.vstack([A, np.ones((1, n))])
        b = np.concatenate([b, [3.0 * n]])
        out.append((A, b, rng.uniform(-2, 10, size=n)))
    return out


@pytest.mark.parametrize("path", PATHS, ids=PATH_IDS)
@pytest.mark.parametrize("rule", [0, 1], ids=["dantzig", "bland"])
@pytest.mark.parametrize("tie", [False, True], ids=["uniform", "ties"])
def test_mixed_sign_lps(sx, path, rule, tie):
    statuses = set()
    for A, b, c in _mixed(7 + tie, 16, tie):
        statuses.add(check(sx, A, b, c, rule=rule, **path).status)
    assert statuses <= {oracle.OPTIMAL, oracle.INFEASIBLE}
    assert len(statuses) == 2                       # both outcomes exercised


@pytest.mark.parametrize("path", PATHS, ids=PATH_IDS)
def test_dense_with_lower_bounds(sx, path):
    # dense generator LP plus 25 "at least" rows -a_i x <= -t_i (feasible, active-ish)
    A, b, c = lpgen.dense_lp(300, 400, 11)
    rng = np.random.default_rng(0)
    L = rng.uniform(1, 10, size=(25, 400))
    A2 = np.vstack([A, -L])
    b2 = np.concatenate([b, -rng.uniform(5, 50, size=25)])
    o = check(sx, A2, b2, c, **path)
    assert o.status == oracle.OPTIMAL and o.phase1_pivots > 0
    assert not oracle.certificate(A2, b2, c, *gpu(sx, A2, b2, c, **path)[1:3]).violations


def test_options_and_errors(sx):
    A = np.array([[1.0, 1.0], [-1.0, 0.0]])
    b = np.array([4.0, -1.0])
    c = np.array([1.0, 2.0])
    with pytest.raises(sx.SimplexError) as e:
        sx.Simplex(A, b, c, phase1=False)
    assert e.value.code == sx.E_NEG_RHS
    with sx.Simplex(A, b, c, virtual_ranks=2, lookahead=1) as s:   # Phase I on several parts
        assert s.solve() == sx.OPTIMAL
    with sx.Simplex(A, b, c) as s:                 # reset with a different sign pattern count
        with pytest.raises(sx.SimplexError) as e:
            s.reset(A, np.array([4.0, 1.0]), c)
        assert e.value.code == sx.E_ARG


DRIVE_PATHS = [dict(lookahead=1), dict(lookahead=16), dict(lookahead=16, overlap=False),
               dict(lookahead=1, virtual_ranks=3), dict(lookahead=16, virtual_ranks=2),
               dict(lookahead=16, virtual_ranks=3, exchange=2)]
DRIVE_IDS = ["pass1", "look16", "look16serial", "slabs3", "mpart2", "mpart3peer"]


@pytest.mark.parametrize("path", DRIVE_PATHS, ids=DRIVE_IDS)
def test_drive_out_on_device(sx, path):
    """Equality pairs leave artificials basic at zero after Phase I; the device drive-out
    (k_drive_find / pick / col / force + the update, no host round trip per pivot) pivots them
    out on the first eligible column over all parts — trace bit-identical to or_solve_2phase."""
    from lpgen import fixtures
    A, b, c = fixtures.with_lower_bounds(120, 150, 3, frac=0.1, eq=6)
    o = check(sx, A, b, c, **path)
    assert o.status == oracle.OPTIMAL


@pytest.mark.parametrize("path", [dict(lookahead=1), dict(lookahead=16), dict(lookahead=16, virtual_ranks=2)],
                         ids=["pass1", "look16", "mpart2"])
def test_iterate_across_drive_out(sx, path):
    """simplex_iterate in windows of 1 and 3 pivots never exceeds its window, also when the window
    ends inside the drive-out (which then resumes at the same row): same trace as the oracle."""
    from lpgen import fixtures
    A, b, c = fixtures.with_lower_bounds(120, 150, 3, frac=0.1, eq=6)
    o = oracle.solve_2phase(A, b, c)
    for win in (1, 3):
        with sx.Simplex(A, b, c, **path) as s:
            total, st = 0, sx.RUNNING
            while st == sx.RUNNING:
                done, st = s.iterate(win)
                assert 0 <= done <= win
                total += done
            k, r = s.trace()
            x, y, obj, piv, _ = s.solution()
        assert st == o.status and total == o.pivots == piv
        assert np.array_equal(k, o.trace_k) and np.array_equal(r, o.trace_r)
        assert obj == o.objective and np.array_equal(x, o.x)


@pytest.mark.parametrize("path", [dict(), dict(lookahead=16, virtual_ranks=3)], ids=["default", "slabs3"])
def test_phase1_2000_with_drive_out(sx, path):
    """A 2000x2000 dense LP with 10 % ">=" rows (b_i < 0) and 20 equality pairs (2020 rows): Phase I
    (18089 pivots), 20 device drive-out pivots, Phase II — bit-identical to or_solve_2phase (its
    row-parallel build, bitwise equal to the single-thread one: tests/test_oracle_omp.py), and
    certified optimal from the raw data."""
    from lpgen import fixtures
    A, b, c = fixtures.with_lower_bounds(2000, 2000, 3, frac=0.1, eq=20)
    o = oracle.solve_2phase(A, b, c, parallel=True)
    st, x, y, obj, piv, k, r = gpu(sx, A, b, c, **path)
    assert st == o.status == oracle.OPTIMAL and piv == o.pivots
    assert np.array_equal(k, o.trace_k) and np.array_equal(r, o.trace_r)
    assert obj == o.objective and np.array_equal(x, o.x) and np.array_equal(y, o.y)
    assert not oracle.certificate(A, b, c, x, y).violations
