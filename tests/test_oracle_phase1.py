"""Pins of the oracle's two-phase method against
things other than itself: SPEC worked examples, the one-phase oracle (b >= 0 reproduces it
bit for bit), brute-force vertex enumeration (which handles any sign of b and detects
infeasibility as "no feasible vertex"), and the optimality certificate on the raw data."""
import numpy as np
import pytest

import oracle
from lpgen import fixtures as F

import lpgen


def arr(x):
    return np.asarray(x, dtype=np.float64)


def test_b_nonnegative_is_one_phase_bitwise():
    # all b >= 0 -> zero Phase-I iterations; then Phase II = the one-phase method
    for A, b, c in [F.classic(), F.chvatal(), lpgen.dense_lp(40, 50, 3), F.klee_minty(5)]:
        two = oracle.solve_2phase(A, b, c)
        one = oracle.solve(A, b, c)
        assert two.phase1_pivots == 0
        assert two.status == one.status and two.trace() == one.trace()
        assert two.objective == one.objective
        assert np.array_equal(two.x, one.x) and np.array_equal(two.y, one.y)


def test_spec_examples():
    # x >= 2 (as -x <= -2) with x <= 4 -> feasible; max x -> 4
    r = oracle.solve_2phase(arr([[-1.0], [1.0]]), arr([-2.0, 4.0]), arr([1.0]))
    assert r.status == oracle.OPTIMAL and r.objective == 4.0 and r.x.tolist() == [4.0]
    # x <= 1 and -x <= -3 -> infeasible
    r = oracle.solve_2phase(arr([[1.0], [-1.0]]), arr([1.0, -3.0]), arr([1.0]))
    assert r.status == oracle.INFEASIBLE
    # x >= 1, maximize x -> unbounded in Phase II
    r = oracle.solve_2phase(arr([[-1.0]]), arr([-1.0]), arr([1.0]))
    assert r.status == oracle.UNBOUNDED


def _mixed_cases(seed, count, tie_heavy=False):
    rng = np.random.default_rng(seed)
    out = []
    for _ in range(count):
        m = int(rng.integers(1, 6))
        n = int(rng.integers(1, 12 - m))
        if tie_heavy:
            A = rng.integers(-2, 4, size=(m, n)).astype(float)
            b = rng.integers(-4, 6, size=m).astype(float)
        else:
            A = rng.uniform(-3, 10, size=(m, n))
            b = rng.uniform(-n, 2 * n, size=m)
        A = np.vstack([A, np.ones((1, n))])            # sum(x) <= 3n keeps every LP bounded
        b = np.concatenate([b, [3.0 * n]])
        c = rng.uniform(-2, 10, size=n)
        out.append((A, b, c))
    return out


@pytest.mark.parametrize("rule", [oracle.DANTZIG, oracle.BLAND])
@pytest.mark.parametrize("tie", [False, True])
def test_brute_force_mixed_signs(rule, tie):
    seen = {oracle.OPTIMAL: 0, oracle.INFEASIBLE: 0}
    for A, b, c in _mixed_cases(31 + tie, 80, tie):
        r = oracle.solve_2phase(A, b, c, rule=rule)
        found, bf, _ = oracle.brute_force(A, b, c)
        if not found:
            assert r.status == oracle.INFEASIBLE, (A, b, c)
            seen[oracle.INFEASIBLE] += 1
            continue
        assert r.status == oracle.OPTIMAL, (A, b, c, r.status)
        assert abs(r.objective - bf) <= 1e-9 * max(1.0, abs(bf))
        cert = oracle.certificate(A, b, c, r.x, r.y)
        assert not cert.violations, cert.violations
        seen[oracle.OPTIMAL] += 1
    assert seen[oracle.OPTIMAL] > 10 and seen[oracle.INFEASIBLE] > 3


def test_planted_with_negative_rhs():
    # planted optimum, then rows with slack s_i > 0 shifted by a constant times a feasible
    # direction are NOT needed: flip the sign convention instead — add constraints
    # -sum_j x_j <= -t (t below the optimum's sum) which are inactive at x*: same optimum
    A, b, c, xs, ys = F.planted(30, 40, 7, 10)
    t = 0.5 * xs.sum()
    A2 = np.vstack([A, -np.ones((1, 40))])
    b2 = np.concatenate([b, [-t]])
    r = oracle.solve_2phase(A2, b2, c)
    assert r.status == oracle.OPTIMAL and r.phase1_pivots > 0
    obj = float(c @ xs)
    assert abs(r.objective - obj) <= 1e-9 * abs(obj)
    assert np.max(np.abs(r.x - xs)) <= 1e-7
    assert not oracle.certificate(A2, b2, c, r.x, r.y).violations


def drive_out_pivots(A, b, res):
    """Drive-out pivots in a two-phase trace (reading p4): replay the basis through the Phase I
    pivots; the pivots right after them on rows whose basic variable is still artificial."""
    m, n = A.shape
    basis, art = [], 0
    for i in range(m):
        if b[i] < 0:
            basis.append(n + m + art)
            art += 1
        else:
            basis.append(n + i)
    for k, r in zip(res.trace_k[:res.phase1_pivots], res.trace_r[:res.phase1_pivots]):
        basis[r - 1] = int(k)
    left = sorted(i + 1 for i in range(m) if basis[i] >= n + m)
    d = 0
    for r in res.trace_r[res.phase1_pivots:]:
        if d < len(left) and r == left[d]:
            d += 1
        else:
            break
    return d, len(left)


def test_lower_bound_fixture_needs_drive_out():
    """lpgen.fixtures.with_lower_bounds with equality pairs: Phase I ends with artificials basic
    at zero, the drive-out pivots them out, and the final answer is certified optimal from the
    raw data (primal / dual feasibility, strong duality)."""
    from lpgen import fixtures
    A, b, c = fixtures.with_lower_bounds(120, 150, 3, frac=0.1, eq=6)
    r = oracle.solve_2phase(A, b, c)
    assert r.status == oracle.OPTIMAL and r.phase1_pivots > 0
    d, left = drive_out_pivots(A, b, r)
    assert left >= 1 and d >= 1
    assert not oracle.certificate(A, b, c, r.x, r.y).violations
