"""Pins of the CPU oracle against things other than itself (-m "not gpu").

Each test names what fixes the expected value: a worked example (SPEC.md /
textbook, tests/golden/worked_examples.json), a closed form (Klee–Minty,
diagonal, planted optimum), exact rational arithmetic (reading c8), brute-force
vertex enumeration, or an invariant of the method.
"""
import json
import os
from fractions import Fraction

import numpy as np
import pytest

import oracle
from lpgen import fixtures as F

GOLD = json.load(open(os.path.join(os.path.dirname(__file__), "golden", "worked_examples.json")))


def arr(x):
    return np.asarray(x, dtype=np.float64)


# ---------------------------------------------------------------- a0 build
def test_build_spec_m1():
    g = GOLD["build_m1"]
    T, basis = oracle.build_tableau(arr(g["A"]), arr(g["b"]), arr(g["c"]))
    assert T.shape == (2, 3)
    assert T[0].tolist() == g["row0"] and T[1].tolist() == g["row1"]
    assert basis.tolist() == g["basis"]


def test_build_classic_unit_slacks():
    A, b, c = F.classic()
    T, basis = oracle.build_tableau(A, b, c)
    m, n = A.shape
    assert T.shape == (m + 1, n + m + 1)
    for i in range(1, m + 1):           # SPEC.md:68 unit-column invariant, bitwise
        e = np.zeros(m + 1)
        e[i] = 1.0
        assert np.array_equal(T[:, basis[i - 1]], e)
    assert np.array_equal(T[0, :n], -c) and np.array_equal(T[1:, -1], b)
    assert np.array_equal(T[1:, :n], A)


def test_build_rejects():
    with pytest.raises(oracle.OracleError) as e:
        oracle.build_tableau(arr([[1.0]]), arr([-1.0]), arr([1.0]))
    assert e.value.code == oracle.E_NEG_RHS                       # SPEC.md:67, reading c11
    with pytest.raises(oracle.OracleError) as e:
        oracle.build_tableau(arr([[np.nan]]), arr([1.0]), arr([1.0]))
    assert e.value.code == oracle.E_NONFINITE


# ---------------------------------------------------------------- a1 pricing
@pytest.mark.parametrize("ex", GOLD["price"], ids=lambda e: e["cite"])
def test_price_spec(ex):
    k, v = oracle.price(arr(ex["row"]))
    assert k == ex["k"]
    if k >= 0:
        assert v == ex["v"]


@pytest.mark.parametrize("ex", GOLD["merge"], ids=lambda e: e["cite"])
def test_merge_spec(ex):
    # lexicographic (value, column) fold of per-lane candidates
    best = (np.inf, -1)
    for k, v in ex["cands"]:
        if (v, k) < best:
            best = (v, k)
    assert best[1] == ex["k"]


def test_price_any_partition_equals_scan():
    # SPEC.md:272 reduction equivalence: argmin over any partition = sequential scan
    rng = np.random.default_rng(7)
    for _ in range(200):
        row = rng.integers(-5, 3, size=rng.integers(1, 60)).astype(np.float64)
        k, v = oracle.price(row)
        cuts = sorted(rng.choice(np.arange(1, row.size), size=min(3, row.size - 1), replace=False)) \
            if row.size > 1 else []
        bounds = [0, *cuts, row.size]
        best = (np.inf, -1)
        for a, b_ in zip(bounds[:-1], bounds[1:]):
            kk, vv = oracle.price(row[a:b_])
            if kk >= 0 and (vv, kk + a) < best:
                best = (vv, kk + a)
        assert best[1] == k


# ---------------------------------------------------------------- a2 ratio test
def _tab_from_col(col, rhs):
    m = len(col)
    T = np.zeros((m + 1, 2))
    T[1:, 0] = col
    T[1:, 1] = rhs
    return T


@pytest.mark.parametrize("ex", GOLD["ratio"], ids=lambda e: e["cite"])
def test_ratio_spec(ex):
    T = _tab_from_col(ex["col"], ex["rhs"])
    r, q = oracle.ratio(T, 0)
    assert r == ex["r"]
    if r > 0:
        assert q == ex["q"]
        if "pivot" in ex:
            assert T[r, 0] == ex["pivot"]


def test_ratio_tolerance_excludes_tiny_positive():
    # reading c5/c6: T[i][k] <= 1e-10 is not eligible, even if positive
    T = _tab_from_col([1e-11, 0.0], [1.0, 1.0])
    assert oracle.ratio(T, 0)[0] == -1
    T = _tab_from_col([1e-11, 2e-10], [1e-20, 1.0])
    assert oracle.ratio(T, 0)[0] == 2


def test_ratio_division_is_ieee():
    # q must be the correctly rounded quotient (reading c8), checked in exact rationals
    rng = np.random.default_rng(3)
    for _ in range(300):
        col = rng.uniform(0.1, 10, size=4)
        rhs = rng.uniform(0, 100, size=4)
        r, q = oracle.ratio(_tab_from_col(col, rhs), 0)
        exact = [float(Fraction(rhs[i]) / Fraction(col[i])) for i in range(4)]
        assert q == min(exact)
        assert r == 1 + exact.index(min(exact))


# ---------------------------------------------------------------- a4 pivot
def test_pivot_spec():
    ex = GOLD["pivot"][0]
    T = arr(ex["T"]).copy()
    oracle.pivot(T, ex["r"], ex["k"])
    assert T.tolist() == ex["after"]


def test_pivot_identity_case():
    # pivot column already e_r: unchanged except row r divided by 1
    T = arr([[0.0, 3.0, 5.0], [1.0, 2.0, 7.0], [0.0, 4.0, 1.0]])
    before = T.copy()
    oracle.pivot(T, 1, 0)
    assert np.array_equal(T, before)


def test_pivot_arithmetic_is_div_then_fma_exact():
    # Reading c8, checked element by element against exact rational arithmetic:
    # prow_j = RN(T[r][j] / p);  T[i][j] = RN(T[i][j] - T[i][k] * prow_j)  (one rounding: fma)
    rng = np.random.default_rng(11)
    for trial in range(20):
        m1, W = 5, 7
        T = rng.uniform(-10, 10, size=(m1, W))
        r, k = 1 + trial % (m1 - 1), trial % (W - 1)
        T0 = T.copy()
        oracle.pivot(T, r, k)
        p = Fraction(T0[r, k])
        prow = [float(Fraction(T0[r, j]) / p) for j in range(W)]
        for i in range(m1):
            for j in range(W):
                if i == r:
                    want = prow[j]
                else:
                    want = float(Fraction(T0[i, j]) - Fraction(T0[i, k]) * Fraction(prow[j]))
                assert T[i, j] == want, (trial, i, j)
        assert T[r, k] == 1.0 and all(T[i, k] == 0.0 for i in range(m1) if i != r)


def test_classic_first_pivot_objective_30():
    # entering x2 (col 1), leaving row 2 (2x2 <= 12) -> objective 0 -> 30
    A, b, c = F.classic()
    T, _ = oracle.build_tableau(A, b, c)
    k, _ = oracle.price(T[0, :-1])
    r, _ = oracle.ratio(T, k)
    assert (k, r) == (1, 2)
    oracle.pivot(T, r, k)
    assert T[0, -1] == 30.0


# ---------------------------------------------------------------- whole loop, worked examples
@pytest.mark.parametrize("name", ["classic", "chvatal", "entering_tie", "ratio_tie"])
def test_worked_solves(name):
    g = GOLD[name]
    A, b, c = (F.classic() if name == "classic" else (arr(g["A"]), arr(g["b"]), arr(g["c"])))
    res = oracle.solve(A, b, c, keep_tableau=True)
    assert res.status == oracle.OPTIMAL
    assert [list(t) for t in res.trace()] == g["trace"]
    assert res.objective == g["objective"]
    assert res.x.tolist() == g["x"]
    if "y" in g:
        assert res.y.tolist() == g["y"]
    if "rhs_after" in g:
        assert res.T[1:, -1].tolist() == g["rhs_after"]
    found, bf, _ = oracle.brute_force(A, b, c)
    assert found and abs(bf - res.objective) <= 1e-9 * max(1, abs(bf))


def test_zero_iteration_and_unbounded():
    g = GOLD["zero_iteration"]
    res = oracle.solve(arr(g["A"]), arr(g["b"]), arr(g["c"]))
    assert res.status == oracle.OPTIMAL and res.pivots == 0 and res.objective == 0.0
    assert not res.x.any()
    res = oracle.solve(*F.unbounded_1d())
    assert res.status == oracle.UNBOUNDED and res.pivots == 0


def test_beale_cycles_to_iteration_limit():
    g = GOLD["beale"]
    A, b, c = F.beale()
    res = oracle.solve(A, b, c)
    cap = 20 * (3 + 4)
    assert res.status == oracle.ITERATION_LIMIT and res.pivots == cap
    tr = [list(t) for t in res.trace()]
    assert tr[:6] == g["cycle"]
    assert all(tr[i] == tr[i % 6] for i in range(cap))
    found, bf, x = oracle.brute_force(A, b, c)
    assert found and abs(bf - g["optimum"]) < 1e-12


def test_iteration_cap_precedence():
    # reading c12: a problem needing exactly `cap` pivots returns OPTIMAL, cap-1 -> ITERATION_LIMIT
    A, b, c = F.klee_minty(4)          # 15 pivots
    assert oracle.solve(A, b, c, max_pivots=15).status == oracle.OPTIMAL
    res = oracle.solve(A, b, c, max_pivots=14)
    assert res.status == oracle.ITERATION_LIMIT and res.pivots == 14


def test_stop_after_prefix_matches_full():
    A, b, c = F.klee_minty(6)
    full = oracle.solve(A, b, c, keep_tableau=True, max_pivots=100)
    pre = oracle.solve(A, b, c, stop_after=10, keep_tableau=True, max_pivots=100)
    assert pre.status == oracle.RUNNING and pre.pivots == 10
    assert pre.trace() == full.trace()[:10]


# ---------------------------------------------------------------- closed forms
@pytest.mark.parametrize("n", range(2, 13))
def test_klee_minty(n):
    # Klee & Minty (1972): Dantzig's rule visits all 2^n vertices -> 2^n - 1 pivots,
    # optimum 5^n at x = (0, ..., 0, 5^n); the tableau stays in exact integers.
    A, b, c = F.klee_minty(n)
    res = oracle.solve(A, b, c, max_pivots=2 ** n + 5, keep_tableau=True)
    assert res.status == oracle.OPTIMAL
    assert res.pivots == 2 ** n - 1
    assert res.objective == 5.0 ** n
    want = np.zeros(n)
    want[-1] = 5.0 ** n
    assert np.array_equal(res.x, want)
    assert np.array_equal(res.T, np.round(res.T))


@pytest.mark.parametrize("m,seed", [(5, 0), (40, 1), (300, 2)])
def test_diagonal(m, seed):
    # A = diag(d): pivots never interact, so Dantzig enters columns in order of
    # (-c_j, j), each leaving its own row j+1; obj = sum c_i b_i / d_i.
    A, b, c = F.diagonal(m, seed)
    res = oracle.solve(A, b, c)
    order = sorted(range(m), key=lambda j: (-c[j], j))
    assert res.trace() == [(j, j + 1) for j in order]
    d = np.diag(A)
    assert res.objective == pytest.approx(float(sum(Fraction(c[i]) * Fraction(b[i]) / Fraction(d[i])
                                                    for i in range(m))), rel=1e-14)
    assert np.array_equal(res.x, b / d)


@pytest.mark.parametrize("m,n,s,seed", [(20, 30, 6, 1), (60, 80, 20, 2), (150, 200, 40, 3)])
def test_planted_optimum(m, n, s, seed):
    A, b, c, xs, ys = F.planted(m, n, seed, s)
    res = oracle.solve(A, b, c)
    assert res.status == oracle.OPTIMAL
    obj = float(c @ xs)
    assert abs(res.objective - obj) <= 1e-9 * max(1, abs(obj))
    assert np.max(np.abs(res.x - xs)) <= 1e-7
    assert np.max(np.abs(res.y - ys)) <= 1e-7


# ---------------------------------------------------------------- brute force on tiny LPs
def _tiny_cases():
    rng = np.random.default_rng(2024)
    cases = []
    for t in range(60):
        m = int(rng.integers(1, 7))
        n = int(rng.integers(1, 13 - m))
        if t % 2:
            A, b, c = F.tie_heavy(m, n, int(rng.integers(1 << 30)))
            A[A.sum(axis=1) == 0, 0] = 1.0      # keep every tiny LP bounded below-rows
            A[:, A.sum(axis=0) == 0] = 1.0
        else:
            A = rng.uniform(1, 10, size=(m, n))
            b = rng.uniform(n, 2 * n, size=m)
            c = rng.uniform(1, 10, size=n)
        cases.append((A, b, c))
    return cases


def test_brute_force_tiny():
    for A, b, c in _tiny_cases():
        res = oracle.solve(A, b, c)
        assert res.status == oracle.OPTIMAL
        found, bf, _ = oracle.brute_force(A, b, c)
        assert found
        assert abs(res.objective - bf) <= 1e-9 * max(1.0, abs(bf))
        cert = oracle.certificate(A, b, c, res.x, res.y)
        assert not cert.violations, cert.violations


# ---------------------------------------------------------------- invariants every pivot
@pytest.mark.parametrize("kind", ["dense", "ties"])
def test_invariants_every_pivot(kind):
    rng = np.random.default_rng(5 if kind == "dense" else 6)
    for _ in range(10):
        m, n = int(rng.integers(3, 25)), int(rng.integers(3, 25))
        if kind == "dense":
            A, b, c = rng.uniform(1, 10, (m, n)), rng.uniform(n, 2 * n, m), rng.uniform(1, 10, n)
        else:
            A, b, c = F.tie_heavy(m, n, int(rng.integers(1 << 30)))
            A[:, A.sum(axis=0) == 0] = 1.0
        T, basis = oracle.build_tableau(A, b, c)
        prev = T[0, -1]
        for _it in range(20 * (m + n)):
            k, _ = oracle.price(T[0, :-1])
            if k < 0:
                break
            r, q = oracle.ratio(T, k)
            assert r > 0
            oracle.pivot(T, r, k)
            basis[r - 1] = k
            for i in range(1, m + 1):        # basic columns bitwise unit
                e = np.zeros(m + 1)
                e[i] = 1.0
                assert np.array_equal(T[:, basis[i - 1]], e)
            assert T[0, -1] >= prev          # monotone objective
            if q > 0:
                assert T[0, -1] > prev
            prev = T[0, -1]
            assert T[1:, -1].min() >= -1e-9  # feasibility preserved


# ---------------------------------------------------------------- certificate sanity
def test_certificate_flags_counterexamples():
    A, b, c = F.classic()
    res = oracle.solve(A, b, c)
    assert not oracle.certificate(A, b, c, res.x, res.y).violations
    # SPEC.md:97-98 constructed counterexamples
    bad_y = res.y.copy()
    bad_y[2] -= 0.5
    assert oracle.certificate(A, b, c, res.x, bad_y).violations
    bad_x = res.x.copy()
    bad_x[0] += 1.0
    assert oracle.certificate(A, b, c, bad_x, res.y).violations


# ---------------------------------------------------------------- Bland's rule (NEXT #3)
def test_bland_steps_by_definition():
    # entering: FIRST index with T[0][j] < -tol, not the most negative
    assert oracle.price_bland(arr([0.0, -1.0, -5.0])) == 1
    assert oracle.price_bland(arr([0.0, 0.5, 1e-9])) == -1
    # leaving: exact ratio tie (3 = 3/1 = 6/2) -> smallest BASIC-VARIABLE index, not lowest row
    T = _tab_from_col([1.0, 2.0], [3.0, 6.0])
    assert oracle.ratio_bland(T, 0, basis=[7, 4])[0] == 2
    assert oracle.ratio_bland(T, 0, basis=[4, 7])[0] == 1
    assert oracle.ratio_bland(_tab_from_col([-1.0, 0.0], [1.0, 1.0]), 0, basis=[1, 2])[0] == -1


def test_bland_terminates_on_beale():
    # the cycling instance terminates OPTIMAL under Bland, at the true
    # optimum 1/20 (brute force), where Dantzig + lowest-row ties cycles to the cap
    A, b, c = F.beale()
    res = oracle.solve(A, b, c, rule=oracle.BLAND)
    assert res.status == oracle.OPTIMAL
    found, bf, xb = oracle.brute_force(A, b, c)
    assert abs(res.objective - bf) <= 1e-12 and abs(bf - 0.05) < 1e-12
    assert np.allclose(res.x, [0.04, 0.0, 1.0, 0.0], atol=1e-12)
    assert oracle.solve(A, b, c).status == oracle.ITERATION_LIMIT


def test_bland_brute_force_and_certificates():
    # degenerate, tie-heavy tiny LPs: Bland always terminates at the brute-force optimum
    for A, b, c in _tiny_cases():
        res = oracle.solve(A, b, c, rule=oracle.BLAND)
        assert res.status == oracle.OPTIMAL
        found, bf, _ = oracle.brute_force(A, b, c)
        assert abs(res.objective - bf) <= 1e-9 * max(1.0, abs(bf))
        assert not oracle.certificate(A, b, c, res.x, res.y).violations


def test_bland_invariants_every_pivot():
    rng = np.random.default_rng(8)
    for _ in range(10):
        m, n = int(rng.integers(3, 25)), int(rng.integers(3, 25))
        A, b, c = F.tie_heavy(m, n, int(rng.integers(1 << 30)))
        A[:, A.sum(axis=0) == 0] = 1.0
        T, basis = oracle.build_tableau(A, b, c)
        prev = T[0, -1]
        for _it in range(20 * (m + n)):
            k = oracle.price_bland(T[0, :-1])
            if k < 0:
                break
            r, q = oracle.ratio_bland(T, k, basis)
            assert r > 0
            oracle.pivot(T, r, k)
            basis[r - 1] = k
            for i in range(1, m + 1):
                e = np.zeros(m + 1)
                e[i] = 1.0
                assert np.array_equal(T[:, basis[i - 1]], e)
            assert T[0, -1] >= prev
            prev = T[0, -1]
        else:
            raise AssertionError("Bland's rule did not terminate")
        # the stepwise run and or_solve_rule agree
        res = oracle.solve(A, b, c, rule=oracle.BLAND, keep_tableau=True)
        assert np.array_equal(res.T, T)
