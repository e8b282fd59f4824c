"""GPU parity: libsimplex (sm_100a kernels through the C ABI) against the CPU oracle.

Bar (BASELINE.json north_star): identical entering/leaving index sequence, objective
within 1e-9 relative, x within 1e-7 absolute.  Under the arithmetic pin (reading c8)
the tableau is expected to be BIT-identical, so these tests assert exact equality of
traces, objective, x, y and the whole-tableau digest, and additionally check the
north_star tolerances and the certificate (strong duality) where relevant.
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
GOLDEN_DIR = os.path.join(os.path.dirname(__file__), "golden")


@pytest.fixture(scope="module")
def sx(cuda_device):
    import paper_2211_10979_b200 as sx
    return sx


def gpu_solve(sx, A, b, c, **kw):
    kw.setdefault("lookahead", 1)           # this file covers the one-pivot-per-pass path
    with sx.Simplex(A, b, c, **kw) as s:
        st = s.solve()
        x, y, obj, piv, st2 = s.solution()
        k, r = s.trace()
        T, _ = s.tableau()
        h = s.tableau_hash()
    assert st == st2
    return dict(status=st, x=x, y=y, obj=obj, pivots=piv, k=k, r=r, T=T, hash=h)


def assert_same(g, o, *, tableau=True):
    assert g["status"] == o.status
    assert g["pivots"] == o.pivots
    assert np.array_equal(g["k"], o.trace_k) and np.array_equal(g["r"], o.trace_r)
    assert g["obj"] == o.objective                      # bitwise (c8); contract: 1e-9 rel
    assert np.array_equal(g["x"], o.x)                  # contract: 1e-7 abs
    assert np.array_equal(g["y"], o.y)
    if tableau and o.T is not None:
        assert np.array_equal(g["T"], o.T)
        assert g["hash"] == oracle.tableau_hash(o.T)


def cases_small():
    out = [("classic",) + F.classic(), ("chvatal",) + F.chvatal(), ("unbounded",) + F.unbounded_1d(),
           ("beale",) + F.beale()]
    for name in ("entering_tie", "ratio_tie", "zero_iteration"):
        g = GOLD[name]
        out.append((name, np.array(g["A"], float), np.array(g["b"], float), np.array(g["c"], float)))
    return out


@pytest.mark.parametrize("case", cases_small(), ids=lambda c: c[0])
def test_worked_examples(sx, case):
    name, A, b, c = case
    o = oracle.solve(A, b, c, keep_tableau=True)
    g = gpu_solve(sx, A, b, c)
    assert_same(g, o)


@pytest.mark.parametrize("n", [3, 6, 10, 12])
def test_klee_minty(sx, n):
    A, b, c = F.klee_minty(n)
    o = oracle.solve(A, b, c, max_pivots=2 ** n + 5, keep_tableau=True)
    g = gpu_solve(sx, A, b, c, max_pivots=2 ** n + 5)
    assert g["pivots"] == 2 ** n - 1 and g["obj"] == 5.0 ** n
    assert_same(g, o)


@pytest.mark.parametrize("seed", range(1, 41))
def test_dense_64(sx, seed):
    A, b, c = lpgen.dense_lp(64, 64, seed)
    o = oracle.solve(A, b, c, keep_tableau=True)
    assert_same(gpu_solve(sx, A, b, c), o)


@pytest.mark.parametrize("seed", range(12))
def test_tie_heavy(sx, seed):
    rng = np.random.default_rng(seed)
    m, n = int(rng.integers(3, 40)), int(rng.integers(3, 40))
    A, b, c = F.tie_heavy(m, n, seed)
    A[:, A.sum(axis=0) == 0] = 1.0
    o = oracle.solve(A, b, c, keep_tableau=True)
    assert_same(gpu_solve(sx, A, b, c), o)


@pytest.mark.parametrize("m,n", [(1, 1), (1, 700), (700, 1), (3, 1500), (257, 513), (333, 1021),
                                 (1100, 90)])
def test_ragged_shapes(sx, m, n):
    # several column chunks (512 doubles), ragged chunk tails, many CTA segments
    A, b, c = lpgen.dense_lp(m, n, 1000 + m + n)
    o = oracle.solve(A, b, c, keep_tableau=True)
    assert_same(gpu_solve(sx, A, b, c), o)


@pytest.mark.parametrize("P", [2, 3, 4, 8])
def test_virtual_ranks_match(sx, P):
    # multi-GPU data flow (column slabs, candidate gather, column broadcast, redundant
    # ratio test) on one GPU: results identical to P = 1 and to the oracle
    A, b, c = lpgen.dense_lp(120, 200, 77)
    o = oracle.solve(A, b, c, keep_tableau=True)
    assert_same(gpu_solve(sx, A, b, c, virtual_ranks=P), o)


def test_virtual_ranks_ties(sx):
    A, b, c = F.tie_heavy(30, 37, 5)
    A[:, A.sum(axis=0) == 0] = 1.0
    o = oracle.solve(A, b, c, keep_tableau=True)
    for P in (2, 5, 8):
        assert_same(gpu_solve(sx, A, b, c, virtual_ranks=P), o)


def test_iterate_stepwise_bitwise(sx):
    # after EVERY pivot the device tableau equals the oracle's bit for bit
    A, b, c = lpgen.dense_lp(64, 64, 3)
    with sx.Simplex(A, b, c, segment_pivots=4, lookahead=1) as s:
        for t in range(1, 40):
            done, st = s.iterate(1)
            o = oracle.solve(A, b, c, stop_after=t, keep_tableau=True)
            if o.status != oracle.RUNNING:
                assert done == 0 and st == o.status
                break
            assert done == 1 and st == sx.RUNNING
            T, _ = s.tableau()
            assert np.array_equal(T, o.T), t
            assert s.tableau_hash() == oracle.tableau_hash(o.T)


def test_iterate_then_solve_equals_solve(sx):
    A, b, c = lpgen.dense_lp(300, 400, 9)
    o = oracle.solve(A, b, c, keep_tableau=True)
    with sx.Simplex(A, b, c, lookahead=1) as s:
        d1, st = s.iterate(17)
        assert d1 == 17 and st == sx.RUNNING
        d2, st = s.iterate(5)
        assert d2 == 5
        st = s.solve()
        x, y, obj, piv, _ = s.solution()
        k, r = s.trace()
    assert st == o.status and piv == o.pivots and obj == o.objective
    assert np.array_equal(k, o.trace_k) and np.array_equal(r, o.trace_r)


def test_reset_and_device_io(sx):
    import torch
    A, b, c = lpgen.dense_lp(200, 150, 4)
    o = oracle.solve(A, b, c, keep_tableau=True)
    A2, b2, c2 = lpgen.dense_lp(200, 150, 5)
    o2 = oracle.solve(A2, b2, c2)
    dA, db, dc = (torch.from_numpy(v).cuda() for v in (A, b, c))
    with sx.Simplex(dA, db, dc, lookahead=1) as s:
        assert s.solve() == sx.OPTIMAL
        dx = torch.empty(150, dtype=torch.float64, device="cuda")
        dy = torch.empty(200, dtype=torch.float64, device="cuda")
        _, _, obj, piv, _ = s.solution(dx, dy)
        assert obj == o.objective and piv == o.pivots
        assert np.array_equal(dx.cpu().numpy(), o.x) and np.array_equal(dy.cpu().numpy(), o.y)
        s.reset(A2, b2, c2)                       # host inputs, same shape
        assert s.solve() == o2.status
        x, y, obj, piv, _ = s.solution()
        assert obj == o2.objective and np.array_equal(x, o2.x) and piv == o2.pivots
        s.reset(dA, db, dc)
        s.solve()
        assert s.tableau_hash() == oracle.tableau_hash(o.T)


def test_errors(sx):
    A, b, c = F.classic()
    bad = A.copy()
    bad[1, 1] = np.nan
    with pytest.raises(sx.SimplexError) as e:
        sx.Simplex(bad, b, c)
    assert e.value.code == sx.E_NONFINITE if hasattr(sx, "E_NONFINITE") else -2
    with pytest.raises(sx.SimplexError) as e:
        sx.Simplex(A, -b, c, phase1=False)
    assert e.value.code == -3
    with pytest.raises(sx.SimplexError) as e:
        sx.Simplex(A, b, np.array([np.inf, 1.0]))
    assert e.value.code == -2
    with pytest.raises(sx.SimplexError) as e:
        sx.Simplex(A, b, c, virtual_ranks=100)     # more parts than columns
    assert e.value.code == -1


@pytest.mark.parametrize("seed", [2, 3, 4, 5])
def test_dense_1000_seeds_default_path(sx, seed):
    """SURVEY.md §8(d) seeds of the 1000x1000 config through the library default (rank-16
    look-ahead pipelined with the pass), against the oracle run live, plus the certificates
    computed from the raw (A, b, c): primal feasibility, dual feasibility, strong duality."""
    A, b, c = lpgen.dense_lp(1000, 1000, seed)
    o = oracle.solve(A, b, c, keep_tableau=True)
    g = gpu_solve(sx, A, b, c, lookahead=0)
    assert_same(g, o)
    x, y, obj = g["x"], g["y"], g["obj"]
    assert np.max(A @ x - b) <= 1e-6 and np.min(x) >= -1e-9
    assert np.min(y) >= -1e-7 and np.min(A.T @ y - c) >= -1e-6
    assert abs(c @ x - b @ y) <= 1e-9 * max(1.0, abs(obj))


@pytest.mark.parametrize("key", [(4000, 4000, 2), (4000, 4000, 3), (8000, 8000, 2)])
def test_golden_more_seeds_default_path(sx, key):
    """The other §8(d) seeds of the 4000^2 / 8000^2 configs (goldens written by
    scripts/make_golden.py from the oracle alone) through the bench's launch configuration."""
    path = os.path.join(GOLDEN_DIR, "dense_%dx%d_s%d.npz" % key)
    if not os.path.exists(path):
        pytest.skip("golden file not generated: " + os.path.basename(path))
    g = np.load(path)
    A, b, c = lpgen.dense_lp(*key)
    with sx.Simplex(A, b, c) as s:
        st = s.solve()
        x, y, obj, piv, _ = s.solution()
        k, r = s.trace()
        h = s.tableau_hash()
    assert st == int(g["status"]) and piv == int(g["pivots"])
    assert np.array_equal(k, g["trace_k"]) and np.array_equal(r, g["trace_r"])
    assert obj == float(g["objective"]) and np.array_equal(y, g["y"])
    xs = np.zeros(key[1])
    xs[g["x_idx"]] = g["x_val"]
    assert np.array_equal(x, xs)
    assert h == int(g["tableau_hash"])


@pytest.mark.parametrize("key", [(1000, 1000, 1), (4000, 4000, 1), (8000, 8000, 1)])
def test_golden_full_size(sx, key):
    """Bench-size configs against tests/golden (written by scripts/make_golden.py, oracle only)."""
    path = os.path.join(GOLDEN_DIR, "dense_%dx%d_s%d.npz" % key)
    if not os.path.exists(path):
        pytest.fail("missing golden file " + path)
    g = np.load(path)
    A, b, c = lpgen.dense_lp(*key)
    with sx.Simplex(A, b, c, lookahead=1) as s:
        st = s.solve()
        x, y, obj, piv, _ = s.solution()
        k, r = s.trace()
        h = s.tableau_hash()
    assert st == int(g["status"]) and piv == int(g["pivots"])
    assert np.array_equal(k, g["trace_k"]) and np.array_equal(r, g["trace_r"])
    assert obj == float(g["objective"])
    assert abs(obj - float(g["objective"])) <= 1e-9 * abs(float(g["objective"]))
    xs = np.zeros(key[1])
    xs[g["x_idx"]] = g["x_val"]
    assert np.max(np.abs(x - xs)) <= 1e-7 and np.array_equal(x, xs)
    assert np.array_equal(y, g["y"])
    assert h == int(g["tableau_hash"])
    cert = oracle.certificate(A, b, c, x, y)
    assert not cert.violations, cert.violations


def test_nccl_exchange_path_one_rank(sx):
    """The multi-GPU exchange (k_pack -> ncclAllGather captured in the CUDA graph ->
    k_select from the gathered buffer) run through a real 1-rank NCCL communicator."""
    A, b, c = lpgen.dense_lp(150, 230, 21)
    o = oracle.solve(A, b, c, keep_tableau=True)
    g = gpu_solve(sx, A, b, c, exchange=1)
    assert_same(g, o)


def test_wide_prefix_20000x40000_pipelined_512(sx):
    """BASELINE config 5 in the launch configuration bench.py times (library default: rank-16
    look-ahead, selection pipelined with the pass, two 9.6 GB tableau buffers): 32 blocks, the
    first 512 pivots, against the oracle's 512-pivot prefix run (tests/golden/*_p512.npz)."""
    g = np.load(os.path.join(GOLDEN_DIR, "dense_20000x40000_s1_p512.npz"))
    A, b, c = lpgen.dense_lp(20000, 40000, 1)
    with sx.Simplex(A, b, c) as s:
        done, st = s.iterate(512)
        assert done == 512 and st == sx.RUNNING
        k, r = s.trace()
        h = s.tableau_hash()
        x, y, obj, piv, _ = s.solution()
    assert np.array_equal(k, g["trace_k"]) and np.array_equal(r, g["trace_r"])
    assert obj == float(g["objective"])
    assert np.array_equal(y, g["y"])
    xs = np.zeros(40000)
    xs[g["x_idx"]] = g["x_val"]
    assert np.array_equal(x, xs)
    assert h == int(g["tableau_hash"])


def test_wide_prefix_20000x40000(sx):
    """BASELINE config 5 (~9.6 GB tableau): the first 32 pivots, row 0, rhs column and the
    whole-tableau digest against the oracle's prefix run (tests/golden/*_p32.npz)."""
    path = os.path.join(GOLDEN_DIR, "dense_20000x40000_s1_p32.npz")
    g = np.load(path)
    A, b, c = lpgen.dense_lp(20000, 40000, 1)
    for look in (1, 16):                     # one pivot per pass, and two rank-16 blocks
        with sx.Simplex(A, b, c, lookahead=look) as s:
            done, st = s.iterate(32)
            assert done == 32 and st == sx.RUNNING
            k, r = s.trace()
            h = s.tableau_hash()
            x, y, obj, piv, _ = s.solution()
        assert np.array_equal(k, g["trace_k"]) and np.array_equal(r, g["trace_r"])
        assert obj == float(g["objective"])
        assert np.array_equal(y, g["y"])
        xs = np.zeros(40000)
        xs[g["x_idx"]] = g["x_val"]
        assert np.array_equal(x, xs)
        assert h == int(g["tableau_hash"])



def _wide_prefixes():
    import glob
    import re
    out = {}
    for p in glob.glob(os.path.join(GOLDEN_DIR, "dense_20000x40000_s1_p*.npz")):
        mt = re.search(r"_p(\d+)\.npz$", p)
        if mt:
            out[int(mt.group(1))] = p
    return out


def test_wide_full_solve_20000x40000(sx):
    """BASELINE config 5 (the north_star's largest tableau, 9.6 GB) solved to the end on the
    library default path (the launch configuration bench.py times), checked against:
      * EVERY oracle prefix golden written by scripts/make_golden_long.py (the row-parallel oracle,
        bitwise equal to the single-thread one): the solve is stopped at exactly P pivots and its
        trace, objective, y, x and whole-tableau digest compared bit for bit, then resumed;
      * the oracle's full-solve golden when it exists (status, pivot count, whole trace, objective,
        x, y, digest);
      * always: a full optimality certificate from the RAW (A, b, c) in extended precision —
        primal feasibility (Ax <= b + 1e-6, x >= -1e-9), dual feasibility (A^T y >= c - 1e-7,
        y >= -1e-7) and strong duality |c^T x - b^T y| <= 1e-9 max(1, |obj|) (north_star)."""
    A, b, c = lpgen.dense_lp(20000, 40000, 1)
    pre = _wide_prefixes()
    full = os.path.join(GOLDEN_DIR, "dense_20000x40000_s1.npz")
    with sx.Simplex(A, b, c) as s:
        done = 0
        for P in sorted(pre):
            d, st = s.iterate(P - done)
            done += d
            assert done == P and st == sx.RUNNING
            g = np.load(pre[P])
            k, r = s.trace()
            x, y, obj, piv, _ = s.solution()
            assert piv == P
            assert np.array_equal(k, g["trace_k"]) and np.array_equal(r, g["trace_r"]), P
            assert obj == float(g["objective"]) and np.array_equal(y, g["y"]), P
            xs = np.zeros(40000)
            xs[g["x_idx"]] = g["x_val"]
            assert np.array_equal(x, xs), P
            assert s.tableau_hash() == int(g["tableau_hash"]), P
        st = s.solve()
        x, y, obj, piv, _ = s.solution()
        k, r = s.trace()
        h = s.tableau_hash()
    assert st == sx.OPTIMAL
    if os.path.exists(full):
        g = np.load(full)
        assert piv == int(g["pivots"]) and st == int(g["status"])
        assert np.array_equal(k, g["trace_k"]) and np.array_equal(r, g["trace_r"])
        assert obj == float(g["objective"]) and np.array_equal(y, g["y"])
        xs = np.zeros(40000)
        xs[g["x_idx"]] = g["x_val"]
        assert np.array_equal(x, xs) and h == int(g["tableau_hash"])
    cert = oracle.certificate(A, b, c, x, y)
    assert not cert.violations, cert.violations
    assert cert.gap_rel <= 1e-9
