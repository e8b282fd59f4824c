"""GPU parity of the pair schedule (lookahead 17..32): bank 0 (16 pivots) selected from the
tableau, bank 1 selected from the SAME tableau chaining bank 0 first, then ONE pass applies the
up-to-32 chains per element in the oracle's order.  The claim is bitwise identity with single
pivots (the chains are the oracle's operations in the oracle's order), so every
check is exact equality with the oracle: trace, objective, x, y and the whole tableau."""
import os

import numpy as np
import pytest

import lpgen
import oracle
from lpgen import fixtures as F

from test_gpu_parity import GOLD, GOLDEN_DIR, assert_same, gpu_solve  # noqa: F401

pytestmark = pytest.mark.gpu

LOOKS = [17, 24, 32]


@pytest.fixture(scope="module")
def sx(cuda_device):
    import paper_2211_10979_b200 as sx
    return sx


@pytest.mark.parametrize("look", LOOKS)
@pytest.mark.parametrize("name", ["classic", "chvatal", "unbounded", "beale", "entering_tie", "ratio_tie",
                                  "zero_iteration"])
def test_worked_examples(sx, name, look):
    if name in ("classic", "chvatal", "beale"):
        A, b, c = getattr(F, name)()
    elif name == "unbounded":
        A, b, c = F.unbounded_1d()
    else:
        g = GOLD[name]
        A, b, c = (np.array(g[k], float) for k in ("A", "b", "c"))
    o = oracle.solve(A, b, c, keep_tableau=True)
    assert_same(gpu_solve(sx, A, b, c, lookahead=look), o)


@pytest.mark.parametrize("look", LOOKS)
def test_klee_minty(sx, look):
    """Repeated pivot rows inside a block of 32 (Klee-Minty revisits rows constantly)."""
    A, b, c = F.klee_minty(9)                      # 511 pivots
    o = oracle.solve(A, b, c, max_pivots=600, keep_tableau=True)
    assert_same(gpu_solve(sx, A, b, c, max_pivots=600, lookahead=look), o)


@pytest.mark.parametrize("seed", [1, 2, 3, 4, 5, 6])
def test_dense_64(sx, seed):
    A, b, c = lpgen.dense_lp(64, 64, seed)
    o = oracle.solve(A, b, c, keep_tableau=True)
    assert_same(gpu_solve(sx, A, b, c, lookahead=32), o)


@pytest.mark.parametrize("look", [20, 32])
@pytest.mark.parametrize("seed", range(10))
def test_tie_heavy(sx, seed, look):
    rng = np.random.default_rng(seed)
    m, n = int(rng.integers(3, 40)), int(rng.integers(3, 40))
    A, b, c = F.tie_heavy(m, n, seed)
    A[:, A.sum(axis=0) == 0] = 1.0
    o = oracle.solve(A, b, c, keep_tableau=True)
    assert_same(gpu_solve(sx, A, b, c, lookahead=look), o)


@pytest.mark.parametrize("m,n", [(1, 1), (1, 700), (700, 1), (3, 1500), (257, 513), (1100, 90)])
def test_ragged_shapes(sx, m, n):
    A, b, c = lpgen.dense_lp(m, n, 1000 + m + n)
    o = oracle.solve(A, b, c, keep_tableau=True)
    assert_same(gpu_solve(sx, A, b, c, lookahead=32), o)


@pytest.mark.parametrize("cap", [7, 16, 21, 32, 40])
def test_iteration_cap_in_either_bank(sx, cap):
    """The cap falls inside bank 0, at the bank boundary, inside bank 1, at the pass boundary."""
    A, b, c = F.klee_minty(6)                      # 63 pivots
    o = oracle.solve(A, b, c, max_pivots=cap, keep_tableau=True)
    assert o.status == oracle.ITERATION_LIMIT
    assert_same(gpu_solve(sx, A, b, c, max_pivots=cap, lookahead=32), o)


@pytest.mark.parametrize("seg", [16, 32, 64])
def test_iterate_stepwise_bitwise(sx, seg):
    A, b, c = lpgen.dense_lp(64, 64, 3)
    with sx.Simplex(A, b, c, lookahead=32, segment_pivots=seg) as s:
        done_total = 0
        for step in (1, 3, 17, 16, 2, 33):
            done, st = s.iterate(step)
            done_total += done
            o = oracle.solve(A, b, c, stop_after=done_total, keep_tableau=True)
            T, _ = s.tableau()
            assert np.array_equal(T, o.T), done_total
            if st != sx.RUNNING:
                break


@pytest.mark.parametrize("key", [(1000, 1000, 1), (4000, 4000, 1)])
def test_golden(sx, key):
    g = np.load(os.path.join(GOLDEN_DIR, "dense_%dx%d_s%d.npz" % key))
    A, b, c = lpgen.dense_lp(*key)
    with sx.Simplex(A, b, c, lookahead=32) as s:
        st = s.solve()
        x, y, obj, piv, _ = s.solution()
        k, r = s.trace()
        h = s.tableau_hash()
    assert st == int(g["status"]) and piv == int(g["pivots"])
    assert np.array_equal(k, g["trace_k"]) and np.array_equal(r, g["trace_r"])
    assert obj == float(g["objective"]) and np.array_equal(y, g["y"])
    assert h == int(g["tableau_hash"])


def test_lookahead_limits(sx):
    A, b, c = F.classic()
    with pytest.raises(sx.SimplexError):
        sx.Simplex(A, b, c, lookahead=33)
    with pytest.raises(sx.SimplexError):
        sx.Simplex(A, b, c, lookahead=32, virtual_ranks=2)
