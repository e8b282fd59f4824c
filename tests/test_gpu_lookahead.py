"""GPU parity of the rank-s look-ahead path: s pivots selected
ahead from chained corrections, one tableau pass applies them.  The claim is BITWISE
identity with s single pivots, so every check is exact equality with the oracle.  Every
case runs both schedules: the software pipeline (block b+1 selected while block b's pass
runs, two tableau buffers; the default) and select-then-pass in place (overlap=False)."""
import os

import numpy as np
import pytest

import lpgen
import oracle
from lpgen import fixtures as F

from test_gpu_parity import GOLD, GOLDEN_DIR, assert_same, gpu_solve  # noqa: F401

pytestmark = pytest.mark.gpu

LOOKS = [2, 4, 8, 16]


@pytest.fixture(scope="module")
def sx(cuda_device):
    import paper_2211_10979_b200 as sx
    return sx


@pytest.fixture(params=[True, False], ids=["pipe", "serial"])
def ov(request):
    return request.param


@pytest.mark.parametrize("look", LOOKS)
@pytest.mark.parametrize("name", ["classic", "chvatal", "unbounded", "beale", "entering_tie", "ratio_tie",
                                  "zero_iteration"])
def test_worked_examples(sx, name, look, ov):
    if name == "classic":
        A, b, c = F.classic()
    elif name == "chvatal":
        A, b, c = F.chvatal()
    elif name == "unbounded":
        A, b, c = F.unbounded_1d()
    elif name == "beale":
        A, b, c = F.beale()
    else:
        g = GOLD[name]
        A, b, c = (np.array(g[k], float) for k in ("A", "b", "c"))
    o = oracle.solve(A, b, c, keep_tableau=True)
    assert_same(gpu_solve(sx, A, b, c, lookahead=look, overlap=ov), o)


@pytest.mark.parametrize("look", LOOKS)
def test_klee_minty(sx, look, ov):
    A, b, c = F.klee_minty(9)                      # 511 pivots, many repeated pivot rows
    o = oracle.solve(A, b, c, max_pivots=600, keep_tableau=True)
    assert_same(gpu_solve(sx, A, b, c, max_pivots=600, lookahead=look, overlap=ov), o)


@pytest.mark.parametrize("look", LOOKS)
@pytest.mark.parametrize("seed", [1, 2, 3, 4, 5, 6])
def test_dense_64(sx, seed, look, ov):
    A, b, c = lpgen.dense_lp(64, 64, seed)
    o = oracle.solve(A, b, c, keep_tableau=True)
    assert_same(gpu_solve(sx, A, b, c, lookahead=look, overlap=ov), o)


@pytest.mark.parametrize("look", [3, 8, 16])
@pytest.mark.parametrize("seed", range(10))
def test_tie_heavy(sx, seed, look, ov):
    rng = np.random.default_rng(seed)
    m, n = int(rng.integers(3, 40)), int(rng.integers(3, 40))
    A, b, c = F.tie_heavy(m, n, seed)
    A[:, A.sum(axis=0) == 0] = 1.0
    o = oracle.solve(A, b, c, keep_tableau=True)
    assert_same(gpu_solve(sx, A, b, c, lookahead=look, overlap=ov), o)


@pytest.mark.parametrize("look", [5, 16])
@pytest.mark.parametrize("m,n", [(1, 1), (1, 700), (700, 1), (3, 1500), (257, 513), (1100, 90)])
def test_ragged_shapes(sx, m, n, look, ov):
    A, b, c = lpgen.dense_lp(m, n, 1000 + m + n)
    o = oracle.solve(A, b, c, keep_tableau=True)
    assert_same(gpu_solve(sx, A, b, c, lookahead=look, overlap=ov), o)


def test_iteration_cap_inside_a_block(sx, ov):
    A, b, c = F.klee_minty(6)                      # 63 pivots; cap 21 falls inside a block of 8
    o = oracle.solve(A, b, c, max_pivots=21, keep_tableau=True)
    assert o.status == oracle.ITERATION_LIMIT
    assert_same(gpu_solve(sx, A, b, c, max_pivots=21, lookahead=8, overlap=ov), o)


@pytest.mark.parametrize("seg", [8, 16, 40])
def test_iterate_stepwise_bitwise(sx, ov, seg):
    A, b, c = lpgen.dense_lp(64, 64, 3)
    with sx.Simplex(A, b, c, lookahead=8, segment_pivots=seg, overlap=ov) as s:
        done_total = 0
        for step in (1, 3, 7, 8, 2, 16):
            done, st = s.iterate(step)
            done_total += done
            o = oracle.solve(A, b, c, stop_after=done_total, keep_tableau=True)
            T, _ = s.tableau()
            assert np.array_equal(T, o.T), done_total
            if st != sx.RUNNING:
                break


@pytest.mark.parametrize("key", [(1000, 1000, 1), (4000, 4000, 1)])
@pytest.mark.parametrize("look", [8, 16])
def test_golden(sx, key, look, ov):
    g = np.load(os.path.join(GOLDEN_DIR, "dense_%dx%d_s%d.npz" % key))
    A, b, c = lpgen.dense_lp(*key)
    with sx.Simplex(A, b, c, lookahead=look, overlap=ov) as s:
        st = s.solve()
        x, y, obj, piv, _ = s.solution()
        k, r = s.trace()
        h = s.tableau_hash()
    assert st == int(g["status"]) and piv == int(g["pivots"])
    assert np.array_equal(k, g["trace_k"]) and np.array_equal(r, g["trace_r"])
    assert obj == float(g["objective"]) and np.array_equal(y, g["y"])
    assert h == int(g["tableau_hash"])


def test_golden_8000_default_path(sx):
    """The bench workload through the library default (rank-16 look-ahead) against the
    oracle's full 8000x8000 solve (tests/golden, ~69 min of single-thread oracle)."""
    g = np.load(os.path.join(GOLDEN_DIR, "dense_8000x8000_s1.npz"))
    A, b, c = lpgen.dense_lp(8000, 8000, 1)
    with sx.Simplex(A, b, c) as s:
        st = s.solve()
        x, y, obj, piv, _ = s.solution()
        k, r = s.trace()
        h = s.tableau_hash()
    assert st == int(g["status"]) and piv == int(g["pivots"]) == 25395
    assert np.array_equal(k, g["trace_k"]) and np.array_equal(r, g["trace_r"])
    assert obj == float(g["objective"]) and np.array_equal(y, g["y"])
    xs = np.zeros(8000)
    xs[g["x_idx"]] = g["x_val"]
    assert np.array_equal(x, xs)
    assert h == int(g["tableau_hash"])
    cert = oracle.certificate(A, b, c, x, y)
    assert not cert.violations, cert.violations


# ---- multi-part rank-s look-ahead (column slabs; k_mlook + one candidate-column exchange per
# pivot, then one pass per slab): virtual slabs on one GPU and the real 1-rank NCCL exchange

@pytest.fixture(params=[2, 0], ids=["peer", "direct"])
def xch(request):
    """exchange 2: the peer-memory protocol (slot stores + released flags, waited on by the
    next k_mlook); 0 on virtual slabs: slots written into the shared gather buffer, stream
    order only."""
    return request.param


@pytest.mark.parametrize("look", [4, 16])
@pytest.mark.parametrize("P", [2, 3, 5, 8])
def test_multipart_dense(sx, P, look, xch):
    A, b, c = lpgen.dense_lp(120, 200, 77)
    o = oracle.solve(A, b, c, keep_tableau=True)
    assert_same(gpu_solve(sx, A, b, c, virtual_ranks=P, lookahead=look, exchange=xch), o)


@pytest.mark.parametrize("P", [2, 4])
def test_multipart_klee_minty_and_ties(sx, P, xch):
    A, b, c = F.klee_minty(8)                      # repeated pivot rows inside blocks
    o = oracle.solve(A, b, c, max_pivots=300, keep_tableau=True)
    assert_same(gpu_solve(sx, A, b, c, max_pivots=300, virtual_ranks=P, lookahead=16, exchange=xch), o)
    for seed in range(4):
        A, b, c = F.tie_heavy(25, 31, seed)
        A[:, A.sum(axis=0) == 0] = 1.0
        o = oracle.solve(A, b, c, keep_tableau=True)
        assert_same(gpu_solve(sx, A, b, c, virtual_ranks=P, lookahead=8, exchange=xch), o)


@pytest.mark.parametrize("look", [5, 16])
@pytest.mark.parametrize("P", [2, 3, 4])
def test_multipart_peer_exchange_without_pipeline(sx, P, look):
    """k_mblock per block, select-then-pass (overlap = 0); the default (overlap = 1) selects block
    b+1 from the tableau before block b's slab passes while they run, on two buffers per slab."""
    A, b, c = lpgen.dense_lp(150, 170, 9)
    o = oracle.solve(A, b, c, keep_tableau=True)
    assert_same(gpu_solve(sx, A, b, c, virtual_ranks=P, lookahead=look, exchange=2, overlap=False), o)
    assert_same(gpu_solve(sx, A, b, c, virtual_ranks=P, lookahead=look, exchange=2, overlap=True), o)


@pytest.mark.parametrize("P", [2, 5])
def test_multipart_peer_exchange_per_pivot_launches(sx, P):
    """The peer-memory protocol with one k_mlook launch per pivot (exchange = 3) instead of
    one k_mblock per block (the virtual slabs then run in stream order, not concurrently)."""
    A, b, c = lpgen.dense_lp(120, 200, 77)
    o = oracle.solve(A, b, c, keep_tableau=True)
    assert_same(gpu_solve(sx, A, b, c, virtual_ranks=P, lookahead=16, exchange=3), o)


def test_multipart_peer_exchange_reset_and_options(sx):
    """The exchange counters are monotone over the handle's life: a reset and a second solve
    reuse the flags; exchange = 2 (peer memory required) works on one GPU; bad values fail."""
    A, b, c = lpgen.dense_lp(90, 140, 5)
    o = oracle.solve(A, b, c, keep_tableau=True)
    with sx.Simplex(A, b, c, virtual_ranks=3, lookahead=16, exchange=2) as s:
        for _ in range(3):
            st = s.solve()
            x, y, obj, piv, _ = s.solution()
            k, r = s.trace()
            assert st == o.status and piv == o.pivots and obj == o.objective
            assert np.array_equal(k, o.trace_k) and np.array_equal(r, o.trace_r)
            assert np.array_equal(x, o.x) and np.array_equal(y, o.y)
            s.reset(A, b, c)
    with pytest.raises(sx.SimplexError):
        sx.Simplex(A, b, c, virtual_ranks=2, exchange=4)


@pytest.mark.parametrize("m,n", [(1, 9), (7, 1), (300, 40), (90, 1100)])
def test_multipart_ragged(sx, m, n):
    A, b, c = lpgen.dense_lp(m, n, 500 + m + n)
    o = oracle.solve(A, b, c, keep_tableau=True)
    P = min(3, n + m)
    assert_same(gpu_solve(sx, A, b, c, virtual_ranks=P, lookahead=16), o)


def test_multipart_bland_and_cap(sx):
    A, b, c = lpgen.dense_lp(60, 80, 4)
    o = oracle.solve(A, b, c, rule=oracle.BLAND, keep_tableau=True)
    assert_same(gpu_solve(sx, A, b, c, virtual_ranks=3, lookahead=16, pivot_rule=sx.BLAND), o)
    A, b, c = F.klee_minty(6)
    o = oracle.solve(A, b, c, max_pivots=21, keep_tableau=True)
    assert_same(gpu_solve(sx, A, b, c, virtual_ranks=2, lookahead=8, max_pivots=21), o)


def test_multipart_iterate_stepwise(sx, xch):
    A, b, c = lpgen.dense_lp(64, 64, 3)
    with sx.Simplex(A, b, c, lookahead=8, segment_pivots=16, virtual_ranks=3, exchange=xch) as s:
        done_total = 0
        for step in (1, 3, 7, 8, 2, 16, 50):
            done, st = s.iterate(step)
            done_total += done
            o = oracle.solve(A, b, c, stop_after=done_total, keep_tableau=True)
            T, _ = s.tableau()
            assert np.array_equal(T, o.T), done_total
            if st != sx.RUNNING:
                break


def test_multipart_nccl_one_rank(sx):
    """k_mlook with the captured ncclAllGather of candidate columns, 1-rank communicator
    (exchange = 1 on one column part)."""
    A, b, c = lpgen.dense_lp(150, 230, 21)
    o = oracle.solve(A, b, c, keep_tableau=True)
    assert_same(gpu_solve(sx, A, b, c, lookahead=16, exchange=1), o)


def test_multipart_golden_1000(sx):
    g = np.load(os.path.join(GOLDEN_DIR, "dense_1000x1000_s1.npz"))
    A, b, c = lpgen.dense_lp(1000, 1000, 1)
    with sx.Simplex(A, b, c, virtual_ranks=4) as s:          # automatic: rank-16 look-ahead
        st = s.solve()
        x, y, obj, piv, _ = s.solution()
        k, r = s.trace()
        h = s.tableau_hash()
    assert st == int(g["status"]) and piv == int(g["pivots"])
    assert np.array_equal(k, g["trace_k"]) and np.array_equal(r, g["trace_r"])
    assert obj == float(g["objective"]) and np.array_equal(y, g["y"])
    assert h == int(g["tableau_hash"])


# Which selection kernel a handle runs (stats.path): k_look2, the shared-memory selection
# (path 3), when one column part has m + 1 <= 4096 rows and a pitch <= 8192
# doubles; k_lookahead (path 0) beyond.  Both must be bitwise the oracle's pivots on each side of
# the boundary, with the cluster's round-robin 32-element chunks ending raggedly.
_ORACLE_120 = {}


@pytest.mark.parametrize("m,n,want", [(1000, 1000, 3), (2000, 2000, 3), (4095, 300, 3), (4096, 200, 0),
                                      (4100, 300, 0), (3000, 5300, 0), (77, 4000, 3)])
def test_selection_kernel_choice(sx, m, n, want, ov):
    A, b, c = lpgen.dense_lp(m, n, 7)
    if (m, n) not in _ORACLE_120:
        _ORACLE_120[(m, n)] = oracle.solve(A, b, c, max_pivots=120, keep_tableau=True)
    o = _ORACLE_120[(m, n)]
    with sx.Simplex(A, b, c, max_pivots=120, overlap=ov) as s:
        assert s.stats().path == want
    assert_same(gpu_solve(sx, A, b, c, max_pivots=120, lookahead=0, overlap=ov), o)


def test_look2_two_columns_iterate_windows(sx, ov):
    """k_look2's two-column configuration (pitch > 4096 doubles) stopped inside blocks: every window
    end leaves a partial bank whose hand-off the next launch chains first (spre < 16)."""
    A, b, c = lpgen.dense_lp(2600, 2000, 11)             # pitch 4608: two own columns per thread
    with sx.Simplex(A, b, c, overlap=ov) as s:
        assert s.stats().path == 3
        done_total = 0
        for step in (5, 23, 37, 16, 19):
            done, st = s.iterate(step)
            done_total += done
            o = oracle.solve(A, b, c, stop_after=done_total, keep_tableau=True)
            T, _ = s.tableau()
            k, r = s.trace()
            assert np.array_equal(k, o.trace_k) and np.array_equal(r, o.trace_r), done_total
            assert np.array_equal(T, o.T), done_total
            if st != sx.RUNNING:
                break
