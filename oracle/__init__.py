"""oracle — plain CPU reference for the dense-tableau simplex hot path.

TEST INFRASTRUCTURE ONLY.  Only tests/, ``__graft_entry__.smoke()`` and
bench.py's ``cpu_baseline`` / ``--impl reference`` legs may import this package.
The product (``paper_2211_10979_b200``) never imports it, and it imports
nothing from the product.

The arithmetic lives in ``simplex_oracle.c`` (single-threaded C, IEEE binary64,
``-ffp-contract=off``, explicit ``fma``), one function per step of PAPER.md §III;
this module is ctypes marshalling only, plus the certificate checks of
SPEC.md:90-98 computed from the RAW (A, b, c) in extended precision.
"""
from __future__ import annotations

import ctypes as C
import os
import subprocess
from dataclasses import dataclass, field

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
_SRC = os.path.join(_HERE, "simplex_oracle.c")
_LIB = os.path.join(_HERE, "liboracle.so")

RUNNING, OPTIMAL, UNBOUNDED, INFEASIBLE, ITERATION_LIMIT = -1, 0, 2, 3, 4
STATUS_NAME = {RUNNING: "RUNNING", OPTIMAL: "OPTIMAL", UNBOUNDED: "UNBOUNDED", INFEASIBLE: "INFEASIBLE",
               ITERATION_LIMIT: "ITERATION_LIMIT"}
E_ARG, E_NONFINITE, E_NEG_RHS, E_OOM = -1, -2, -3, -4

TOL_OPT = 1e-7      # SURVEY.md §8(c) c3 / SPEC.md:110
TOL_PIV = 1e-10     # c5 / SPEC.md:110


_LIB_OMP = os.path.join(_HERE, "liboracle_omp.so")


def build(force: bool = False, parallel: bool = False) -> str:
    """Compile simplex_oracle.c -> liboracle.so (gcc, -O2 -ffp-contract=off).
    parallel=True builds liboracle_omp.so: the same source with -fopenmp, which
    splits only or_pivot's independent row loop (bitwise identical results)."""
    out = _LIB_OMP if parallel else _LIB
    if force or not os.path.exists(out) or os.path.getmtime(out) < os.path.getmtime(_SRC):
        cmd = ["gcc", "-O2", "-ffp-contract=off", "-fno-fast-math", "-march=x86-64-v3",
               "-fPIC", "-shared"] + (["-fopenmp"] if parallel else []) + \
              ["-o", out + ".tmp", _SRC, "-lm"]
        subprocess.check_call(cmd)
        os.replace(out + ".tmp", out)
    return out


_libs = {}


def lib(parallel: bool = False):
    """The oracle library; parallel=True -> the row-parallel -fopenmp build
    (threads from OMP_NUM_THREADS)."""
    if parallel not in _libs:
        L = C.CDLL(build(parallel=parallel))
        i64, dp, ip = C.c_int64, C.POINTER(C.c_double), C.POINTER(C.c_int64)
        L.or_build.argtypes = [i64, i64, dp, dp, dp, dp, ip]
        L.or_build.restype = C.c_int
        L.or_price.argtypes = [dp, i64, C.c_double, dp]
        L.or_price.restype = i64
        L.or_ratio.argtypes = [i64, i64, dp, i64, C.c_double, dp]
        L.or_ratio.restype = i64
        L.or_pivot.argtypes = [i64, i64, dp, i64, i64, dp, dp]
        L.or_pivot.restype = None
        L.or_extract.argtypes = [i64, i64, dp, ip, dp, dp, dp]
        L.or_extract.restype = None
        L.or_solve.argtypes = [i64, i64, dp, dp, dp, C.c_double, C.c_double, i64, i64,
                               C.POINTER(C.c_int32), C.POINTER(C.c_int32), i64,
                               dp, dp, dp, ip, C.POINTER(C.c_int), dp, ip]
        L.or_solve.restype = C.c_int
        L.or_price_bland.argtypes = [dp, i64, C.c_double]
        L.or_price_bland.restype = i64
        L.or_ratio_bland.argtypes = [i64, i64, dp, i64, C.c_double, ip, dp]
        L.or_ratio_bland.restype = i64
        L.or_solve_rule.argtypes = [i64, i64, dp, dp, dp, C.c_double, C.c_double, i64, i64, C.c_int,
                                    C.POINTER(C.c_int32), C.POINTER(C.c_int32), i64,
                                    dp, dp, dp, ip, C.POINTER(C.c_int), dp, ip]
        L.or_solve_rule.restype = C.c_int
        L.or_solve_2phase.argtypes = [i64, i64, dp, dp, dp, C.c_double, C.c_double, i64, C.c_int,
                                      C.POINTER(C.c_int32), C.POINTER(C.c_int32), i64,
                                      dp, dp, dp, ip, C.POINTER(C.c_int), ip]
        L.or_solve_2phase.restype = C.c_int
        L.or_brute_force.argtypes = [i64, i64, dp, dp, dp, C.c_double, dp, dp]
        L.or_brute_force.restype = C.c_int
        L.or_iterate.argtypes = [i64, i64, dp, ip, C.c_double, C.c_double, i64, i64, C.c_int,
                                 C.POINTER(C.c_int32), C.POINTER(C.c_int32), i64, ip, dp, dp]
        L.or_iterate.restype = C.c_int
        _libs[parallel] = L
    return _libs[parallel]


def _dp(a):
    return a.ctypes.data_as(C.POINTER(C.c_double)) if a is not None else None


def _f64(a):
    return np.ascontiguousarray(a, dtype=np.float64)


class OracleError(RuntimeError):
    def __init__(self, code):
        super().__init__(f"oracle error {code}")
        self.code = code


# ---------------------------------------------------------------- single steps
def build_tableau(A, b, c):
    """Table I -> (T (m+1, n+m+1), basis (m,))."""
    A, b, c = _f64(A), _f64(b), _f64(c)
    m, n = A.shape
    T = np.empty((m + 1, n + m + 1))
    basis = np.empty(m, dtype=np.int64)
    err = lib().or_build(m, n, _dp(A), _dp(b), _dp(c), _dp(T),
                         basis.ctypes.data_as(C.POINTER(C.c_int64)))
    if err:
        raise OracleError(err)
    return T, basis


def price(row0, tol_opt=TOL_OPT):
    """Step 1 over a row fragment -> (k or -1, value)."""
    row0 = _f64(row0)
    v = C.c_double()
    k = lib().or_price(_dp(row0), row0.size, tol_opt, C.byref(v))
    return int(k), v.value


def ratio(T, k, tol_piv=TOL_PIV):
    """Step 2 on a full tableau -> (r in [1, m] or -1, min ratio)."""
    T = _f64(T)
    q = C.c_double()
    r = lib().or_ratio(T.shape[0] - 1, T.shape[1], _dp(T), k, tol_piv, C.byref(q))
    return int(r), q.value


def price_bland(row0, tol_opt=TOL_OPT):
    """Bland's entering rule: first j with T[0][j] < -tol_opt, or -1."""
    row0 = _f64(row0)
    return int(lib().or_price_bland(_dp(row0), row0.size, tol_opt))


def ratio_bland(T, k, basis, tol_piv=TOL_PIV):
    """Bland's leaving rule: min ratio, exact ties -> smallest basic-variable index."""
    T = _f64(T)
    basis = np.ascontiguousarray(basis, dtype=np.int64)
    q = C.c_double()
    r = lib().or_ratio_bland(T.shape[0] - 1, T.shape[1], _dp(T), k, tol_piv,
                             basis.ctypes.data_as(C.POINTER(C.c_int64)), C.byref(q))
    return int(r), q.value


def pivot(T, r, k):
    """Step 3, in place on a C-contiguous float64 tableau."""
    assert T.dtype == np.float64 and T.flags.c_contiguous
    col = np.empty(T.shape[0])
    prow = np.empty(T.shape[1])
    lib().or_pivot(T.shape[0] - 1, T.shape[1], _dp(T), r, k, _dp(col), _dp(prow))
    return T


def extract(T, basis, n):
    m = T.shape[0] - 1
    x, y, obj = np.empty(n), np.empty(m), C.c_double()
    T = _f64(T)
    basis = np.ascontiguousarray(basis, dtype=np.int64)
    lib().or_extract(m, n, _dp(T), basis.ctypes.data_as(C.POINTER(C.c_int64)),
                     _dp(x), _dp(y), C.byref(obj))
    return x, y, obj.value


# ---------------------------------------------------------------- whole solve
@dataclass
class Result:
    status: int
    pivots: int
    objective: float
    x: np.ndarray
    y: np.ndarray
    trace_k: np.ndarray
    trace_r: np.ndarray
    T: np.ndarray | None = None
    basis: np.ndarray | None = None

    @property
    def status_name(self):
        return STATUS_NAME[self.status]

    def trace(self):
        return list(zip(self.trace_k.tolist(), self.trace_r.tolist()))


DANTZIG, BLAND = 0, 1


def solve(A, b, c, *, tol_opt=TOL_OPT, tol_piv=TOL_PIV, max_pivots=0, stop_after=-1,
          trace_cap=None, keep_tableau=False, rule=DANTZIG, parallel=False) -> Result:
    """Run the oracle (§III Steps Init/1/2/3/Iterate); rule DANTZIG or BLAND.
    parallel=True runs the row-parallel build (same bits, see build())."""
    A, b, c = _f64(A), _f64(b), _f64(c)
    m, n = A.shape
    if trace_cap is None:
        trace_cap = max_pivots if max_pivots > 0 else 20 * (m + n)
        if stop_after >= 0:
            trace_cap = min(trace_cap, stop_after)
    tk = np.zeros(max(trace_cap, 1), dtype=np.int32)
    tr = np.zeros(max(trace_cap, 1), dtype=np.int32)
    x, y = np.empty(n), np.empty(m)
    obj, piv, st = C.c_double(), C.c_int64(), C.c_int()
    T = np.empty((m + 1, n + m + 1)) if keep_tableau else None
    basis = np.empty(m, dtype=np.int64) if keep_tableau else None
    err = lib(parallel).or_solve_rule(m, n, _dp(A), _dp(b), _dp(c), tol_opt, tol_piv, max_pivots, stop_after, rule,
                         tk.ctypes.data_as(C.POINTER(C.c_int32)),
                         tr.ctypes.data_as(C.POINTER(C.c_int32)), trace_cap,
                         _dp(x), _dp(y), C.byref(obj), C.byref(piv), C.byref(st),
                         _dp(T), basis.ctypes.data_as(C.POINTER(C.c_int64)) if keep_tableau else None)
    if err:
        raise OracleError(err)
    npiv = piv.value
    keep = min(npiv, trace_cap)
    return Result(st.value, npiv, obj.value, x, y, tk[:keep].copy(), tr[:keep].copy(), T, basis)


def iterate(T, basis, it, *, tol_opt=TOL_OPT, tol_piv=TOL_PIV, cap=None, stop_at=-1,
            rule=DANTZIG, parallel=False):
    """Continue the Iterate loop in place on a built tableau T (as from
    build_tableau) and basis, after ``it`` pivots already done.  Returns
    (status, total pivots, trace_k, trace_r) with the trace of THIS call only; a
    RUNNING status means stop_at was reached and a later call resumes the identical
    sequence.  cap defaults to 20(m+n) (reading c12)."""
    assert T.dtype == np.float64 and T.flags.c_contiguous and basis.dtype == np.int64
    m = T.shape[0] - 1
    n = T.shape[1] - m - 1
    if cap is None:
        cap = 20 * (m + n)
    tcap = max(1, (stop_at - it) if stop_at >= 0 else cap - it + 1)
    tk = np.zeros(tcap, dtype=np.int32)
    tr = np.zeros(tcap, dtype=np.int32)
    itc = C.c_int64(it)
    col, prow = np.empty(m + 1), np.empty(T.shape[1])
    st = lib(parallel).or_iterate(m, n, _dp(T), basis.ctypes.data_as(C.POINTER(C.c_int64)),
                                  tol_opt, tol_piv, cap, stop_at, rule,
                                  tk.ctypes.data_as(C.POINTER(C.c_int32)),
                                  tr.ctypes.data_as(C.POINTER(C.c_int32)), tcap,
                                  C.byref(itc), _dp(col), _dp(prow))
    done = itc.value - it
    return int(st), itc.value, tk[:done].copy(), tr[:done].copy()


def solve_2phase(A, b, c, *, tol_opt=TOL_OPT, tol_piv=TOL_PIV, max_pivots=0, rule=DANTZIG,
                 trace_cap=None, parallel=False):
    """Two-phase method: b may have negative entries.
    Returns a Result (no tableau) with .phase1_pivots."""
    A, b, c = _f64(A), _f64(b), _f64(c)
    m, n = A.shape
    if trace_cap is None:
        trace_cap = max_pivots if max_pivots > 0 else 20 * (m + n)
    tk = np.zeros(max(trace_cap, 1), dtype=np.int32)
    tr = np.zeros(max(trace_cap, 1), dtype=np.int32)
    x, y = np.empty(n), np.empty(m)
    obj, piv, st, p1 = C.c_double(), C.c_int64(), C.c_int(), C.c_int64(-1)
    err = lib(parallel).or_solve_2phase(m, n, _dp(A), _dp(b), _dp(c), tol_opt, tol_piv, max_pivots, rule,
                                tk.ctypes.data_as(C.POINTER(C.c_int32)),
                                tr.ctypes.data_as(C.POINTER(C.c_int32)), trace_cap,
                                _dp(x), _dp(y), C.byref(obj), C.byref(piv), C.byref(st), C.byref(p1))
    if err:
        raise OracleError(err)
    keep = min(piv.value, trace_cap)
    res = Result(st.value, piv.value, obj.value, x, y, tk[:keep].copy(), tr[:keep].copy())
    res.phase1_pivots = p1.value
    return res


def brute_force(A, b, c, feas_tol=1e-9):
    """Vertex enumeration: (found, objective, x) for m+n <= 24."""
    A, b, c = _f64(A), _f64(b), _f64(c)
    m, n = A.shape
    x = np.zeros(n)
    obj = C.c_double()
    found = lib().or_brute_force(m, n, _dp(A), _dp(b), _dp(c), feas_tol, C.byref(obj), _dp(x))
    if found < 0:
        raise ValueError("brute force limited to m+n <= 24")
    return bool(found), obj.value, x


# ---------------------------------------------------------------- certificates
@dataclass
class Certificate:
    primal_violation: float       # max(Ax - b), max(-x)   (want <= 1e-6 / 1e-9)
    dual_violation: float         # max(c - A^T y), max(-y) (want <= 1e-7)
    duality_gap: float            # |c^T x - b^T y|
    objective: float
    violations: list = field(default_factory=list)

    @property
    def gap_rel(self):
        return self.duality_gap / max(1.0, abs(self.objective))


def certificate(A, b, c, x, y, *, feas_tol=1e-6, dual_tol=1e-7, gap_tol=1e-9) -> Certificate:
    """Optimality certificate from the RAW data (north_star strong duality
    |c^T x - b^T y| <= 1e-9 max(1, |obj|)).  Extended precision (np.longdouble)."""
    L = np.longdouble
    A, b, c, x, y = (np.asarray(v, dtype=L) for v in (A, b, c, x, y))
    Ax = A @ x
    ATy = A.T @ y
    cx = float((c * x).sum())
    by = float((b * y).sum())
    pv = float(max((Ax - b).max(initial=-np.inf), (-x).max(initial=-np.inf)))
    dv = float(max((c - ATy).max(initial=-np.inf), (-y).max(initial=-np.inf)))
    cert = Certificate(pv, dv, abs(cx - by), cx)
    if pv > feas_tol:
        cert.violations.append(f"primal infeasible by {pv:g}")
    if dv > dual_tol:
        cert.violations.append(f"dual infeasible by {dv:g}")
    if cert.gap_rel > gap_tol:
        cert.violations.append(f"duality gap {cert.gap_rel:g} (rel)")
    return cert


# ---------------------------------------------------------------- tableau hash
_H_GOLDEN = np.uint64(0x9E3779B97F4A7C15)
_H_SALT = np.uint64(0xD1B54A32D192ED03)


def _mix64(z):
    with np.errstate(over="ignore"):
        z = (z ^ (z >> np.uint64(30))) * np.uint64(0xBF58476D1CE4E5B9)
        z = (z ^ (z >> np.uint64(27))) * np.uint64(0x94D049BB133111EB)
        return z ^ (z >> np.uint64(31))


def tableau_hash(T, chunk_rows=256) -> int:
    """Order-independent 64-bit digest of a logical (m+1) x W tableau, used to compare
    tableaux bit for bit without shipping them:
        H = sum_e mix64(bits(T_e) ^ (e * 0x9E3779B97F4A7C15 + 0xD1B54A32D192ED03))  mod 2^64
    with e = i*W + j the logical element index and -0.0 canonicalised to +0.0
    (signed zeros never affect a decision).  Test-side
    definition; the CUDA debug kernel implements the same formula independently."""
    T = np.asarray(T, dtype=np.float64)
    rows, W = T.shape
    total = np.uint64(0)
    with np.errstate(over="ignore"):
        for r0 in range(0, rows, chunk_rows):
            blk = T[r0:r0 + chunk_rows]
            bits = np.ascontiguousarray(blk).view(np.uint64).copy()
            bits[bits == np.uint64(0x8000000000000000)] = np.uint64(0)
            e = (np.arange(r0 * W, (r0 + blk.shape[0]) * W, dtype=np.uint64)).reshape(blk.shape)
            h = _mix64(bits ^ (e * _H_GOLDEN + _H_SALT))
            total = total + h.sum(dtype=np.uint64)
    return int(total)
