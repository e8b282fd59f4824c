"""One small solve per library path, for compute-sanitizer (memcheck / racecheck / synccheck /
initcheck).  Each case runs a bounded number of pivots and checks the trace against the CPU
oracle's prefix run, so a sanitizer run also proves the kernels still compute the right thing.

    compute-sanitizer --tool racecheck python scripts/sanitize_cases.py CASE [M N PIVOTS]

CASE: small (k_solve_small), pass1 (k_select/k_update), look16 (pipelined k_lookahead +
k_update_s), look16serial, pair32, slabs3 (virtual slabs, one pivot per pass), mblock2 (virtual
slabs, k_mblock peer-memory protocol, exchange=2), mlook3 (exchange=3: k_mlook per pivot),
phase1 (Phase I + device drive-out), all."""
import os
import sys

import numpy as np

sys.path.insert(0, os.path.join(os.path.dirname(os.path.abspath(__file__)), ".."))
import lpgen  # noqa: E402
import oracle  # noqa: E402
import paper_2211_10979_b200 as sx  # noqa: E402
from lpgen import fixtures  # noqa: E402

CASES = {"small": dict(), "pass1": dict(lookahead=1), "look16": dict(lookahead=16),
         "look16serial": dict(lookahead=16, overlap=False), "pair32": dict(lookahead=32),
         "slabs3": dict(lookahead=1, virtual_ranks=3), "mblock2": dict(lookahead=16, virtual_ranks=2, exchange=2),
         "mlook3": dict(lookahead=16, virtual_ranks=3, exchange=3), "phase1": dict(lookahead=16)}


def run(case, m, n, piv):
    kw = CASES[case]
    if case == "phase1":
        A, b, c = fixtures.with_lower_bounds(m, n, 3, frac=0.1, eq=4)
        o = oracle.solve_2phase(A, b, c)
        with sx.Simplex(A, b, c, **kw) as s:
            st = s.solve()
            k, r = s.trace()
        ok = st == o.status and np.array_equal(k, o.trace_k) and np.array_equal(r, o.trace_r)
    else:
        A, b, c = lpgen.dense_lp(m, n, 1)
        o = oracle.solve(A, b, c, stop_after=piv, keep_tableau=True)
        with sx.Simplex(A, b, c, **kw) as s:
            if case == "small":
                assert s.stats().path == 1, "tableau too large for the one-CTA path"
            s.iterate(piv)
            k, r = s.trace()
            T, _ = s.tableau()
        ok = np.array_equal(k, o.trace_k) and np.array_equal(r, o.trace_r) and np.array_equal(T, o.T)
    print(f"sanitize case {case} {m}x{n}: {'OK' if ok else 'MISMATCH'} ({len(k)} pivots)", flush=True)
    return ok


if __name__ == "__main__":
    case = sys.argv[1]
    m, n = int(sys.argv[2]) if len(sys.argv) > 2 else 64, int(sys.argv[3]) if len(sys.argv) > 3 else 64
    piv = int(sys.argv[4]) if len(sys.argv) > 4 else 48
    import torch
    torch.cuda.set_device(0)
    ok = all(run(cs, m, n, piv) for cs in (CASES if case == "all" else [case]))
    sys.exit(0 if ok else 1)
