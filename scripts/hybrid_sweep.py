"""θ sweep of the hybrid CPU lane (the shape of PAPER.md Tables VI-VIII:
improvement of the CPU+GPU split over the GPU alone as a function of the CPU's column share θ).

    python scripts/hybrid_sweep.py 8000x8000 [pivots] [thetas]  -> JSON line

Every θ runs the same first `pivots` pivots of the seed-1 LP with one pivot per pass (the
hybrid lane exchanges candidates every pivot), CUDA events around simplex_iterate; θ = 0 is the
GPU alone on the same path.  The library default (rank-16 look-ahead, pipelined) is reported for
context.  The first pivots of every θ are checked against the θ = 0 trace (bitwise parity)."""
import json
import os
import sys
import time

sys.path.insert(0, os.path.join(os.path.dirname(os.path.abspath(__file__)), ".."))
import numpy as np  # noqa: E402
import torch  # noqa: E402

import lpgen  # noqa: E402
import paper_2211_10979_b200 as sx  # noqa: E402

sz = sys.argv[1] if len(sys.argv) > 1 else "8000x8000"
piv = int(sys.argv[2]) if len(sys.argv) > 2 else 400
thetas = [float(v) for v in (sys.argv[3] if len(sys.argv) > 3 else
                             "0,0.0005,0.001,0.0025,0.005,0.01,0.02,0.05,0.1").split(",")]
m, n = map(int, sz.split("x"))
torch.cuda.set_device(0)
A, b, c = lpgen.dense_lp(m, n, 1)


def run(**kw):
    with sx.Simplex(A, b, c, **kw) as s:
        s.iterate(16)                             # warm-up (graphs, host threads, clocks)
        torch.cuda.synchronize()
        st0 = s.stats()
        t0 = time.perf_counter()
        done, _ = s.iterate(piv)
        torch.cuda.synchronize()
        dt = time.perf_counter() - t0
        st = s.stats()
        k, _ = s.trace()
    return done / dt, st, st0, k


out = {"workload": f"{m}x{n} seed 1", "pivots": piv, "host_cores": os.cpu_count(), "rows": []}
ref_k = None
for th in thetas:
    kw = dict(lookahead=1) if th == 0 else dict(host_share=th)
    pps, st, st0, k = run(**kw)
    if ref_k is None:
        ref_k = k
    same = bool(np.array_equal(k, ref_k[:len(k)]))
    done = st.pivots - st0.pivots
    row = {"theta": th, "host_cols": int(st.host_cols), "pivots_per_s": pps,
           "host_update_us_per_pivot": 1e3 * (st.host_ms_total - st0.host_ms_total) / max(1, done),
           "host_wait_us_per_pivot": 1e3 * (st.host_wait_ms_total - st0.host_wait_ms_total) / max(1, done),
           "trace_equals_gpu_only": same}
    out["rows"].append(row)
    print(json.dumps(row), flush=True)
base = out["rows"][0]["pivots_per_s"]
for row in out["rows"]:
    row["improvement_pct"] = 100.0 * (row["pivots_per_s"] / base - 1.0)
pps, _, _, _ = run()
out["library_default_pivots_per_s"] = pps
out["note"] = ("theta = 0: GPU alone, one pivot per pass (k_select + k_update); theta > 0: the last round(theta(n+m)) "
               "columns on the host cores (OpenMP), one host<->GPU exchange per pivot; library default: rank-16 "
               "look-ahead pipelined, GPU only")
print(json.dumps(out), flush=True)
