"""Write tests/golden/dense_<m>x<n>_s<seed>[_p<K>].npz by running the CPU oracle.

Calls only oracle/ (the CPU reference) and lpgen/ (the shared seeded input
generator).  No value here ever comes from the CUDA path.  Usage:
    python scripts/make_golden.py M N SEED [PREFIX_PIVOTS] [bland]
A prefix run stops after PREFIX_PIVOTS pivots (status RUNNING) and also stores
row 0, the rhs column and the whole-tableau hash (oracle.tableau_hash).
Environment: GOLDEN_PARALLEL=1 runs the row-parallel oracle build (liboracle_omp.so,
bitwise identical to the single-thread build, tests/test_oracle_omp.py) with
OMP_NUM_THREADS threads; GOLDEN_OUT=DIR writes the files there instead of tests/golden."""
import hashlib
import json
import os
import sys
import time

import numpy as np

sys.path.insert(0, os.path.join(os.path.dirname(os.path.abspath(__file__)), ".."))
import lpgen  # noqa: E402
import oracle  # noqa: E402


def main():
    m, n, seed = int(sys.argv[1]), int(sys.argv[2]), int(sys.argv[3])
    prefix = int(sys.argv[4]) if len(sys.argv) > 4 else -1
    rule = sys.argv[5] if len(sys.argv) > 5 else "dantzig"
    parallel = os.environ.get("GOLDEN_PARALLEL", "0") == "1"
    A, b, c = lpgen.dense_lp(m, n, seed)
    t0 = time.perf_counter()
    res = oracle.solve(A, b, c, stop_after=prefix, keep_tableau=True,
                       rule=oracle.BLAND if rule == "bland" else oracle.DANTZIG, parallel=parallel)
    dt = time.perf_counter() - t0
    T = res.T
    nz = np.nonzero(res.x)[0]
    tr = np.stack([res.trace_k, res.trace_r], 1).astype("<i4")
    out = dict(m=m, n=n, seed=seed, prefix=prefix, status=res.status, pivots=res.pivots,
               objective=res.objective, trace_k=res.trace_k, trace_r=res.trace_r,
               x_idx=nz.astype(np.int64), x_val=res.x[nz], y=res.y,
               row0=T[0].copy(), rhs=T[:, -1].copy(), basis=res.basis,
               tableau_hash=np.uint64(oracle.tableau_hash(T)), oracle_seconds=dt)
    tag = f"dense_{m}x{n}_s{seed}" + (f"_p{prefix}" if prefix >= 0 else "") + (f"_{rule}" if rule != "dantzig" else "")
    out_dir = os.environ.get("GOLDEN_OUT") or os.path.join(os.path.dirname(os.path.abspath(__file__)), "..",
                                                           "tests", "golden")
    os.makedirs(out_dir, exist_ok=True)
    path = os.path.join(out_dir, tag + ".npz")
    np.savez_compressed(path, **out)
    meta = dict(m=m, n=n, seed=seed, prefix=prefix, rule=rule, status=oracle.STATUS_NAME[res.status],
                pivots=res.pivots, objective=res.objective, objective_hex=float(res.objective).hex(),
                trace_sha256_16=hashlib.sha256(tr.tobytes()).hexdigest()[:16],
                first5=res.trace()[:5], last=res.trace()[-1:] if res.pivots else [],
                nnz_x=int(nz.size), tableau_hash=hex(oracle.tableau_hash(T)),
                oracle_seconds=dt,
                oracle_threads=int(os.environ.get("OMP_NUM_THREADS", os.cpu_count())) if parallel else 1,
                source="scripts/make_golden.py -> oracle/" + ("liboracle_omp.so (row-parallel build of "
                       "simplex_oracle.c)" if parallel else "simplex_oracle.c") + " (CPU oracle only)")
    with open(path[:-4] + ".json", "w") as f:
        json.dump(meta, f, indent=1)
    print(json.dumps(meta))


if __name__ == "__main__":
    main()
