"""Write tests/golden/dense_<m>x<n>_s<seed>[_p<K>].npz by running the CPU oracle.

Calls only oracle/ (the CPU reference) and lpgen/ (the shared seeded input
generator).  No value here ever comes from the CUDA path.  Usage:
    python scripts/make_golden.py M N SEED [PREFIX_PIVOTS] [bland]
A prefix run stops after PREFIX_PIVOTS pivots (status RUNNING) and also stores
row 0, the rhs column and the whole-tableau hash (oracle.tableau_hash)."""
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
    A, b, c = lpgen.dense_lp(m, n, seed)
    t0 = time.perf_counter()
    res = oracle.solve(A, b, c, stop_after=prefix, keep_tableau=True,
                       rule=oracle.BLAND if rule == "bland" else oracle.DANTZIG)
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
    path = os.path.join(os.path.dirname(os.path.abspath(__file__)), "..", "tests", "golden", tag + ".npz")
    np.savez_compressed(path, **out)
    meta = dict(m=m, n=n, seed=seed, prefix=prefix, rule=rule, status=oracle.STATUS_NAME[res.status],
                pivots=res.pivots, objective=res.objective, objective_hex=float(res.objective).hex(),
                trace_sha256_16=hashlib.sha256(tr.tobytes()).hexdigest()[:16],
                first5=res.trace()[:5], last=res.trace()[-1:] if res.pivots else [],
                nnz_x=int(nz.size), tableau_hash=hex(oracle.tableau_hash(T)),
                oracle_seconds_single_thread=dt,
                source="scripts/make_golden.py -> oracle/simplex_oracle.c (CPU oracle only)")
    with open(path[:-4] + ".json", "w") as f:
        json.dump(meta, f, indent=1)
    print(json.dumps(meta))


if __name__ == "__main__":
    main()
