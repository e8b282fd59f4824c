"""Full-solve golden for the largest config (SURVEY.md §8(d) "Oracle baseline" (ii)):
run the CPU oracle's row-parallel build (liboracle_omp.so — the same simplex_oracle.c
with -fopenmp on or_pivot's row loop, proven bitwise equal to the single-thread build
by tests/test_oracle_omp.py) on the dense LP (m, n, seed) in resumable chunks.

Calls only oracle/ and lpgen/; no value here ever comes from the CUDA path.

    OMP_NUM_THREADS=8 python scripts/make_golden_long.py M N SEED [--ckpt DIR]
        [--chunk 1024] [--milestones 4096,16384,65536] [--ckpt-every 8192]

Outputs (tests/golden/):
  dense_<m>x<n>_s<seed>_p<K>.npz/.json  prefix goldens at each milestone K (same
                                        format as scripts/make_golden.py prefix runs)
  dense_<m>x<n>_s<seed>.npz/.json       the full solve (status, pivots, objective,
                                        x, y, whole trace, row 0, rhs, basis, hash)
  dense_<m>x<n>_s<seed>_progress.json   pivots done so far (updated every chunk)
The checkpoint DIR (default /tmp/golden_ckpt_<m>x<n>_s<seed>) holds the tableau, basis,
counter and trace so an interrupted run resumes the identical pivot sequence.
"""
import argparse
import hashlib
import json
import os
import sys
import time

import numpy as np

ROOT = os.path.join(os.path.dirname(os.path.abspath(__file__)), "..")
sys.path.insert(0, ROOT)
import lpgen  # noqa: E402
import oracle  # noqa: E402

GOLDEN = os.environ.get("GOLDEN_OUT") or os.path.join(ROOT, "tests", "golden")   # GOLDEN_OUT: e.g. gpurun_out/golden
os.makedirs(GOLDEN, exist_ok=True)


def save_golden(tag, m, n, seed, prefix, status, pivots, T, basis, tk, tr, secs, threads):
    x, y, obj = oracle.extract(T, basis, n)
    nz = np.nonzero(x)[0]
    h = oracle.tableau_hash(T)
    trace = np.stack([tk, tr], 1).astype("<i4")
    out = dict(m=m, n=n, seed=seed, prefix=prefix, status=status, pivots=pivots, objective=obj,
               trace_k=tk, trace_r=tr, x_idx=nz.astype(np.int64), x_val=x[nz], y=y,
               row0=T[0].copy(), rhs=T[:, -1].copy(), basis=basis.copy(),
               tableau_hash=np.uint64(h), oracle_seconds=secs)
    path = os.path.join(GOLDEN, tag + ".npz")
    np.savez_compressed(path + ".tmp.npz", **out)
    os.replace(path + ".tmp.npz", path)
    meta = dict(m=m, n=n, seed=seed, prefix=prefix, rule="dantzig", status=oracle.STATUS_NAME[status],
                pivots=pivots, objective=obj, objective_hex=float(obj).hex(),
                trace_sha256_16=hashlib.sha256(trace.tobytes()).hexdigest()[:16],
                first5=[list(map(int, p)) for p in trace[:5]],
                last=[list(map(int, p)) for p in trace[-1:]], nnz_x=int(nz.size),
                tableau_hash=hex(h), oracle_seconds=secs, oracle_threads=threads,
                source="scripts/make_golden_long.py -> oracle/liboracle_omp.so "
                       "(row-parallel build of simplex_oracle.c; CPU oracle only)")
    with open(path[:-4] + ".json", "w") as f:
        json.dump(meta, f, indent=1)
    print(json.dumps({k: meta[k] for k in ("prefix", "status", "pivots", "objective_hex",
                                            "trace_sha256_16", "tableau_hash")}), flush=True)


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("m", type=int)
    ap.add_argument("n", type=int)
    ap.add_argument("seed", type=int)
    ap.add_argument("--ckpt", default=None)
    ap.add_argument("--chunk", type=int, default=512)
    ap.add_argument("--milestones", default="4096,16384,65536")
    ap.add_argument("--ckpt-every", type=int, default=8192, help="0: never checkpoint")
    ap.add_argument("--max-seconds", type=float, default=0.0,
                    help="> 0: checkpoint and exit (code 3) once this much wall time has passed, so a run "
                         "can be split over several time-limited sessions that share the checkpoint dir")
    a = ap.parse_args()
    m, n, seed = a.m, a.n, a.seed
    threads = int(os.environ.get("OMP_NUM_THREADS", os.cpu_count()))
    ck = a.ckpt or f"/tmp/golden_ckpt_{m}x{n}_s{seed}"
    os.makedirs(ck, exist_ok=True)
    tag = f"dense_{m}x{n}_s{seed}"
    milestones = sorted(int(v) for v in a.milestones.split(",") if v)
    state = os.path.join(ck, "state.json")
    if os.path.exists(state):
        st = json.load(open(state))
        T = np.fromfile(os.path.join(ck, "T.f64"), dtype=np.float64).reshape(m + 1, n + m + 1)
        basis = np.load(os.path.join(ck, "basis.npy"))
        tk = list(np.load(os.path.join(ck, "trace_k.npy")))
        tr = list(np.load(os.path.join(ck, "trace_r.npy")))
        it, secs = st["it"], st["secs"]
        print(f"resumed at pivot {it}", flush=True)
    else:
        A, b, c = lpgen.dense_lp(m, n, seed)
        T, basis = oracle.build_tableau(A, b, c)
        del A
        tk, tr, it, secs = [], [], 0, 0.0
    last_ck = it
    status = oracle.RUNNING
    wall0 = time.time()

    def checkpoint():
        T.tofile(os.path.join(ck, "T.f64.tmp"))
        os.replace(os.path.join(ck, "T.f64.tmp"), os.path.join(ck, "T.f64"))
        np.save(os.path.join(ck, "basis.npy"), basis)
        np.save(os.path.join(ck, "trace_k.npy"), np.array(tk, np.int32))
        np.save(os.path.join(ck, "trace_r.npy"), np.array(tr, np.int32))
        json.dump(dict(it=it, secs=secs), open(state + ".tmp", "w"))
        os.replace(state + ".tmp", state)
        print(f"checkpoint at pivot {it}, {secs:.0f} s", flush=True)

    while status == oracle.RUNNING:
        if a.max_seconds > 0 and time.time() - wall0 > a.max_seconds:
            checkpoint()
            print(f"paused at pivot {it} after {time.time() - wall0:.0f} s of this session", flush=True)
            sys.exit(3)
        t0 = time.perf_counter()
        stop = min([it + a.chunk] + [ms for ms in milestones if ms > it])
        status, it, k, r = oracle.iterate(T, basis, it, stop_at=stop, parallel=True)
        secs += time.perf_counter() - t0
        tk.extend(k.tolist())
        tr.extend(r.tolist())
        with open(os.path.join(GOLDEN, tag + "_progress.json"), "w") as f:
            json.dump(dict(pivots_done=it, status=oracle.STATUS_NAME[status], oracle_seconds=secs,
                           s_per_pivot=secs / max(it, 1), threads=threads), f)
        ref = os.path.join(ROOT, "tests", "golden", f"{tag}_p{it}.npz")
        if status == oracle.RUNNING and os.path.exists(ref):
            # an existing committed prefix golden (an earlier oracle run): must agree bit for bit
            g = np.load(ref)
            same = (np.array_equal(np.array(tk, np.int32), g["trace_k"])
                    and np.array_equal(np.array(tr, np.int32), g["trace_r"])
                    and oracle.tableau_hash(T) == int(g["tableau_hash"]))
            print(f"check vs committed prefix golden p{it}: {'identical' if same else 'DIFFERENT'}",
                  flush=True)
            if not same:
                sys.exit(1)
        for ms in milestones:
            if it == ms and status == oracle.RUNNING:
                save_golden(f"{tag}_p{ms}", m, n, seed, ms, status, it, T, basis,
                            np.array(tk, np.int32), np.array(tr, np.int32), secs, threads)
        if status == oracle.RUNNING and a.ckpt_every > 0 and it - last_ck >= a.ckpt_every:
            checkpoint()
            last_ck = it
    save_golden(tag, m, n, seed, -1, status, it, T, basis, np.array(tk, np.int32),
                np.array(tr, np.int32), secs, threads)


if __name__ == "__main__":
    main()
