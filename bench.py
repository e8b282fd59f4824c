"""bench.py — time the dense-tableau simplex hot path on B200 (libsimplex) and print ONE JSON line.

    python bench.py [--gpus N] [--steps K] [--warmup W] [--workload 8000x8000] [--seed 1]
    python bench.py --impl reference ...          # the CPU oracle arm (rank 0 only)
    torchrun --nproc-per-node N bench.py --gpus N ...

A "step" is one full pass of the hot path over one
synthetic LP: build Table I from the device-resident (A, b, c) -> pivot loop to
termination (pricing, ratio test, fused row-scale + rank-1 update, all on the
device) -> extract x, y, objective.  value = pivots of all timed solves / device
time (CUDA events on the launching stream, barrier + synchronize on both sides,
max over ranks).  The default workload is the BASELINE.json config quoted at
1/2/4/8 B200 that fits one GPU with a full solve in seconds: 8000x8000, seed 1.
With N > 1 the same LP is column-partitioned over the N ranks (strong scaling).
"""
from __future__ import annotations

import argparse
import json
import os
import statistics
import subprocess
import sys
import time

import numpy as np

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

PAPER_CONTEXT = ("paper (PAPER.md Tables III-V, 25000x25000, Turing): 0.2044 s/pivot RTX 2080Ti, "
                 "0.1732 s/pivot Titan RTX, 0.1157 s/pivot both; 0.4773 s/pivot 32-core Xeon")


def workload_name(m, n, seed, rule="dantzig"):
    """config.workload — the SAME string on both arms (the driver compares them)."""
    return (f"dense random LP m={m} n={n} FP64 seed {seed}, slack basis, "
            + ("Dantzig + lowest-index ties" if rule == "dantzig" else "Bland's rule"))


def host_info():
    """CPU model, core count and this process's allowed cores (lscpu-equivalent, no subprocess)."""
    model = "unknown"
    try:
        for line in open("/proc/cpuinfo"):
            if line.startswith("model name"):
                model = line.split(":", 1)[1].strip()
                break
    except OSError:
        pass
    mem_gb = None
    try:
        for line in open("/proc/meminfo"):
            if line.startswith("MemTotal"):
                mem_gb = round(int(line.split()[1]) / 2**20, 1)
                break
    except OSError:
        pass
    return {"cpu_model": model, "nproc": os.cpu_count(), "mem_total_gb": mem_gb,
            "allowed_cores": len(os.sched_getaffinity(0))}


class pinned_to_one_core:
    """taskset-equivalent: pin the calling thread to one allowed core for the oracle timing
    (SURVEY.md §8(d) "Pin the oracle with taskset to one core"), restore afterwards."""

    def __enter__(self):
        self.host = host_info()                     # before pinning: the box's cores
        self.prev = os.sched_getaffinity(0)
        self.core = sorted(self.prev)[0]
        os.sched_setaffinity(0, {self.core})
        return self

    def __exit__(self, *exc):
        os.sched_setaffinity(0, self.prev)


def parse():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=3)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--workload", default="8000x8000")
    ap.add_argument("--seed", type=int, default=1)
    ap.add_argument("--impl", default="libsimplex", choices=["libsimplex", "reference"])
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--cpu-sample-seconds", type=float, default=15.0)
    ap.add_argument("--roofline-pivots", type=int, default=4000)
    ap.add_argument("--lookahead", type=int, default=0,
                    help="pivots per tableau pass (0: library default = 16 on one column part, 1 with "
                         "N > 1; 1: one pass per pivot; 2..16: rank-s look-ahead)")
    ap.add_argument("--no-overlap", action="store_true",
                    help="rank-s look-ahead without the software pipeline (select, then pass)")
    ap.add_argument("--pivot-rule", default="dantzig", choices=["dantzig", "bland"],
                    help="entering/leaving rule (bland = SURVEY.md §8(f) NEXT #3)")
    ap.add_argument("--single-pass-pivots", type=int, default=1000,
                    help="pivots of the one-pivot-per-pass k_update roofline window (0: skip)")
    ap.add_argument("--exchange", type=int, default=0,
                    help="simplex_options.exchange for N > 1 (0: peer memory when reachable, else NCCL; "
                         "1: NCCL); a peer-memory failure at N > 1 falls back to 1 and says so")
    ap.add_argument("--largest", default="20000x40000",
                    help="the north_star's largest tableau: a sub-record of simplex_iterate windows "
                         "('none' to skip; skipped when it is the main workload)")
    ap.add_argument("--largest-window", type=int, default=1600)
    ap.add_argument("--largest-parity-max", type=int, default=20000,
                    help="largest prefix golden (pivots) the largest leg checks bit for bit")
    return ap.parse_args()


def dist_env():
    return int(os.environ.get("RANK", "0")), int(os.environ.get("WORLD_SIZE", "1")), \
        int(os.environ.get("LOCAL_RANK", "0"))


def solver_look(lookahead, world):
    """Pivots per tableau pass the library uses (mirrors simplex_options.lookahead = 0)."""
    if lookahead > 0:
        return lookahead
    return 16


def reduce_max(v, world, dev):
    """Max of a per-rank scalar over all ranks (multi-GPU times are max over ranks)."""
    if world <= 1:
        return v
    import torch
    t = torch.tensor([float(v)], dtype=torch.float64, device=dev)
    torch.distributed.all_reduce(t, op=torch.distributed.ReduceOp.MAX)
    return float(t.item())


def reduce_sum(v, world, dev):
    if world <= 1:
        return v
    import torch
    t = torch.tensor([float(v)], dtype=torch.float64, device=dev)
    torch.distributed.all_reduce(t)
    return float(t.item())


def load_peaks():
    p = os.path.join(ROOT, "MEASURED_PEAKS.json")
    if os.path.exists(p):
        d = json.load(open(p))
        return float(d["hbm_gbs"]), "measured (MEASURED_PEAKS.json hbm_gbs, torch copy read+write)"
    return 6650.0, "fallback (B200_PROFILING.md: 6.65 TB/s)"


def ncu_entry(workload, nranks, look=1):
    p = os.path.join(ROOT, "profiles", "ncu_update_traffic.json")
    if not os.path.exists(p):
        return None
    d = json.load(open(p))
    return d.get(f"{workload}/s{look}/p{nranks}" if look > 1 else f"{workload}/p{nranks}")


def ncu_duration(workload, nranks, look=1):
    e = ncu_entry(workload, nranks, look)
    return e.get("ncu_duration_us") if e else None


def ncu_l2(workload, nranks, look=1):
    e = ncu_entry(workload, nranks, look)
    return e.get("l2_bytes_per_launch") if e else None


def ncu_traffic(workload, nranks, look=1):
    """dram read+write bytes per pass launch (k_update, or k_update_s for look > 1) from a
    committed ncu --set full capture."""
    p = os.path.join(ROOT, "profiles", "ncu_update_traffic.json")
    if not os.path.exists(p):
        return None
    d = json.load(open(p))
    e = d.get(f"{workload}/s{look}/p{nranks}" if look > 1 else f"{workload}/p{nranks}")
    return e.get("dram_bytes_per_launch") if e else None


class ClockSampler:
    """nvidia-smi clocks + throttle reasons DURING the timed region (B200_PROFILING.md)."""
    Q = ("index,clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.active,"
         "clocks_event_reasons.hw_slowdown,clocks_event_reasons.hw_thermal_slowdown,"
         "clocks_event_reasons.sw_thermal_slowdown,clocks_event_reasons.sw_power_cap")

    def __init__(self):
        self.proc = None
        self.path = f"/tmp/bench_clocks_{os.getpid()}.csv"

    def start(self):
        try:
            self.f = open(self.path, "w")
            self.proc = subprocess.Popen(["nvidia-smi", f"--query-gpu={self.Q}", "--format=csv,noheader,nounits",
                                          "-lms", "200"], stdout=self.f, stderr=subprocess.DEVNULL)
        except Exception:
            self.proc = None

    def stop(self):
        if not self.proc:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["nvidia-smi unavailable"]}
        self.proc.terminate()
        self.proc.wait()
        self.f.close()
        if os.path.getsize(self.path) == 0:          # a timed region shorter than one 200 ms period
            try:
                out = subprocess.run(["nvidia-smi", f"--query-gpu={self.Q}", "--format=csv,noheader,nounits"],
                                     capture_output=True, text=True, timeout=20).stdout
                with open(self.path, "w") as f:
                    f.write(out)
            except Exception:
                pass
        sm, smax, reasons = [], [], set()
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        for line in open(self.path):
            p = [x.strip() for x in line.split(",")]
            if len(p) < 9:
                continue
            try:
                sm.append(float(p[1]))
                smax.append(float(p[2]))
            except ValueError:
                continue
            for nm, v in zip(names, p[5:9]):
                if v.lower().startswith("active"):
                    reasons.add(nm)
        os.unlink(self.path)
        return {"sm_mhz": statistics.median(sm) if sm else None, "sm_max_mhz": max(smax) if smax else None,
                "reasons": sorted(reasons), "samples": len(sm)}


def cpu_baseline(A, b, c, seconds):
    """The oracle (oracle/, single-threaded C) as it stands, on a bounded sample of the SAME
    workload: the first P pivots, P sized for ~`seconds` of CPU work.  pivots/s =
    P / (t(P pivots) - t(0 pivots)) so the tableau build is not counted."""
    import oracle
    m, n = A.shape
    oracle.lib()                                      # load (and if needed build) it untimed
    with pinned_to_one_core() as pin:
        oracle.solve(A, b, c, stop_after=2)               # warm
        t0 = time.perf_counter()
        oracle.solve(A, b, c, stop_after=2)
        t_two = time.perf_counter() - t0
        # a whole solve is at most 20(m+n) pivots; time complete solves only when even that bound
        # stays well inside the budget (64x64: ~1 ms per solve), else a prefix of the solve
        full = oracle.solve(A, b, c) if t_two * 10 * (m + n) < seconds else None
        t_full = time.perf_counter() - t0 - t_two
        if full is not None and t_full < seconds / 10:
            # a whole solve is short (64x64: ~1 ms): time R complete solves, build included
            R = int(max(1, seconds / 2 / max(t_full, 1e-6)))
            t0 = time.perf_counter()
            for _ in range(R):
                oracle.solve(A, b, c)
            dt = time.perf_counter() - t0
            return {"value": R * full.pivots / dt, "unit": "pivots/s", "cores": 1, "kind": "oracle",
                    "sample": f"{R} complete solves of the {m}x{n} seed LP ({full.pivots} pivots each, tableau "
                              f"build included; oracle/simplex_oracle.c, 1 thread pinned to core {pin.core}), "
                              f"{dt:.1f} s", "time_to_solve_us": 1e6 * dt / R, "host": pin.host}
        t0 = time.perf_counter()
        oracle.solve(A, b, c, stop_after=0)
        t_build = time.perf_counter() - t0
        t0 = time.perf_counter()
        oracle.solve(A, b, c, stop_after=2)
        per = max((time.perf_counter() - t0 - t_build) / 2, 1e-6)
        P = int(max(2, min(100000, seconds / per)))
        t0 = time.perf_counter()
        r = oracle.solve(A, b, c, stop_after=P)
        dt = time.perf_counter() - t0 - t_build
    return {"value": r.pivots / dt, "unit": "pivots/s", "cores": 1, "kind": "oracle",
            "sample": f"first {r.pivots} pivots of the {m}x{n} seed solve (oracle/simplex_oracle.c, 1 thread "
                      f"pinned to core {pin.core}, tableau build excluded), {dt:.1f} s",
            "host": pin.host}


def run_reference(args):
    """The reference arm: the CPU oracle (oracle/, single-threaded C) as it stands, on this
    arm's workload.  The tableau is built once (untimed); each step is a bounded sample of
    the same solve — the next P pivots through the oracle's own step functions (Step 1
    or_price, Step 2 or_ratio, Step 3 or_pivot), P sized for ~3 s of CPU work."""
    rank, world, _ = dist_env()
    if rank != 0:
        return 0
    m, n = map(int, args.workload.split("x"))
    import lpgen
    import oracle
    A, b, c = lpgen.dense_lp(m, n, args.seed)
    T, basis = oracle.build_tableau(A, b, c)
    done = [0]

    bland = args.pivot_rule == "bland"

    def pivots(P):
        for _ in range(P):
            k = oracle.price_bland(T[0, :-1]) if bland else oracle.price(T[0, :-1])[0]
            if k < 0:
                return
            r = oracle.ratio_bland(T, k, basis)[0] if bland else oracle.ratio(T, k)[0]
            if r < 0:
                return
            oracle.pivot(T, r, k)
            basis[r - 1] = k
            done[0] += 1

    with pinned_to_one_core() as pin:
        t0 = time.perf_counter()
        pivots(1)
        per = max(time.perf_counter() - t0, 1e-6)
        P = int(max(1, min(100000, 3.0 / per)))
        for _ in range(args.warmup):
            pivots(P)
        d0 = done[0]
        t0 = time.perf_counter()
        for _ in range(args.steps):
            pivots(P)
        dt = time.perf_counter() - t0
    v = (done[0] - d0) / dt
    line = {"metric": "pivots/s", "value": v, "unit": "pivots/s", "impl": "reference", "n_gpus": args.gpus,
            "steps": args.steps, "warmup": args.warmup, "ms_per_step": 1000 * dt / args.steps,
            "higher_is_better": True, "scaling": "strong", "vs_baseline": None, "dtype": "f64",
            "data": "synthetic (lpgen SplitMix64 dense LP: A,c~U[1,10), b~U[n,2n))",
            "config": {"workload": workload_name(m, n, args.seed, args.pivot_rule), "m": m, "n": n},
            "cpu_baseline": {"value": v, "unit": "pivots/s", "cores": 1, "kind": "oracle",
                             "sample": f"each step: the next {P} pivots of the {m}x{n} solve through the "
                                       f"oracle's step functions (tableau built once, untimed; 1 thread pinned "
                                       f"to core {pin.core})", "host": pin.host},
            "e2e": {"value": v, "unit": "pivots/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0}}
    print(json.dumps(line), flush=True)
    return 0


def golden_prefixes(m, n, seed):
    """{P: path} of the oracle-written prefix goldens tests/golden/dense_<m>x<n>_s<seed>_p<P>.npz."""
    import glob
    import re
    out = {}
    for p in glob.glob(os.path.join(ROOT, "tests", "golden", f"dense_{m}x{n}_s{seed}_p*.npz")):
        mt = re.search(r"_p(\d+)\.npz$", p)
        if mt:
            out[int(mt.group(1))] = p
    return out


def check_prefix(solver, g, P):
    """The solver stands at exactly P pivots: its trace, objective, y and whole-tableau digest
    against the oracle's P-pivot prefix golden (bit for bit)."""
    k, r = solver.trace()
    _, y, obj, piv, _ = solver.solution()
    h = solver.tableau_hash()
    return bool(piv == P and np.array_equal(k[:P], g["trace_k"]) and np.array_equal(r[:P], g["trace_r"])
                and obj == float(g["objective"]) and np.array_equal(y, g["y"]) and h == int(g["tableau_hash"]))


def measure_tcoll(m, world, dev, iters=200):
    """t_coll(P) (SURVEY.md §8(d) "Multi-GPU roofline"): the per-pivot exchange of the
    column-partitioned method — every rank contributes its candidate column (m+3 doubles: the
    column, its index and value) and receives every rank's — as an exchange-only loop of NCCL
    allgathers, CUDA events on the launching stream, max over ranks.  (The library's default
    multi-rank exchange is the same data moved with peer-memory stores inside k_mblock.)"""
    import torch
    import torch.distributed as dist
    x = torch.zeros(m + 3, dtype=torch.float64, device=dev)
    out = torch.empty(world * (m + 3), dtype=torch.float64, device=dev)
    for _ in range(20):
        dist.all_gather_into_tensor(out, x)
    dist.barrier()
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(iters):
        dist.all_gather_into_tensor(out, x)
    e1.record()
    torch.cuda.synchronize()
    us = e0.elapsed_time(e1) * 1e3 / iters
    return reduce_max(us, world, dev)


def gather_list(v, world):
    if world <= 1:
        return [v]
    import torch.distributed as dist
    out = [None] * world
    dist.all_gather_object(out, v)
    return out


def largest_leg(args, world, group, dev, peak, barrier, exchange=0):
    """The north_star's largest tableau (20000x40000 by default) as a sub-record of every line:
    pivots/s as the median of 3 simplex_iterate windows ("median of 3 windows
    ... driven by simplex_iterate"), the device-timed pass roofline, and the first pivots checked
    bit for bit against the largest oracle prefix golden available (trace, objective, y, digest)."""
    import torch
    import lpgen
    import paper_2211_10979_b200 as sx
    m, n = map(int, args.largest.split("x"))
    t0 = time.perf_counter()
    A, b, c = lpgen.dense_lp(m, n, args.seed)
    t_gen = time.perf_counter() - t0
    t0 = time.perf_counter()
    s = sx.Simplex(A, b, c, group=group, time_kernels=True, exchange=exchange)
    del A
    barrier()
    t_create = time.perf_counter() - t0
    st = s.stats()
    # parity first: the largest oracle prefix golden available (<= largest_parity_max pivots)
    parity = {"checked": False}
    pre = {P: p for P, p in golden_prefixes(m, n, args.seed).items() if P <= args.largest_parity_max}
    if pre:
        P = max(pre)
        s.iterate(P)
        ok = check_prefix(s, np.load(pre[P]), P)
        parity = {"checked": True, "vs": os.path.relpath(pre[P], ROOT), "pivots": P,
                  "bitwise_trace_objective_y_tableau_digest": ok}
        if not ok:
            raise SystemExit(f"PARITY FAILURE (largest leg) vs {pre[P]}")
    s.iterate(64)                                          # warm-up (graphs built, clocks up)
    barrier()
    first = s.stats().pivots
    wins, passes = [], []
    for _ in range(3):
        a0 = s.stats()
        barrier()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        done, status = s.iterate(args.largest_window)
        e1.record()
        barrier()
        ms = reduce_max(e0.elapsed_time(e1), world, dev)
        a1 = s.stats()
        wins.append(done / (ms / 1e3))
        if a1.update_launches > a0.update_launches:
            passes.append((a1.update_ms_total - a0.update_ms_total) / (a1.update_launches - a0.update_launches))
        if status != sx.RUNNING:
            break
    pass_ms = statistics.median(passes) if passes else None
    achieved = st.bytes_per_pivot / (pass_ms / 1e3) / 1e9 if pass_ms else None
    per_rank = gather_list(achieved / peak if achieved else None, world)
    s.close()
    full = os.path.join(ROOT, "tests", "golden", f"dense_{m}x{n}_s{args.seed}.json")
    return {"workload": workload_name(m, n, args.seed), "metric": "pivots/s",
            "value": statistics.median(wins), "windows_pivots_per_s": wins,
            "window_pivots": args.largest_window, "first_window_starts_at_pivot": first, "n_gpus": world,
            "how": "median of 3 simplex_iterate windows after 64 warm-up pivots; CUDA events on the "
                   "launching stream, barrier + synchronize both sides, max over ranks",
            "roofline": {"bound": "hbm", "kernel": "k_update_s (rank-16 look-ahead pass)",
                         "avg_launch_us": pass_ms * 1e3 if pass_ms else None, "achieved": achieved, "peak": peak,
                         "unit": "GB/s", "frac": achieved / peak if achieved else None,
                         "per_rank_frac": per_rank, "bytes_per_launch": st.bytes_per_pivot,
                         "traffic": ncu_traffic(args.largest, world, 16)},
            "t_roof_single_pass_us": st.bytes_per_pivot / peak / 1e3,
            "parity": parity,
            "full_solve_golden": os.path.relpath(full, ROOT) if os.path.exists(full) else None,
            "setup_s": {"generate": t_gen, "create": t_create}}


def main():
    args = parse()
    if args.impl == "reference":
        return run_reference(args)
    rank, world, local_rank = dist_env()
    import torch
    if not torch.cuda.is_available():
        raise SystemExit("bench.py needs a CUDA device (libsimplex has no CPU fallback)")
    torch.cuda.set_device(local_rank)
    group = None
    if world > 1:
        import torch.distributed as dist
        dist.init_process_group("nccl", device_id=torch.device("cuda", local_rank))
        group = dist.group.WORLD
    import lpgen
    import paper_2211_10979_b200 as sx

    m, n = map(int, args.workload.split("x"))
    A, b, c = lpgen.dense_lp(m, n, args.seed)
    dev = torch.device("cuda", local_rank)
    dA, db, dc = (torch.from_numpy(v).to(dev) for v in (A, b, c))
    dx = torch.empty(n, dtype=torch.float64, device=dev)
    dy = torch.empty(m, dtype=torch.float64, device=dev)
    torch.cuda.synchronize()

    rule = sx.BLAND if args.pivot_rule == "bland" else sx.DANTZIG
    exchange = args.exchange
    fallback = None

    def make(**kw):
        return sx.Simplex(dA, db, dc, group=group, pivot_rule=rule, exchange=exchange, **kw)

    try:
        solver = make(lookahead=args.lookahead, overlap=not args.no_overlap)
    except sx.SimplexError as e:
        if world <= 1 or exchange == 1:
            raise
        fallback = f"exchange {exchange} failed at create ({e}); NCCL exchange (1) used"
        exchange = 1
        solver = make(lookahead=args.lookahead, overlap=not args.no_overlap)
    st = solver.stats()
    small = st.path == 1                                     # one-CTA shared-memory solve (k_solve_small)
    tableau_bytes = 8 * (m + 1) * (n + m + 1)
    l2 = torch.cuda.get_device_properties(dev).L2_cache_size
    flush = None
    if st.bytes_per_pivot // 2 < 2 * l2:                      # slab fits in L2: flush between steps
        flush = torch.empty(2 * l2 // 4, dtype=torch.float32, device=dev)

    def barrier():
        if world > 1:
            torch.distributed.barrier()
        torch.cuda.synchronize()

    def one_step(reload=True):
        if reload and small:                                 # one call, one launch, one sync
            _, _, obj, piv, status = solver.solve_lp(dA, db, dc, dx, dy)
            return status, obj, piv
        if reload:
            solver.reset(dA, db, dc)
        status = solver.solve()
        _, _, obj, piv, _ = solver.solution(dx, dy)
        return status, obj, piv

    # ---- correctness gate before timing: the oracle's golden for this workload —
    # the full solve when it exists (trace + objective bit for bit), else the largest prefix
    # golden (trace, objective, y and whole-tableau digest at exactly P pivots), then the rest
    parity = {"checked": False}
    suffix = "" if args.pivot_rule == "dantzig" else f"_{args.pivot_rule}"
    gpath = os.path.join(ROOT, "tests", "golden", f"dense_{m}x{n}_s{args.seed}{suffix}.npz")
    pre = golden_prefixes(m, n, args.seed) if not suffix else {}
    if not os.path.exists(gpath) and pre:
        P = max(pre)
        try:
            solver.iterate(P)
        except sx.SimplexError as e:             # e.g. a peer-memory exchange timeout on N > 1
            if world <= 1 or exchange == 1:
                raise
            fallback = f"exchange {exchange} failed in the first solve ({e}); NCCL exchange (1) used"
            exchange = 1
            solver.close()
            solver = make(lookahead=args.lookahead, overlap=not args.no_overlap)
            solver.iterate(P)
        ok = check_prefix(solver, np.load(pre[P]), P)
        parity = {"checked": True, "vs": os.path.relpath(pre[P], ROOT), "prefix_pivots": P,
                  "bitwise_trace_objective_y_tableau_digest": ok}
        if not ok:
            raise SystemExit(f"PARITY FAILURE vs {pre[P]}")
    try:
        status, obj, piv = one_step(reload=False)
    except sx.SimplexError as e:
        if world <= 1 or exchange == 1:
            raise
        fallback = f"exchange {exchange} failed in the first solve ({e}); NCCL exchange (1) used"
        exchange = 1
        solver.close()
        solver = make(lookahead=args.lookahead, overlap=not args.no_overlap)
        status, obj, piv = one_step(reload=False)
    k, r = solver.trace()
    if os.path.exists(gpath):
        g = np.load(gpath)
        ok = (piv == int(g["pivots"]) and obj == float(g["objective"]) and np.array_equal(k, g["trace_k"])
              and np.array_equal(r, g["trace_r"]))
        parity = {"checked": True, "vs": os.path.relpath(gpath, ROOT), "bitwise_trace_and_objective": bool(ok)}
        if not ok:
            raise SystemExit(f"PARITY FAILURE vs {gpath}: pivots {piv} vs {int(g['pivots'])}")
    xh, yh = dx.cpu().numpy(), dy.cpu().numpy()
    L = np.longdouble
    gap = abs(float((c.astype(L) * xh.astype(L)).sum() - (b.astype(L) * yh.astype(L)).sum()))
    parity["duality_gap_rel"] = gap / max(1.0, abs(obj))
    parity["status"] = sx.STATUS_NAME[status]

    for _ in range(args.warmup):
        one_step()
    barrier()

    s0 = solver.stats()
    clocks = ClockSampler() if rank == 0 else None
    if clocks:
        clocks.start()
    times, pivs = [], 0
    for _ in range(args.steps):
        if flush is not None:
            flush.zero_()
        barrier()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        status, obj, piv = one_step()
        e1.record()
        barrier()
        times.append(e0.elapsed_time(e1))
        pivs += piv
    clk = clocks.stop() if clocks else None
    s1 = solver.stats()
    total_ms = sum(times)
    if world > 1:
        total_ms = reduce_max(total_ms, world, dev)
    value = pivs / (total_ms / 1e3)
    loop_ms = reduce_max(s1.loop_ms_total - s0.loop_ms_total, world, dev)

    # ---- roofline pass: the same solve with the pass timed.  The pipelined rank-s pass is timed
    # on the device (%globaltimer in the kernel: first CTA start -> last CTA end, the production
    # launch sequence); the one-pivot k_update with CUDA events around every launch (event nodes in
    # the captured graph, on the stream the kernel runs on).  Kept out of the value steps.
    prof = make(time_kernels=True, lookahead=args.lookahead, overlap=not args.no_overlap)
    barrier()
    window = min(piv, args.roofline_pivots)
    prof.iterate(window)
    barrier()
    sp = prof.stats()
    prof.close()
    upd_launches = sp.update_launches
    upd_ms = sp.update_ms_total
    avg_upd_s = upd_ms / 1e3 / max(1, upd_launches)
    achieved = st.bytes_per_pivot / avg_upd_s / 1e9
    peak, peak_src = load_peaks()
    prof_loop_ms = sp.loop_ms_total
    look = 1 if small else solver_look(args.lookahead, world)
    small_roof = None
    if small:
        # the whole solve is ONE launch of ONE CTA with the tableau in shared memory: the bound
        # is that SM's shared-memory crossbar (128 B/cycle/SM, B300_MICROARCH.md "LDS/STS",
        # at the max SM clock), which every pivot streams twice (read + write of each element)
        smhz = 1965.0
        try:
            smhz = float(json.load(open(os.path.join(ROOT, "MEASURED_PEAKS.json")))["sm_max_mhz"])
        except Exception:
            pass
        smem_peak = 128.0 * smhz * 1e6 / 1e9
        per_piv_us = upd_ms * 1e3 / max(1, window)
        small_roof = {"bound": "smem", "kernel": "k_solve_small (whole solve, one CTA, tableau in shared memory)",
                      "achieved": st.bytes_per_pivot / (per_piv_us * 1e-6) / 1e9, "peak": smem_peak,
                      "unit": "GB/s", "frac": st.bytes_per_pivot / (per_piv_us * 1e-6) / 1e9 / smem_peak,
                      "peak_source": "128 B/cycle/SM shared-memory crossbar (B300_MICROARCH.md LDS/STS) x "
                                     f"{smhz:.0f} MHz (MEASURED_PEAKS.json sm_max_mhz)",
                      "traffic": None, "bytes_per_pivot": st.bytes_per_pivot, "us_per_pivot": per_piv_us,
                      "launch_us": upd_ms * 1e3, "pivots_per_launch": window,
                      "note": "latency path (PAPER.md:161, 290): per pivot two block-wide argmins and two "
                              "barriers of 1024 threads dominate; the HBM roofline does not apply"}
    per_rank_frac = gather_list(achieved / peak, world)

    # ---- the one-pivot-per-pass kernel (k_update) measured the same way, for reference
    single = None
    if (look > 1 or small) and args.single_pass_pivots > 0:
        p1 = make(time_kernels=True, lookahead=1)
        barrier()
        p1.iterate(min(piv, args.single_pass_pivots))
        barrier()
        s1p = p1.stats()
        p1.close()
        a1 = s1p.update_ms_total / 1e3 / max(1, s1p.update_launches)
        single = {"kernel": "k_update (one pivot per pass)", "avg_launch_us": a1 * 1e6,
                  "achieved": st.bytes_per_pivot / a1 / 1e9, "peak": peak, "unit": "GB/s",
                  "frac": st.bytes_per_pivot / a1 / 1e9 / peak, "launches_timed": s1p.update_launches,
                  "traffic": ncu_traffic(args.workload, world)}

    # ---- the rank-s pass alone (select-then-pass schedule: all SMs, in place), for reference
    alone = None
    if look > 1 and not args.no_overlap and args.single_pass_pivots > 0 and world == 1:
        p2 = make(time_kernels=True, lookahead=args.lookahead, overlap=False)
        barrier()
        p2.iterate(min(piv, args.roofline_pivots))
        barrier()
        s2p = p2.stats()
        p2.close()
        a2 = s2p.update_ms_total / 1e3 / max(1, s2p.update_launches)
        alone = {"kernel": f"k_update_s (rank-{look}, select-then-pass schedule: every SM, in place)",
                 "avg_launch_us": a2 * 1e6, "achieved": st.bytes_per_pivot / a2 / 1e9, "peak": peak,
                 "unit": "GB/s", "frac": st.bytes_per_pivot / a2 / 1e9 / peak,
                 "launches_timed": s2p.update_launches}

    # ---- multi-GPU roofline terms: t_coll(P) from an exchange-only loop,
    # t_roof(P) = 16(m+1)(ceil((n+m)/P)+1)/peak + t_coll(P) per pivot (the one-pass-per-pivot
    # roofline the north_star defines); the look-ahead moves 1/look of those bytes per pivot
    t_coll = measure_tcoll(m, world, dev) if world > 1 else 0.0
    slab_bytes = 16.0 * (m + 1) * (-(-(n + m) // world) + 1)
    t_roof_us = slab_bytes / (peak * 1e9) * 1e6 + t_coll
    blocks = -(-pivs // look) if look > 1 else pivs         # passes over the tableau in the timed steps

    # ---- e2e: same metric through the C ABI with HOST buffers (pinned), copies inside
    Ah = torch.from_numpy(A).pin_memory()
    bh, ch = torch.from_numpy(b).pin_memory(), torch.from_numpy(c).pin_memory()
    xh_out = np.empty(n)
    yh_out = np.empty(m)
    barrier()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e2e_reps = args.steps if small else 1                     # a 64^2 solve is ~0.1 ms: average K calls
    if small:
        solver.solve_lp(Ah, bh, ch, xh_out, yh_out)           # (untimed warm-up of the host-input path)
        barrier()
    e0.record()
    if small:
        for _ in range(e2e_reps):
            _, _, obj_e2e, piv_e2e, _ = solver.solve_lp(Ah, bh, ch, xh_out, yh_out)
    else:
        solver.reset(Ah, bh, ch)
        solver.solve()
        _, _, obj_e2e, piv_e2e, _ = solver.solution(xh_out, yh_out)
    e1.record()
    barrier()
    e2e_ms = e0.elapsed_time(e1) / e2e_reps
    if world > 1:
        e2e_ms = reduce_max(e2e_ms, world, dev)
    ns_local = max(0, min(st.col_offset + st.local_cols - 1, n) - st.col_offset)
    h2d = 8 * (m * ns_local + m + ns_local)
    if world > 1:
        h2d = int(reduce_sum(h2d, world, dev))
    d2h = world * 8 * (n + m + 1)
    solver.close()
    del Ah, bh, ch
    barrier()

    # ---- the largest tableau (north_star scaling target) as a sub-record
    largest = None
    if args.largest not in ("none", "", args.workload):
        largest = largest_leg(args, world, group, dev, peak, barrier, exchange)

    # ---- the oracle on the host, rank 0, at every N (the other ranks wait at the barrier)
    cpu = None
    if rank == 0 and not args.no_cpu_baseline:
        cpu = cpu_baseline(A, b, c, args.cpu_sample_seconds)
    barrier()

    if rank == 0:
        line = {
            "metric": "pivots/s", "value": value, "unit": "pivots/s", "n_gpus": world, "steps": args.steps,
            "warmup": args.warmup, "ms_per_step": total_ms / args.steps, "higher_is_better": True,
            "scaling": "strong", "vs_baseline": None, "dtype": "f64",
            "data": f"synthetic (lpgen SplitMix64 dense LP seed {args.seed}: A,c~U[1,10), b~U[n,2n); "
                    "SPEC.md:365-380 recipe)",
            "config": {"workload": workload_name(m, n, args.seed, args.pivot_rule), "m": m, "n": n,
                       "pivots_per_solve": piv, "pivots_per_tableau_pass": look,
                       "schedule": "the whole solve in one single-CTA launch, tableau in shared memory" if small else
                                   ("select block b+1 (16-SM cluster) concurrently with the pass of block b "
                                    "(two tableau buffers)" if look > 1 and not args.no_overlap else
                                    "select, then pass" if look > 1 else "one pivot per pass"),
                       "time_to_solve_ms": total_ms / args.steps, "time_to_solve_us": 1e3 * total_ms / args.steps,
                       "parallelism": f"column slabs x{world}" + ((" (candidate columns exchanged over peer memory per pivot)"
                                                                   if exchange != 1 else
                                                                   " (candidate columns exchanged by NCCL allgather per pivot)")
                                                                  if world > 1 else ""),
                       "exchange": exchange if world > 1 else None, "exchange_fallback": fallback,
                       "l2": ("tableau %.2f GB > L2 %d MB: inputs larger than L2" % (tableau_bytes / 1e9, l2 >> 20))
                       if flush is None else "L2 flushed (write 2xL2) before every timed step",
                       "step": ("simplex_solve_lp: reset (build Table I from device-resident A,b,c) + solve + extract "
                                "in one call (one launch, one synchronisation)") if small else
                               "reset (build Table I from device-resident A,b,c) + solve + extract"},
            "roofline": small_roof if small else {"bound": "hbm",
                         "kernel": (f"k_update_s (rank-{look} look-ahead pass: {look} pivots per tableau "
                                    "stream, TMA loads + TMA bulk stores; runs concurrently with the "
                                    "selection of the next block)") if look > 1 else
                                   "k_update (fused row-scale + rank-1 update)",
                         "achieved": achieved, "peak": peak, "unit": "GB/s", "frac": achieved / peak,
                         "frac_of_8tbs_spec": achieved / 8000.0,
                         "l2_bytes_per_launch": ncu_l2(args.workload, world, look),
                         "per_rank_frac": per_rank_frac,
                         "peak_source": peak_src, "traffic": ncu_traffic(args.workload, world, look),
                         "bytes_per_launch": st.bytes_per_pivot,
                         "bytes_formula": "16*(m+1)*(local columns incl. rhs): every slab element read and "
                                          "written once per pass",
                         "avg_launch_us": avg_upd_s * 1e6, "launches_timed": upd_launches,
                         "timing_source": ("device %globaltimer in the kernel (first CTA start -> last CTA end), "
                                           "production launch sequence, next to the concurrent selection")
                         if look > 1 and not args.no_overlap else "CUDA events around every launch",
                         "ncu_avg_launch_us": ncu_duration(args.workload, world, look),
                         "ncu_note": "ncu's gpu__time_duration (profiles/) is a replayed, serialised, cold-cache "
                                     "launch incl. launch latency and CTA ramp-up; it bounds the device-timed "
                                     "figure from above (~5 % at 8000^2)",
                         "timed_window": f"first {window} pivots of the same solve",
                         "update_share_of_loop": upd_ms / prof_loop_ms if prof_loop_ms > 0 else None,
                         "pivots_per_launch": look,
                         "passes_per_step": blocks / args.steps,
                         "algorithmic_bytes_per_step": st.bytes_per_pivot * blocks / args.steps,
                         "algorithmic_gbs_over_step": st.bytes_per_pivot * blocks / (total_ms / 1e3) / 1e9,
                         "single_pass_equivalent_gb_per_step": st.bytes_per_pivot * pivs / args.steps / 1e9,
                         "single_pass": single, "pass_alone": alone,
                         "note": ("tableau resident in L2 (%.0f MB per buffer < %d MB L2): the pass runs from L2, "
                                  "so its fraction of the HBM peak is not a roofline" % (tableau_bytes / 1e6, l2 >> 20))
                         if 2 * tableau_bytes < l2 else None},
            "multi_gpu": {"P": world, "t_coll_us_per_pivot": t_coll,
                          "t_coll_how": "exchange-only loop: NCCL allgather of (m+3) doubles per rank, 200 "
                                        "iterations, CUDA events, max over ranks" if world > 1 else "1 GPU: no exchange",
                          "t_roof_us_per_pivot": t_roof_us,
                          "t_roof_formula": "16(m+1)(ceil((n+m)/P)+1)/peak + t_coll(P) (one pass per pivot)",
                          "roof_pivots_per_s": 1e6 / t_roof_us,
                          "value_over_single_pass_roof": value / (1e6 / t_roof_us),
                          "loop_ms": loop_ms,
                          "efficiency_inputs": {"value": value, "P": world}},
            "cpu_baseline": cpu,
            "small_path": small,
            "e2e": {"value": piv_e2e / (e2e_ms / 1e3), "unit": "pivots/s", "h2d_bytes_per_step": h2d,
                    "d2h_bytes_per_step": d2h, "ms": e2e_ms,
                    "path": "simplex_solve_lp(pinned host A,b,c -> host x,y)" if small else
                            "simplex_reset(pinned host A,b,c) + simplex_solve + simplex_get_solution(host x,y)"},
            "gpu_launches": int(s1.kernel_launches - s0.kernel_launches),
            "clocks": clk, "parity": parity, "largest": largest, "context": PAPER_CONTEXT,
        }
        print(json.dumps(line), flush=True)
    if world > 1:
        torch.distributed.destroy_process_group()
    return 0


if __name__ == "__main__":
    sys.exit(main())
