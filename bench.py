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
            "sample": f"first {r.pivots} pivots of the {m}x{n} seed solve (oracle/simplex_oracle.c, 1 thread, "
                      f"tableau build excluded), {dt:.1f} s"}


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

    def pivots(P):
        for _ in range(P):
            k, _ = oracle.price(T[0, :-1])
            if k < 0:
                return
            r, _ = oracle.ratio(T, k)
            if r < 0:
                return
            oracle.pivot(T, r, k)
            basis[r - 1] = k
            done[0] += 1

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
            "config": {"workload": f"dense random LP m={m} n={n} FP64 seed {args.seed}", "m": m, "n": n},
            "cpu_baseline": {"value": v, "unit": "pivots/s", "cores": 1, "kind": "oracle",
                             "sample": f"each step: the next {P} pivots of the {m}x{n} solve through the "
                                       "oracle's step functions (tableau built once, untimed)"},
            "e2e": {"value": v, "unit": "pivots/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0}}
    print(json.dumps(line), flush=True)
    return 0


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
    solver = sx.Simplex(dA, db, dc, group=group, lookahead=args.lookahead, pivot_rule=rule,
                        overlap=not args.no_overlap)
    st = solver.stats()
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
        if reload:
            solver.reset(dA, db, dc)
        status = solver.solve()
        _, _, obj, piv, _ = solver.solution(dx, dy)
        return status, obj, piv

    # ---- correctness gate before timing: golden trace/objective when present
    status, obj, piv = one_step(reload=False)
    parity = {"checked": False}
    gpath = os.path.join(ROOT, "tests", "golden", f"dense_{m}x{n}_s{args.seed}.npz")
    if args.pivot_rule != "dantzig":
        gpath = gpath[:-4] + f"_{args.pivot_rule}.npz"
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

    # ---- roofline pass: the same solve with CUDA events around every k_update launch
    # (event-record nodes in the captured graph, on the stream the kernel runs on).  Kept
    # out of the value steps because an event node between two pivot kernels disables the
    # programmatic-dependent-launch edge the production loop uses.  The pipelined rank-s pass
    # is timed on the device instead (globaltimer in the kernel, the production launch
    # sequence), because event nodes would serialize it after the concurrent selection.
    prof = sx.Simplex(dA, db, dc, group=group, time_kernels=True, lookahead=args.lookahead, pivot_rule=rule,
                      overlap=not args.no_overlap)
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
    loop_ms = s1.loop_ms_total - s0.loop_ms_total
    prof_loop_ms = sp.loop_ms_total
    look = solver_look(args.lookahead, world)

    # ---- the one-pivot-per-pass kernel (k_update) measured the same way, for reference
    single = None
    if look > 1 and args.single_pass_pivots > 0:
        p1 = sx.Simplex(dA, db, dc, group=group, time_kernels=True, lookahead=1, pivot_rule=rule)
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
    if look > 1 and not args.no_overlap and args.single_pass_pivots > 0:
        p2 = sx.Simplex(dA, db, dc, group=group, time_kernels=True, lookahead=args.lookahead, pivot_rule=rule,
                        overlap=False)
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

    # ---- e2e: same metric through the C ABI with HOST buffers (pinned), copies inside
    Ah = torch.from_numpy(A).pin_memory()
    bh, ch = torch.from_numpy(b).pin_memory(), torch.from_numpy(c).pin_memory()
    xh_out = np.empty(n)
    yh_out = np.empty(m)
    barrier()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    solver.reset(Ah, bh, ch)
    solver.solve()
    _, _, obj_e2e, piv_e2e, _ = solver.solution(xh_out, yh_out)
    e1.record()
    barrier()
    e2e_ms = e0.elapsed_time(e1)
    if world > 1:
        e2e_ms = reduce_max(e2e_ms, world, dev)
    ns_local = max(0, min(st.col_offset + st.local_cols - 1, n) - st.col_offset)
    h2d = 8 * (m * ns_local + m + ns_local)
    if world > 1:
        h2d = int(reduce_sum(h2d, world, dev))
    d2h = world * 8 * (n + m + 1)

    cpu = None
    if rank == 0 and world == 1 and not args.no_cpu_baseline:
        cpu = cpu_baseline(A, b, c, args.cpu_sample_seconds)

    solver.close()
    if rank == 0:
        line = {
            "metric": "pivots/s", "value": value, "unit": "pivots/s", "n_gpus": world, "steps": args.steps,
            "warmup": args.warmup, "ms_per_step": total_ms / args.steps, "higher_is_better": True,
            "scaling": "strong", "vs_baseline": None, "dtype": "f64",
            "data": f"synthetic (lpgen SplitMix64 dense LP seed {args.seed}: A,c~U[1,10), b~U[n,2n); "
                    "SPEC.md:365-380 recipe)",
            "config": {"workload": f"dense random LP m={m} n={n} FP64 seed {args.seed}, slack basis, "
                                   + ("Dantzig + lowest-index ties" if args.pivot_rule == "dantzig" else
                                      "Bland's rule"), "m": m, "n": n, "pivots_per_solve": piv,
                       "pivots_per_tableau_pass": look,
                       "schedule": ("select block b+1 (16-SM cluster) concurrently with the pass of block b "
                                    "(two tableau buffers)" if look > 1 and not args.no_overlap else
                                    "select, then pass" if look > 1 else "one pivot per pass"),
                       "time_to_solve_ms": total_ms / args.steps,
                       "parallelism": f"column slabs x{world}" + (" (candidate columns exchanged over peer memory per pivot)" if world > 1 else ""),
                       "l2": ("tableau %.2f GB > L2 %d MB: inputs larger than L2" % (tableau_bytes / 1e9, l2 >> 20))
                       if flush is None else "L2 flushed (write 2xL2) before every timed step",
                       "step": "reset (build Table I from device-resident A,b,c) + solve + extract"},
            "roofline": {"bound": "hbm",
                         "kernel": (f"k_update_s (rank-{look} look-ahead pass: {look} pivots per tableau "
                                    "stream, TMA loads + TMA bulk stores; runs concurrently with the "
                                    "selection of the next block)") if look > 1 else
                                   "k_update (fused row-scale + rank-1 update)",
                         "achieved": achieved, "peak": peak, "unit": "GB/s", "frac": achieved / peak,
                         "peak_source": peak_src, "traffic": ncu_traffic(args.workload, world, look),
                         "bytes_per_launch": st.bytes_per_pivot,
                         "bytes_formula": "16*(m+1)*(local columns incl. rhs) per pivot",
                         "avg_launch_us": avg_upd_s * 1e6, "launches_timed": upd_launches,
                         "timed_window": (f"first {window} pivots of the same solve; each pass launch timed on the "
                                          "device (%globaltimer, first CTA start -> last CTA end) while the "
                                          "selection of the next block runs next to it")
                         if look > 1 and not args.no_overlap else
                         f"first {window} pivots of the same solve, CUDA events per launch",
                         "update_share_of_loop": upd_ms / prof_loop_ms if prof_loop_ms > 0 else None,
                         "pivots_per_launch": look,
                         "effective_gbs_per_pivot": st.bytes_per_pivot * pivs / (loop_ms / 1e3) / 1e9
                         if loop_ms > 0 else None,
                         "single_pass": single, "pass_alone": alone,
                         "note": ("tableau resident in L2 (%.0f MB per buffer < %d MB L2): the pass runs from L2, "
                                  "so its fraction of the HBM peak is not a roofline" % (tableau_bytes / 1e6, l2 >> 20))
                         if 2 * tableau_bytes < l2 else None},
            "cpu_baseline": cpu,
            "e2e": {"value": piv_e2e / (e2e_ms / 1e3), "unit": "pivots/s", "h2d_bytes_per_step": h2d,
                    "d2h_bytes_per_step": d2h, "ms": e2e_ms,
                    "path": "simplex_reset(pinned host A,b,c) + simplex_solve + simplex_get_solution(host x,y)"},
            "gpu_launches": int(s1.kernel_launches - s0.kernel_launches),
            "clocks": clk, "parity": parity, "context": PAPER_CONTEXT,
        }
        print(json.dumps(line), flush=True)
    if world > 1:
        torch.distributed.destroy_process_group()
    return 0


if __name__ == "__main__":
    sys.exit(main())
