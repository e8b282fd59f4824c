"""Per-pivot time of the look-ahead schedules on the first `pivots` pivots (experiment).

    python scripts/pair_probe.py 20000x40000 [pivots]
Schedules: rank-16 pipelined (default), rank-16 select-then-pass, pair (rank-32: two selections,
one pass); plus the pair's pass duration (time_kernels)."""
import os
import sys

sys.path.insert(0, os.path.join(os.path.dirname(os.path.abspath(__file__)), ".."))
import torch  # noqa: E402

import lpgen  # noqa: E402
import paper_2211_10979_b200 as sx  # noqa: E402

m, n = map(int, sys.argv[1].split("x"))
piv = int(sys.argv[2]) if len(sys.argv) > 2 else 1600
torch.cuda.set_device(0)
A, b, c = lpgen.dense_lp(m, n, 1)
Ad, bd, cd = (torch.from_numpy(v).cuda() for v in (A, b, c))
del A, b, c


def timed(**kw):
    with sx.Simplex(Ad, bd, cd, **kw) as s:
        s.iterate(64)
        torch.cuda.synchronize()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        done, _ = s.iterate(piv)
        e1.record()
        torch.cuda.synchronize()
        st = s.stats()
        return e0.elapsed_time(e1) * 1e3 / done, st


for name, kw in [("look16 pipelined", {}), ("look16 serial", dict(overlap=False)), ("pair32", dict(lookahead=32))]:
    us, _ = timed(**kw)
    print(f"{m}x{n} {name:18s} {us:8.2f} us/pivot  {1e6 / us:9.0f} pivots/s", flush=True)
_, st = timed(lookahead=32, time_kernels=True)
print(f"{m}x{n} pair32 pass {st.update_ms_total * 1e3 / max(1, st.update_launches):.1f} us "
      f"({16.0 * (m + 1) * (n + m + 1) / (st.update_ms_total / max(1, st.update_launches)) / 1e6:.0f} GB/s)")
