"""Pivots/s of consecutive simplex_iterate windows over one full solve (is a late block slower
than an early one?), with the SM clock sampled during each window.
    python scripts/window_profile.py 8000x8000 [window] [--solves N]"""
import os
import subprocess
import sys
import threading
import time

sys.path.insert(0, os.path.join(os.path.dirname(os.path.abspath(__file__)), ".."))
import torch  # noqa: E402

import lpgen  # noqa: E402
import paper_2211_10979_b200 as sx  # noqa: E402

m, n = map(int, sys.argv[1].split("x"))
win = int(sys.argv[2]) if len(sys.argv) > 2 and sys.argv[2].isdigit() else 3200
solves = int(sys.argv[sys.argv.index("--solves") + 1]) if "--solves" in sys.argv else 2
torch.cuda.set_device(0)
A, b, c = lpgen.dense_lp(m, n, 1)
Ad, bd, cd = (torch.from_numpy(v).cuda() for v in (A, b, c))
clk = []
stop = False


def sampler():
    while not stop:
        r = subprocess.run(["nvidia-smi", "--query-gpu=clocks.sm,power.draw", "--format=csv,noheader,nounits"],
                           capture_output=True, text=True).stdout.strip().split(",")
        try:
            clk.append((time.time(), float(r[0]), float(r[1])))
        except Exception:
            pass
        time.sleep(0.05)


th = threading.Thread(target=sampler, daemon=True)
th.start()
with sx.Simplex(Ad, bd, cd) as s:
    for rep in range(solves):
        s.reset(Ad, bd, cd)
        torch.cuda.synchronize()
        tot = 0
        while True:
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            t0 = time.time()
            e0.record()
            done, st = s.iterate(win)
            e1.record()
            torch.cuda.synchronize()
            t1 = time.time()
            ms = e0.elapsed_time(e1)
            cs = [v for (t, v, p) in clk if t0 <= t <= t1]
            ps = [p for (t, v, p) in clk if t0 <= t <= t1]
            tot += done
            if done:
                print(f"solve {rep} pivots {tot - done:6d}-{tot:6d}: {done / ms * 1e3:8.0f} piv/s  "
                      f"{ms * 1e3 / max(done, 1) * 16:6.1f} us/block  sm {sum(cs) / max(len(cs), 1):6.0f} MHz  "
                      f"{sum(ps) / max(len(ps), 1):5.0f} W", flush=True)
            if st != sx.RUNNING or done == 0:
                break
stop = True
