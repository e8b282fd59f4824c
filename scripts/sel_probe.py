"""Phase breakdown of the look-ahead selection (experiment; SIMPLEX_PROBE hook).

    python scripts/sel_probe.py 8000x8000 [pivots] [--serial]
Runs `pivots` pivots of the seed-1 LP with %globaltimer stamps in k_lookahead (CTA thread 0 of
each of the 16 CTAs, last 64 launches) and prints the mean time per pivot of: phase A (rows:
chained column + ratio test), reduction A (cluster argmin -> r), phase B (columns: chained pivot
row + objective row + pricing), reduction B (-> next k), per CTA min/mean/max."""
import os
import sys

import numpy as np

sys.path.insert(0, os.path.join(os.path.dirname(os.path.abspath(__file__)), ".."))
path = "/tmp/sx_probe.bin"
os.environ["SIMPLEX_PROBE"] = path
import torch  # noqa: E402

import lpgen  # noqa: E402
import paper_2211_10979_b200 as sx  # noqa: E402
import _experiment  # noqa: E402
_experiment.load()

m, n = map(int, sys.argv[1].split("x"))
piv = int(sys.argv[2]) if len(sys.argv) > 2 and sys.argv[2].isdigit() else 2000
serial = "--serial" in sys.argv
torch.cuda.set_device(0)
A, b, c = lpgen.dense_lp(m, n, 1)
Ad, bd, cd = (torch.from_numpy(v).cuda() for v in (A, b, c))
with sx.Simplex(Ad, bd, cd, overlap=not serial) as s:
    s.iterate(piv)
    torch.cuda.synchronize()
K, NE = 16, 10
EV = 2 + NE * K
P = np.fromfile(path, dtype=np.uint64).reshape(64, 16, EV).astype(np.float64)
ok = (P > 0).all(axis=(1, 2)) & (np.diff(P, axis=2) >= 0).all(axis=(1, 2))
ok &= (P[:, :, EV - 1] - P[:, :, 0] < 5e6).all(axis=1)
P = P[ok]                                   # complete launches, stamps of one launch only
if os.environ.get("SIMPLEX_PROBE_DETAIL"):
    P = P * 1e3 / float(os.environ.get("SIMPLEX_PROBE_MHZ", "1965"))   # cycles -> ns
print(f"{len(P)} complete launches ({'serial' if serial else 'pipelined'}), {m}x{n}")
t0 = P[:, :, 0:1]
tot = (P[:, :, EV - 1] - P[:, :, 0]) / 1e3
print(f"launch: {tot.mean():.1f} us (CTA min {tot.min(axis=1).mean():.1f} max {tot.max(axis=1).mean():.1f})")
pro = (P[:, :, 1] - P[:, :, 0]) / 1e3
print(f"prologue (cache fill + first pricing + reduction): {pro.mean():.2f} us")
prev = P[:, :, 1]
names = ["A: loads arrive", "A: chain+ratio", "redA: CTA", "redA: cl.barrier", "redA: fold",
         "B: loads arrive", "B: chain+price", "redB: CTA", "redB: cl.barrier", "redB: fold"]
if os.environ.get("SIMPLEX_PROBE_DETAIL"):      # library built with -DSX_PROBE_DETAIL (k_look2 only)
    names = ["A: loads arrive", "A: rhs+mark", "A: chains", "A: store+div", "redA (all)",
             "B: loads arrive", "B: chains", "B: div+R0+cand", "redB (all)", "(none)"]
    # stamps are SM clock64 cycles: report us at the SM clock given (MHz), default 1965
acc = {nm: [] for nm in names}
for t in range(K):
    for q, nm in enumerate(names):
        cur = P[:, :, 2 + NE * t + q]
        acc[nm].append((cur - prev) / 1e3)
        prev = cur
for nm in names:
    a = np.stack(acc[nm])                                 # [t, launch, cta]
    print(f"{nm:16s} mean {a.mean():6.2f} us   CTA-min {a.min(axis=2).mean():6.2f}  CTA-max {a.max(axis=2).mean():6.2f}"
          f"   t=0 {a[0].mean():6.2f}  t=15 {a[-1].mean():6.2f}")
