"""Per-step phase times of k_lookahead (profiling build):
    SIMPLEX_LIB=paper_2211_10979_b200/libsimplex_prof.so python scripts/lprof.py 8000x8000 [blocks]"""
import ctypes as C
import os
import sys

import numpy as np

sys.path.insert(0, os.path.join(os.path.dirname(os.path.abspath(__file__)), ".."))
import torch  # noqa: E402

import lpgen  # noqa: E402
import paper_2211_10979_b200 as sx  # noqa: E402

m, n = map(int, sys.argv[1].split("x"))
blocks = int(sys.argv[2]) if len(sys.argv) > 2 else 3
skip = int(sys.argv[3]) if len(sys.argv) > 3 else 0
torch.cuda.set_device(0)
A, b, c = lpgen.dense_lp(m, n, 1)
L = sx.lib()
L.simplex_debug_lookahead_profile.argtypes = [C.c_void_p]
CLK = 1965.0  # SM clock stamps (clock64), cycles per microsecond at 1965 MHz
seg = int(os.environ.get("LPROF_SEG", "16"))
with sx.Simplex(A, b, c, lookahead=16, segment_pivots=seg, overlap=os.environ.get("LPROF_OVERLAP", "1") == "1") as s:
    if skip:
        s.iterate(skip)
    for blk in range(blocks):
        s.iterate(seg)
        buf = np.zeros(16 * (16 * 4 + 4), dtype=np.uint64)
        L.simplex_debug_lookahead_profile(C.c_void_p(buf.ctypes.data))
        allt = buf.astype(np.int64).reshape(16, 68)
        t = allt[0]
        # per-CTA end of phase B (slot 4u+3) relative to CTA 0's, averaged over steps
        startA = allt[:, 1:64:4] - allt[:, 0:64:4]
        print("  phase-A duration per CTA (us):", np.round(startA.mean(axis=1) / CLK, 1).tolist())
        rows = []
        for u in range(16):
            a0, a1, a2, a3 = t[4 * u:4 * u + 4]
            nxt = t[4 * u + 4] if u < 15 else t[64]
            rows.append((a1 - a0, a2 - a1, a3 - a2, nxt - a3))
        r = np.array(rows) / CLK
        print(f"block {blk}: phaseA {r[:,0].mean():.2f}  redA {r[:,1].mean():.2f}  phaseB {r[:,2].mean():.2f}  "
              f"redB {r[:,3].mean():.2f} us/step; step total {(t[64]-t[0])/16/CLK:.2f} us")
