"""Drive a few look-ahead blocks for ncu: python scripts/prof_lookahead.py 8000x8000 S blocks."""
import os
import sys

sys.path.insert(0, os.path.join(os.path.dirname(os.path.abspath(__file__)), ".."))
import torch  # noqa: E402

import lpgen  # noqa: E402
import paper_2211_10979_b200 as sx  # noqa: E402

m, n = map(int, sys.argv[1].split("x"))
S = int(sys.argv[2]) if len(sys.argv) > 2 else 16
blocks = int(sys.argv[3]) if len(sys.argv) > 3 else 4
torch.cuda.set_device(0)
A, b, c = lpgen.dense_lp(m, n, 1)
with sx.Simplex(A, b, c, lookahead=S, segment_pivots=S) as s:
    done, st = s.iterate(S * blocks)
    print("pivots", done, sx.STATUS_NAME[st])
