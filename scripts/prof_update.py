"""Drive a few pivots of a workload for ncu captures: python scripts/prof_update.py 8000x8000 [pivots] [P]."""
import os
import sys

sys.path.insert(0, os.path.join(os.path.dirname(os.path.abspath(__file__)), ".."))
import torch  # noqa: E402

import lpgen  # noqa: E402
import paper_2211_10979_b200 as sx  # noqa: E402

m, n = map(int, sys.argv[1].split("x"))
piv = int(sys.argv[2]) if len(sys.argv) > 2 else 6
P = int(sys.argv[3]) if len(sys.argv) > 3 else 1
torch.cuda.set_device(0)
A, b, c = lpgen.dense_lp(m, n, 1)
with sx.Simplex(A, b, c, virtual_ranks=P, segment_pivots=2) as s:
    done, st = s.iterate(piv)
    print("pivots", done, sx.STATUS_NAME[st])
