"""Block time of the multi-part rank-16 look-ahead on one GPU (experiment).

    python scripts/mpart_probe.py 8000x8000 [pivots]
virtual slabs P = 1 (pipelined single part), 2, 4, and the 1-rank NCCL exchange path."""
import os
import sys

sys.path.insert(0, os.path.join(os.path.dirname(os.path.abspath(__file__)), ".."))
import torch  # noqa: E402

import lpgen  # noqa: E402
import paper_2211_10979_b200 as sx  # noqa: E402
import _experiment  # noqa: E402
_experiment.load()

m, n = map(int, sys.argv[1].split("x"))
piv = int(sys.argv[2]) if len(sys.argv) > 2 else 2000
torch.cuda.set_device(0)
A, b, c = lpgen.dense_lp(m, n, 1)
Ad, bd, cd = (torch.from_numpy(v).cuda() for v in (A, b, c))


def timed(label, **kw):
    with sx.Simplex(Ad, bd, cd, **kw) as s:
        s.iterate(64)
        torch.cuda.synchronize()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        done, _ = s.iterate(piv)
        e1.record()
        torch.cuda.synchronize()
        us = e0.elapsed_time(e1) * 1e3
        print(f"{label}: {us / done:.1f} us/pivot, {us / (done / 16):.1f} us/block")


if "--nccl" in sys.argv:
    timed("nccl 1-rank look16", exchange=1)
    timed("nccl 1-rank one pivot per pass", lookahead=1, exchange=1)
    sys.exit(0)
timed("1 part, pipelined")
for P in (2, 4):
    timed(f"{P} virtual slabs look16, peer-memory protocol, pipelined", virtual_ranks=P, exchange=2)
    timed(f"{P} virtual slabs look16, peer-memory protocol, select then pass", virtual_ranks=P, exchange=2,
          overlap=False)
    timed(f"{P} virtual slabs look16, direct (stream order)", virtual_ranks=P)
    timed(f"{P} virtual slabs one pivot per pass", virtual_ranks=P, lookahead=1)
