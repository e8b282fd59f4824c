"""Average look-ahead selection / pass durations vs the pipelined block time (experiment).

    python scripts/pipe_probe.py 8000x8000 [pivots]
Runs the first `pivots` pivots three times: pipelined (block time), time_kernels around the
pass, and (SIMPLEX_TIME_SELECT=1 in a child) around the selection."""
import os
import subprocess
import sys

sys.path.insert(0, os.path.join(os.path.dirname(os.path.abspath(__file__)), ".."))
import torch  # noqa: E402

import lpgen  # noqa: E402
import paper_2211_10979_b200 as sx  # noqa: E402
import _experiment  # noqa: E402
_experiment.load()

m, n = map(int, sys.argv[1].split("x"))
piv = int(sys.argv[2]) if len(sys.argv) > 2 else 4000
torch.cuda.set_device(0)
A, b, c = lpgen.dense_lp(m, n, 1)
Ad, bd, cd = (torch.from_numpy(v).cuda() for v in (A, b, c))


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
        return e0.elapsed_time(e1) * 1e3 / (done / 16), st


if os.environ.get("SIMPLEX_TIME_SELECT"):
    _, st = timed(time_kernels=True)
    print("select_us %.1f" % (st.update_ms_total * 1e3 / max(1, st.update_launches)))
    sys.exit(0)
blk, _ = timed()
print("pipelined block_us %.1f" % blk)
blk2, _ = timed(overlap=False)
print("serial block_us %.1f" % blk2)
_, st = timed(time_kernels=True)
print("pass_us %.1f" % (st.update_ms_total * 1e3 / max(1, st.update_launches)))
subprocess.run([sys.executable] + sys.argv, env=dict(os.environ, SIMPLEX_TIME_SELECT="1"))
