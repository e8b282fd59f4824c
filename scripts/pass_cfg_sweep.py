"""Pipelined block time and device-timed pass per rank-s pass ring configuration (experiment;
SIMPLEX_PASS_CFG hook, read at handle creation), one LP generated once.
    python scripts/pass_cfg_sweep.py 20000x40000 [pivots] [cfgs]"""
import os
import sys

sys.path.insert(0, os.path.join(os.path.dirname(os.path.abspath(__file__)), ".."))
import torch  # noqa: E402

import lpgen  # noqa: E402
import paper_2211_10979_b200 as sx  # noqa: E402
import _experiment  # noqa: E402
_experiment.load(os.environ.get("SIMPLEX_EXPERIMENT_LIB"))

m, n = map(int, sys.argv[1].split("x"))
piv = int(sys.argv[2]) if len(sys.argv) > 2 else 1600
cfgs = (sys.argv[3] if len(sys.argv) > 3 else "0,1,2,3,4,5").split(",")
torch.cuda.set_device(0)
A, b, c = lpgen.dense_lp(m, n, 1)
for cfg in cfgs:
    os.environ["SIMPLEX_PASS_CFG"] = cfg
    with sx.Simplex(A, b, c, time_kernels=True) as s:
        s.iterate(64)
        torch.cuda.synchronize()
        st0 = s.stats()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        done, _ = s.iterate(piv)
        e1.record()
        torch.cuda.synchronize()
        st = s.stats()
    blk = e0.elapsed_time(e1) * 1e3 / (done / 16)
    pas = (st.update_ms_total - st0.update_ms_total) * 1e3 / max(1, st.update_launches - st0.update_launches)
    print(f"{m}x{n} pass_cfg {cfg}: block {blk:.1f} us, pass {pas:.1f} us "
          f"({16.0 * (m + 1) * (n + m + 1) / pas / 1e3:.0f} GB/s)", flush=True)
