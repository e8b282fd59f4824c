"""k_solve_small launch time per pivot vs threads per CTA (experiment; SIMPLEX_SMALL_THREADS hook).
    python scripts/small_probe.py [64x64] [seeds]"""
import os
import sys

sys.path.insert(0, os.path.join(os.path.dirname(os.path.abspath(__file__)), ".."))
import torch  # noqa: E402

import lpgen  # noqa: E402
import paper_2211_10979_b200 as sx  # noqa: E402
import _experiment  # noqa: E402
_experiment.load()

m, n = map(int, (sys.argv[1] if len(sys.argv) > 1 else "64x64").split("x"))
seeds = int(sys.argv[2]) if len(sys.argv) > 2 else 10
torch.cuda.set_device(0)
for nt in (128, 256, 512, 1024):
    os.environ["SIMPLEX_SMALL_THREADS"] = str(nt)
    us, piv = 0.0, 0
    for seed in range(1, seeds + 1):
        A, b, c = lpgen.dense_lp(m, n, seed)
        with sx.Simplex(A, b, c, time_kernels=True) as s:
            for _ in range(3):
                s.reset(A, b, c)
                s.solve()
            st = s.stats()
            us += st.update_ms_total * 1e3 / st.update_launches
            piv += st.pivots
    print(f"{m}x{n} threads {nt}: {us / piv:.3f} us/pivot over {seeds} seeds ({piv} pivots)", flush=True)
