"""Rank-32 pass duration per ring configuration (experiment): python scripts/pair_pass_sweep.py 8000x8000"""
import os
import subprocess
import sys

if len(sys.argv) > 2:
    sys.path.insert(0, os.path.join(os.path.dirname(os.path.abspath(__file__)), ".."))
    import torch
    import lpgen
    import paper_2211_10979_b200 as sx
    import _experiment
    _experiment.load()
    m, n = map(int, sys.argv[1].split("x"))
    torch.cuda.set_device(0)
    A, b, c = lpgen.dense_lp(m, n, 1)
    with sx.Simplex(A, b, c, lookahead=int(sys.argv[2]), time_kernels=True) as s:
        s.iterate(1024)
        st = s.stats()
    us = st.update_ms_total * 1e3 / max(1, st.update_launches)
    print(f"cfg {os.environ.get('SIMPLEX_PASS_CFG')} look {sys.argv[2]}: pass {us:.1f} us "
          f"{16.0 * (m + 1) * (n + m + 1) / us / 1e3:.0f} GB/s", flush=True)
else:
    for look in (32, 24, 16):
        for cfg in range(6):
            subprocess.run([sys.executable, __file__, sys.argv[1], str(look)], env=dict(os.environ, SIMPLEX_PASS_CFG=str(cfg)))
