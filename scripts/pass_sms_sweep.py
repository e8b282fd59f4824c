"""Pipelined rank-16 block time vs the SMs given to the concurrent pass (experiment;
SIMPLEX_PASS_SMS hook): a gentler pass leaves the HBM queues shorter for the selection's
dependent loads.   python scripts/pass_sms_sweep.py 4000x4000 [pivots] [sms,...]"""
import os
import subprocess
import sys

if len(sys.argv) > 1 and sys.argv[1] == "--one":
    sys.path.insert(0, os.path.join(os.path.dirname(os.path.abspath(__file__)), ".."))
    import torch
    import lpgen
    import paper_2211_10979_b200 as sx
    import _experiment
    _experiment.load(os.environ.get("SIMPLEX_EXPERIMENT_LIB"))
    m, n = map(int, sys.argv[2].split("x"))
    piv = int(sys.argv[3])
    torch.cuda.set_device(0)
    A, b, c = lpgen.dense_lp(m, n, 1)
    Ad, bd, cd = (torch.from_numpy(v).cuda() for v in (A, b, c))
    out = []
    for tk in (False, True):
        with sx.Simplex(Ad, bd, cd, time_kernels=tk) as s:
            s.iterate(64)
            torch.cuda.synchronize()
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            e0.record()
            done, _ = s.iterate(piv)
            e1.record()
            torch.cuda.synchronize()
            st = s.stats()
            out.append(e0.elapsed_time(e1) * 1e3 / (done / 16) if not tk else
                       st.update_ms_total * 1e3 / max(1, st.update_launches))
    print(f"{m}x{n} pass_sms {os.environ.get('SIMPLEX_PASS_SMS', 'default')}: block {out[0]:.1f} us, "
          f"pass {out[1]:.1f} us", flush=True)
else:
    sys.path.insert(0, os.path.dirname(os.path.abspath(__file__)))
    import _experiment
    lib = _experiment.load()
    sz = sys.argv[1]
    piv = sys.argv[2] if len(sys.argv) > 2 else "3000"
    sms = (sys.argv[3] if len(sys.argv) > 3 else "0,120,104,88,72,56,40").split(",")
    for v in sms:
        env = dict(os.environ, SIMPLEX_EXPERIMENT_LIB=lib)
        if v != "0":
            env["SIMPLEX_PASS_SMS"] = v
        subprocess.run([sys.executable, __file__, "--one", sz, piv], env=env)
