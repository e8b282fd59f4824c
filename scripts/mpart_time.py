import os, sys
sys.path.insert(0, os.path.join(os.path.dirname(os.path.abspath(__file__)), ".."))
import torch, lpgen, paper_2211_10979_b200 as sx
m, n = map(int, sys.argv[1].split("x"))
torch.cuda.set_device(0)
A, b, c = lpgen.dense_lp(m, n, 1)
Ad, bd, cd = (torch.from_numpy(v).cuda() for v in (A, b, c))
for ov in (True, False):
    with sx.Simplex(Ad, bd, cd, virtual_ranks=2, exchange=2, overlap=ov, time_kernels=True) as s:
        s.iterate(64)
        torch.cuda.synchronize()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record(); done, _ = s.iterate(640); e1.record(); torch.cuda.synchronize()
        st = s.stats()
        print(f"{m}x{n} P=2 overlap={ov}: block {e0.elapsed_time(e1)*1e3/(done/16):.0f} us, "
              f"slab-0 pass {st.update_ms_total*1e3/max(1,st.update_launches):.0f} us ({st.update_launches} launches)", flush=True)
