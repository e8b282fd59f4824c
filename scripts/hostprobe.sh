nproc; lscpu | head -30; free -g; numactl -H 2>/dev/null | head -5; nvidia-smi --query-gpu=name,clocks.max.sm --format=csv
python - <<'PY'
import sys,time,os
sys.path.insert(0,'.')
import numpy as np, oracle, lpgen
os.environ.setdefault("OMP_NUM_THREADS", str(os.cpu_count()))
t=time.time(); A,b,c=lpgen.dense_lp(20000,40000,1); print("gen",time.time()-t, flush=True)
t=time.time(); T,basis=oracle.build_tableau(A,b,c); print("build",time.time()-t, flush=True)
del A
st,it,k,r=oracle.iterate(T,basis,0,stop_at=2,parallel=True)
t=time.time(); st,it,k,r=oracle.iterate(T,basis,it,stop_at=12,parallel=True); print("10 pivots",time.time()-t, os.environ["OMP_NUM_THREADS"], flush=True)
PY
