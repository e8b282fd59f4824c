#!/bin/bash
# Round-2 measurement set (GPU box): bench lines for every single-GPU config and the reference
# (oracle) arm, plus smoke.  Outputs in gpurun_out/final/.
o=gpurun_out/final
mkdir -p $o
python -c "import __graft_entry__ as g; g.smoke()" > $o/smoke.txt 2>&1; tail -4 $o/smoke.txt
python bench.py --steps 20 --warmup 5 > $o/bench_8000.json 2> $o/bench_8000.err; tail -c 400 $o/bench_8000.json
python bench.py --workload 4000x4000 --steps 10 --warmup 3 --largest none --no-cpu-baseline > $o/bench_4000.json 2> $o/bench_4000.err
python bench.py --workload 1000x1000 --steps 20 --warmup 5 --largest none --no-cpu-baseline > $o/bench_1000.json 2> $o/bench_1000.err
python bench.py --workload 64x64 --steps 50 --warmup 5 --largest none > $o/bench_64.json 2> $o/bench_64.err
python bench.py --workload 20000x40000 --steps 1 --warmup 3 --no-cpu-baseline --roofline-pivots 1600 \
  --single-pass-pivots 200 > $o/bench_20000.json 2> $o/bench_20000.err
python bench.py --impl reference --steps 2 --warmup 1 > $o/bench_reference.json 2> $o/bench_reference.err
for f in $o/bench_*.json; do python - "$f" <<'PY'
import json, sys
d = json.loads(open(sys.argv[1]).read().strip().splitlines()[-1])
r = d.get("roofline") or {}
print(sys.argv[1], d.get("value"), d.get("config", {}).get("time_to_solve_ms"), r.get("frac"), (d.get("parity") or {}).get("checked"),
      (d.get("largest") or {}).get("value"), (d.get("clocks") or {}).get("sm_mhz"))
PY
done
