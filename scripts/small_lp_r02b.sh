#!/bin/bash
o=gpurun_out/small; mkdir -p $o
timeout 900 python -m pytest -x -q -m gpu tests/test_gpu_small.py > $o/pytest.txt 2>&1; echo "pytest rc=$?" >> $o/pytest.txt; tail -4 $o/pytest.txt
timeout 600 python bench.py --workload 64x64 --steps 200 --warmup 20 --largest none > $o/bench_64.json 2> $o/bench_64.err
python - <<'PY'
import json
d = json.loads(open("gpurun_out/small/bench_64.json").read().strip().splitlines()[-1])
print({k: d[k] for k in ("value", "ms_per_step")}, d["e2e"]["value"], d["cpu_baseline"]["time_to_solve_us"], d["roofline"].get("avg_launch_us"))
PY
