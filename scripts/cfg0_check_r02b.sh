#!/bin/bash
# the {4,12} pass at 8000^2: parity (goldens on the default path), bench line, ncu of the pass
o=gpurun_out/cfg0; mkdir -p $o
timeout 1200 python -m pytest -x -q -m gpu tests/test_gpu_parity.py tests/test_gpu_lookahead.py -k "8000 or golden" > $o/pytest.txt 2>&1; echo "pytest rc=$?" >> $o/pytest.txt; tail -2 $o/pytest.txt
python bench.py --steps 20 --warmup 5 --largest none --no-cpu-baseline > $o/bench_8000.json 2> $o/bench_8000.err
cat $o/bench_8000.json | python scripts/bench_summary.py
ncu --set full --import-source on --clock-control none -k regex:k_update_s --launch-skip 20 -c 1 \
  -o $o/pass_8000 python scripts/prof_lookahead.py 8000x8000 16 40 > $o/ncu_pass.log 2>&1
python scripts/ncu_summary.py rep $o/pass_8000.ncu-rep pass_8000_cfg0 > $o/ncu_pass_8000.json 2>&1
python scripts/ncu_hotspots.py $o/pass_8000.ncu-rep 30 > $o/hot_pass_8000.txt 2>&1
rm -f $o/pass_8000.ncu-rep
python - <<'PY'
import json
d = json.load(open("gpurun_out/cfg0/ncu_pass_8000.json"))
l = d["launches"][0]
print(l["kernel"][:50], l["gpu__time_duration.sum"], l["dram__bytes_read.sum"], l["dram__bytes_write.sum"])
PY
