#!/bin/bash
# full GPU suite + smoke + bench lines (round 2b)
o=gpurun_out/check; mkdir -p $o
python -c "import __graft_entry__ as g; g.smoke()" > $o/smoke.txt 2>&1; tail -3 $o/smoke.txt
timeout 2400 python -m pytest -q -m gpu tests > $o/pytest.txt 2>&1; echo "pytest rc=$?" >> $o/pytest.txt; tail -4 $o/pytest.txt
for w in 1000x1000 4000x4000; do
  timeout 600 python bench.py --workload $w --steps 10 --warmup 3 --largest none --no-cpu-baseline > $o/bench_$w.json 2> $o/bench_$w.err
done
timeout 900 python bench.py --steps 10 --warmup 3 > $o/bench_8000.json 2> $o/bench_8000.err
timeout 600 python bench.py --workload 64x64 --steps 200 --warmup 20 --largest none > $o/bench_64.json 2> $o/bench_64.err
cat $o/bench_*.json | python scripts/bench_summary.py
