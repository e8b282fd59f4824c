#!/bin/bash
# k_look2 check: parity suites of the look-ahead paths, selection anatomy, bench lines (v2 vs v1).
o=gpurun_out/look2; mkdir -p $o
export SIMPLEX_EXPERIMENT_LIB=$PWD/build/libsimplex_exp.so
timeout 900 python -m pytest -x -q -m gpu tests/test_gpu_lookahead.py tests/test_gpu_pair.py tests/test_gpu_bland.py tests/test_gpu_phase1.py > $o/pytest.txt 2>&1
echo "pytest rc=$?" >> $o/pytest.txt; tail -5 $o/pytest.txt
for w in 4000x4000 8000x8000 1000x1000; do
  timeout 300 python scripts/sel_probe.py $w 3000 > $o/sel_$w.txt 2>&1
done
SIMPLEX_LOOK_V1=1 timeout 300 python scripts/sel_probe.py 8000x8000 3000 > $o/sel_8000x8000_v1.txt 2>&1
timeout 600 python bench.py --workload 4000x4000 --steps 10 --warmup 3 --largest none --no-cpu-baseline > $o/bench_4000.json 2> $o/bench_4000.err
timeout 600 python bench.py --steps 10 --warmup 3 --largest none --no-cpu-baseline > $o/bench_8000.json 2> $o/bench_8000.err
timeout 600 python bench.py --workload 1000x1000 --steps 10 --warmup 3 --largest none --no-cpu-baseline > $o/bench_1000.json 2> $o/bench_1000.err
tail -n 13 $o/sel_*.txt
cat $o/bench_*.json | python scripts/bench_summary.py
for f in $o/bench_*.err; do tail -n 3 $f; done
