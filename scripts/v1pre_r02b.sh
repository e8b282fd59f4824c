#!/bin/bash
o=gpurun_out/v1pre; mkdir -p $o
timeout 900 python -m pytest -x -q -m gpu tests/test_gpu_lookahead.py tests/test_gpu_pair.py tests/test_gpu_bland.py tests/test_gpu_phase1.py -k "8000 or 4000 or golden or klee or selection_kernel or phase1 or bland" > $o/pytest.txt 2>&1; echo "pytest rc=$?" >> $o/pytest.txt; tail -3 $o/pytest.txt
export SIMPLEX_EXPERIMENT_LIB=$PWD/build/libsimplex_exp.so
for i in 1 2; do python scripts/pass_sms_sweep.py 8000x8000 3000 0; done > $o/blocks.txt 2>&1
cat $o/blocks.txt
timeout 300 python scripts/sel_probe.py 8000x8000 3000 > $o/sel_8000.txt 2>&1; tail -13 $o/sel_8000.txt
timeout 900 python bench.py --steps 10 --warmup 3 --largest none --no-cpu-baseline > $o/bench_8000.json 2> $o/bench_8000.err
cat $o/bench_8000.json | python scripts/bench_summary.py
