#!/bin/bash
# early-launched selections (PDL behind the previous pass) vs the normal launch, + parity
o=gpurun_out/early; mkdir -p $o
timeout 1500 python -m pytest -x -q -m gpu tests/test_gpu_lookahead.py tests/test_gpu_parity.py tests/test_gpu_bland.py tests/test_gpu_phase1.py tests/test_gpu_pair.py > $o/pytest.txt 2>&1; echo "pytest rc=$?" >> $o/pytest.txt; tail -2 $o/pytest.txt
export SIMPLEX_EXPERIMENT_LIB=$PWD/build/libsimplex_exp.so
for w in 8000x8000 4000x4000 1000x1000; do
  for i in 1 2; do python scripts/pass_sms_sweep.py $w 4000 0 | sed "s/^/early /"; SIMPLEX_NO_EARLY_SEL=1 python scripts/pass_sms_sweep.py $w 4000 0 | sed "s/^/normal /"; done
done > $o/blocks.txt 2>&1
cat $o/blocks.txt
python bench.py --steps 20 --warmup 5 --largest none --no-cpu-baseline > $o/bench_8000.json 2> $o/bench_8000.err
cat $o/bench_8000.json | python scripts/bench_summary.py
