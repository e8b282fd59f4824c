#!/bin/bash
o=gpurun_out/l512; mkdir -p $o
timeout 900 python -m pytest -x -q -m gpu tests/test_gpu_lookahead.py -k "golden or selection_kernel or klee or tie or seeds" > $o/pytest.txt 2>&1; echo "pytest rc=$?" >> $o/pytest.txt; tail -2 $o/pytest.txt
export SIMPLEX_EXPERIMENT_LIB=$PWD/build/libsimplex_exp.so
for w in 3000x3000 4000x4000 4000x3000; do
  for i in 1 2; do python scripts/pass_sms_sweep.py $w 3000 0 | sed "s/^/512 /"; SIMPLEX_LOOK2_NO512=1 python scripts/pass_sms_sweep.py $w 3000 0 | sed "s/^/256 /"; done
done > $o/blocks.txt 2>&1
cat $o/blocks.txt
