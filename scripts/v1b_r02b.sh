#!/bin/bash
o=gpurun_out/v1b; mkdir -p $o
timeout 900 python -m pytest -x -q -m gpu tests/test_gpu_lookahead.py tests/test_gpu_parity.py -k "8000 or golden" > $o/pytest.txt 2>&1; echo "pytest rc=$?" >> $o/pytest.txt; tail -2 $o/pytest.txt
export SIMPLEX_EXPERIMENT_LIB=$PWD/build/libsimplex_exp.so
for i in 1 2 3; do python scripts/pass_sms_sweep.py 8000x8000 4000 0; done > $o/blocks.txt 2>&1
SIMPLEX_TIME_SELECT=1 python scripts/pass_sms_sweep.py 8000x8000 4000 0 >> $o/blocks.txt 2>&1
cat $o/blocks.txt
