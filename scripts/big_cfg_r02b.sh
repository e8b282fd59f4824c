#!/bin/bash
# pass ring configurations at the largest tableau (pipelined blocks), + look-ahead parity of the build
o=gpurun_out/bigcfg; mkdir -p $o
timeout 900 python -m pytest -x -q -m gpu tests/test_gpu_lookahead.py tests/test_gpu_small.py > $o/pytest.txt 2>&1; echo "pytest rc=$?" >> $o/pytest.txt; tail -2 $o/pytest.txt
export SIMPLEX_EXPERIMENT_LIB=$PWD/build/libsimplex_exp.so
for c in 0 1 2 3 4 5; do SIMPLEX_PASS_CFG=$c timeout 300 python scripts/pass_sms_sweep.py 20000x40000 1600 0 | sed "s/^/cfg$c /"; done > $o/cfg.txt 2>&1
cat $o/cfg.txt
