#!/bin/bash
o=gpurun_out/cfg8000; mkdir -p $o
export SIMPLEX_EXPERIMENT_LIB=$PWD/build/libsimplex_exp.so
for i in 1 2; do for c in 3 0 1 2 5; do SIMPLEX_PASS_CFG=$c timeout 300 python scripts/pass_sms_sweep.py 8000x8000 4000 0 | sed "s/^/cfg$c /"; done; done > $o/cfg.txt 2>&1
cat $o/cfg.txt
