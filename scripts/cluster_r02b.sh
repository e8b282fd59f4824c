#!/bin/bash
o=gpurun_out/cluster; mkdir -p $o
export SIMPLEX_EXPERIMENT_LIB=$PWD/build/libsimplex_exp.so
for w in 1000x1000 2000x2000 500x500; do
  for c in 16 8 4; do SIMPLEX_LOOK_CLUSTER=$c timeout 300 python scripts/pass_sms_sweep.py $w 3000 0 | sed "s/^/cluster$c /"; done
done > $o/cl.txt 2>&1
cat $o/cl.txt
