#!/bin/bash
# L2 policy of the rank-16 pass vs pipelined block time (does keeping the last-written tableau in L2
# shorten the selection's column reads?)
o=gpurun_out/l2pol; mkdir -p $o
export SIMPLEX_EXPERIMENT_LIB=$PWD/build/libsimplex_exp.so
for w in 1000x1000 2000x2000 3000x3000 4000x4000; do
  for m in 0 1 2; do SIMPLEX_PASS_L2=$m timeout 300 python scripts/pass_sms_sweep.py $w 3000 0 | sed "s/^/l2mode$m /"; done
done > $o/l2.txt 2>&1
cat $o/l2.txt
