#!/bin/bash
# pipelined block time at 4000^2 / 2000^2 vs pass SMs and ring config, k_look2 (and k_lookahead for reference)
o=gpurun_out/sweep; mkdir -p $o
export SIMPLEX_EXPERIMENT_LIB=$PWD/build/libsimplex_exp.so
for w in 4000x4000 2000x2000; do
  python scripts/pass_sms_sweep.py $w 3000 0,112,96,80,64 > $o/sms_$w.txt 2>&1
  for c in 0 3 4 5; do SIMPLEX_PASS_CFG=$c python scripts/pass_sms_sweep.py $w 3000 0 | sed "s/^/cfg$c /"; done > $o/cfg_$w.txt 2>&1
  SIMPLEX_LOOK_V1=1 python scripts/pass_sms_sweep.py $w 3000 0,96 > $o/v1_$w.txt 2>&1
done
tail -n 20 $o/*.txt
