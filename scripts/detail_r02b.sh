#!/bin/bash
o=gpurun_out/detail; mkdir -p $o
export SIMPLEX_EXPERIMENT_LIB=$PWD/build/libsimplex_detail.so SIMPLEX_PROBE_DETAIL=1
for w in 4000x4000 1000x1000; do timeout 300 python scripts/sel_probe.py $w 3000 > $o/sel_$w.txt 2>&1; done
cp /tmp/sx_probe.bin $o/ 2>/dev/null; tail -n 13 $o/sel_*.txt
