#!/bin/bash
# ncu source-level capture of one pipelined selection launch (k_look2) at 4000^2 and 8000^2.
o=gpurun_out/ncu_look2; mkdir -p $o
for w in 4000x4000 1000x1000; do
  timeout 600 ncu --set full --import-source on --clock-control none -k regex:k_look -s 20 -c 1 \
    -o $o/look2_$w python scripts/prof_lookahead.py $w 16 24 > $o/ncu_$w.log 2>&1
  python scripts/ncu_hotspots.py $o/look2_$w.ncu-rep 40 > $o/hot_$w.txt 2>&1
done
tail -3 $o/ncu_*.log; for f in $o/hot_*.txt; do echo $f; head -40 $f | cut -c1-240; done
