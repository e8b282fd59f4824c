#!/bin/bash
# Round-2b session probe: fine-grained selection anatomy (experiment build) + baseline bench lines.
o=gpurun_out/probe; mkdir -p $o
export SIMPLEX_EXPERIMENT_LIB=$PWD/build/libsimplex_exp.so
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm,power.draw --format=csv > $o/smi.txt
for w in 4000x4000 8000x8000 1000x1000; do
  timeout 300 python scripts/sel_probe.py $w 3000 > $o/sel_$w.txt 2>&1
  timeout 300 python scripts/sel_probe.py $w 3000 --serial > $o/sel_${w}_serial.txt 2>&1
done
timeout 600 python bench.py --workload 4000x4000 --steps 10 --warmup 3 --largest none --no-cpu-baseline > $o/bench_4000.json 2> $o/bench_4000.err
timeout 600 python bench.py --steps 10 --warmup 3 --largest none --no-cpu-baseline > $o/bench_8000.json 2> $o/bench_8000.err
tail -n 14 $o/sel_*.txt
cat $o/bench_*.json | python scripts/bench_summary.py
