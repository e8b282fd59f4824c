#!/bin/bash
# Round-2 profile set (GPU box): ncu launch list of the default bench command, ncu --set full
# captures of the hot kernels with source, the 1000^2 pass with caches warm (L2 bytes).
# Outputs in gpurun_out/prof/ (ncu-rep files are summarised here with scripts/ncu_summary.py).
set -x
o=gpurun_out/prof
mkdir -p $o
# launch list of the bench command (cold, serialised: shares, not absolutes)
ncu --metrics gpu__time_duration.sum --clock-control none -c 3000 --csv --log-file $o/launches_8000_bench.csv \
  python bench.py --steps 1 --warmup 0 --largest none --no-cpu-baseline --single-pass-pivots 0 --roofline-pivots 64 \
  > $o/launches_bench.out 2>&1
# hot kernels, full sets with source
ncu --set full --import-source on --clock-control none -k regex:k_update_s --launch-skip 20 -c 1 \
  -o $o/pass_8000 python scripts/prof_lookahead.py 8000x8000 16 40 > $o/ncu_pass.log 2>&1
ncu --set full --import-source on --clock-control none -k regex:k_lookahead --launch-skip 20 -c 1 \
  -o $o/select_8000 python scripts/prof_lookahead.py 8000x8000 16 40 > $o/ncu_sel8.log 2>&1
ncu --set full --import-source on --clock-control none -k regex:k_lookahead --launch-skip 20 -c 1 \
  -o $o/select_4000 python scripts/prof_lookahead.py 4000x4000 16 40 > $o/ncu_sel4.log 2>&1
ncu --set full --import-source on --clock-control none -k regex:k_solve_small -c 3 \
  -o $o/small_64 python scripts/sanitize_cases.py small 64 64 48 > $o/ncu_small.log 2>&1
# 1000^2: the tableau is L2-resident, so no cache flush between launches (steady state)
ncu --set full --cache-control none --clock-control none -k regex:k_update_s --launch-skip 20 -c 3 \
  -o $o/pass_1000 python scripts/prof_lookahead.py 1000x1000 16 40 > $o/ncu_pass1000.log 2>&1
ls -la $o
