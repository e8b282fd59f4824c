#!/bin/bash
# selection-phase probe + pipelined block time for each library variant in build/var_*.so
# (environment variants: VARENV="NAME=VALUE ..." applied to every run)
for so in build/var_*.so; do
  for sz in ${SIZES:-8000x8000 4000x4000}; do
    echo "== $so $sz"
    env SIMPLEX_EXPERIMENT_LIB=$so $VARENV timeout 120 python scripts/sel_probe.py $sz 3000 2>&1 | grep -v "^prologue\|complete"
    env SIMPLEX_EXPERIMENT_LIB=$so $VARENV timeout 120 python scripts/pipe_probe.py $sz 4000 2>&1 | grep "pipelined\|pass_us\|select_us"
  done
done
