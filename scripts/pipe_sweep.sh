#!/bin/bash
# pipelined block time for each rank-s pass configuration (SIMPLEX_PASS_CFG) at the given size
sz=${1:-8000x8000}
for c in 0 1 2 3 4 5; do
  echo "cfg $c: $(SIMPLEX_PASS_CFG=$c timeout 120 python scripts/pipe_probe.py $sz 3000 2>&1 | tr '\n' ' ')"
done
