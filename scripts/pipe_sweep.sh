#!/bin/bash
# pipelined block time for each rank-s pass configuration (SIMPLEX_PASS_CFG), 8000^2
for c in 0 1 2 3 4 5; do
  echo "cfg $c: $(SIMPLEX_PASS_CFG=$c timeout 120 python scripts/pipe_probe.py 8000x8000 3000 2>&1 | tr '\n' ' ')"
done
