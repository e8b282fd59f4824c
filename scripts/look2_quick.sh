#!/bin/bash
# quick k_look2 iteration: parity of the look-ahead suites, block times 1000^2..4000^2, detail probe
o=gpurun_out/q; mkdir -p $o
timeout 900 python -m pytest -x -q -m gpu tests/test_gpu_lookahead.py tests/test_gpu_pair.py tests/test_gpu_bland.py tests/test_gpu_phase1.py > $o/pytest.txt 2>&1
echo "pytest rc=$?" >> $o/pytest.txt; tail -3 $o/pytest.txt
export SIMPLEX_EXPERIMENT_LIB=$PWD/build/libsimplex_exp.so
for w in 1000x1000 2000x2000 4000x4000 8000x8000; do python scripts/pass_sms_sweep.py $w 3000 0; done > $o/blocks.txt 2>&1
SIMPLEX_LOOK_V1=1 python scripts/pass_sms_sweep.py 8000x8000 3000 0 >> $o/blocks.txt 2>&1
cat $o/blocks.txt
export SIMPLEX_EXPERIMENT_LIB=$PWD/build/libsimplex_detail.so SIMPLEX_PROBE_DETAIL=1
for w in 4000x4000 8000x8000; do timeout 300 python scripts/sel_probe.py $w 3000 > $o/sel_$w.txt 2>&1; done
tail -n 13 $o/sel_*.txt
