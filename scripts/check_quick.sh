#!/bin/bash
o=gpurun_out/check; mkdir -p $o
timeout 1200 python -m pytest -q -m gpu tests/test_gpu_lookahead.py -k "selection_kernel_choice or golden or klee" > $o/pytest_q.txt 2>&1; echo "pytest rc=$?" >> $o/pytest_q.txt; tail -4 $o/pytest_q.txt
