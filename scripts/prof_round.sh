#!/bin/bash
# Round measurement set (run on the GPU box): bench lines for every single-GPU config, the
# reference (oracle) arm, the ncu launch list of the default bench and ncu captures of its two kernels.
set -x
python bench.py > gpurun_out/bench_8000.json 2> gpurun_out/bench_8000.err
python bench.py --workload 4000x4000 --no-cpu-baseline > gpurun_out/bench_4000.json 2> gpurun_out/bench_4000.err
python bench.py --workload 1000x1000 --no-cpu-baseline > gpurun_out/bench_1000.json 2> gpurun_out/bench_1000.err
python bench.py --workload 20000x40000 --steps 1 --warmup 3 --no-cpu-baseline --roofline-pivots 1600 \
  --single-pass-pivots 200 > gpurun_out/bench_20000.json 2> gpurun_out/bench_20000.err
python bench.py --impl reference --steps 2 --warmup 3 > gpurun_out/bench_reference.json 2> gpurun_out/bench_reference.err
ncu --metrics gpu__time_duration.sum --clock-control none -c 600 --csv --log-file gpurun_out/launches_8000_pipe.csv \
  python scripts/prof_lookahead.py 8000x8000 16 300 > /dev/null 2>&1
ncu --set full --import-source on --clock-control none -k regex:k_update_s --launch-skip 20 -c 1 \
  -o gpurun_out/pipe_pass python scripts/prof_lookahead.py 8000x8000 16 40 > gpurun_out/ncu1.log 2>&1
ncu --set full --import-source on --clock-control none -k regex:k_lookahead --launch-skip 20 -c 1 \
  -o gpurun_out/pipe_select python scripts/prof_lookahead.py 8000x8000 16 40 > gpurun_out/ncu2.log 2>&1
