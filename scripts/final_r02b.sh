#!/bin/bash
# Round-2b measurement set (GPU box): smoke, bench lines for every single-GPU config and the reference
# (oracle) arm, torchrun N=1, then the ncu launch list of the default bench command and full
# captures (with source) of the hot kernels.  Outputs in gpurun_out/final3/.
o=gpurun_out/final3
mkdir -p $o
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm,power.draw,power.limit --format=csv > $o/smi.txt
python -c "import __graft_entry__ as g; g.smoke()" > $o/smoke.txt 2>&1; tail -3 $o/smoke.txt
python bench.py --steps 20 --warmup 5 > $o/bench_8000.json 2> $o/bench_8000.err
python bench.py --workload 4000x4000 --steps 10 --warmup 3 --largest none --no-cpu-baseline > $o/bench_4000.json 2> $o/bench_4000.err
python bench.py --workload 1000x1000 --steps 20 --warmup 5 --largest none --no-cpu-baseline > $o/bench_1000.json 2> $o/bench_1000.err
python bench.py --workload 64x64 --steps 200 --warmup 20 --largest none > $o/bench_64.json 2> $o/bench_64.err
python bench.py --workload 20000x40000 --steps 1 --warmup 3 --no-cpu-baseline --roofline-pivots 1600 \
  --single-pass-pivots 200 --largest none > $o/bench_20000.json 2> $o/bench_20000.err
python bench.py --impl reference --steps 2 --warmup 1 > $o/bench_reference.json 2> $o/bench_reference.err
python -m torch.distributed.run --nnodes=1 --nproc-per-node 1 --master-addr 127.0.0.1 --master-port 29533 \
  bench.py --gpus 1 --steps 3 --warmup 3 --largest none --no-cpu-baseline > $o/bench_8000_torchrun1.json 2> $o/bench_8000_torchrun1.err
cat $o/bench_*.json | python scripts/bench_summary.py
# launch list of the bench command (cold, serialised: shares, not absolutes)
ncu --metrics gpu__time_duration.sum --clock-control none -c 3000 --csv --log-file $o/launches_8000_bench.csv \
  python bench.py --steps 1 --warmup 0 --largest none --no-cpu-baseline --single-pass-pivots 0 --roofline-pivots 64 \
  > $o/launches_bench.out 2>&1
ncu --metrics gpu__time_duration.sum --clock-control none -c 3000 --csv --log-file $o/launches_4000_bench.csv \
  python bench.py --workload 4000x4000 --steps 1 --warmup 0 --largest none --no-cpu-baseline --single-pass-pivots 0 --roofline-pivots 64 \
  > $o/launches_bench4.out 2>&1
# hot kernels, full sets with source
ncu --set full --import-source on --clock-control none -k regex:k_update_s --launch-skip 20 -c 1 \
  -o $o/pass_8000 python scripts/prof_lookahead.py 8000x8000 16 40 > $o/ncu_pass.log 2>&1
ncu --set full --import-source on --clock-control none -k regex:k_lookahead --launch-skip 20 -c 1 \
  -o $o/select_8000 python scripts/prof_lookahead.py 8000x8000 16 40 > $o/ncu_sel8.log 2>&1
ncu --set full --import-source on --clock-control none -k regex:k_look2 --launch-skip 20 -c 1 \
  -o $o/select_4000 python scripts/prof_lookahead.py 4000x4000 16 40 > $o/ncu_sel4.log 2>&1
ncu --set full --import-source on --clock-control none -k regex:k_update_s --launch-skip 20 -c 1 \
  -o $o/pass_4000 python scripts/prof_lookahead.py 4000x4000 16 40 > $o/ncu_pass4.log 2>&1
ncu --set full --import-source on --clock-control none -k regex:k_solve_small -c 3 \
  -o $o/small_64 python -c "
import sys; sys.path.insert(0, '.')
import lpgen, paper_2211_10979_b200 as sx
A, b, c = lpgen.dense_lp(64, 64, 1)
with sx.Simplex(A, b, c) as s:
    for _ in range(3): s.solve_lp(A, b, c)
" > $o/ncu_small.log 2>&1
# summaries here (the reports themselves exceed gpurun's 64 MiB copy-back limit): keep the two
# hottest-kernel reports, summarise every report and launch list
for r in pass_8000 select_8000 select_4000 pass_4000 small_64; do
  python scripts/ncu_summary.py rep $o/$r.ncu-rep $r > $o/ncu_$r.json 2>&1
  python scripts/ncu_hotspots.py $o/$r.ncu-rep 40 > $o/hot_$r.txt 2>&1
done
python scripts/ncu_summary.py launches $o/launches_8000_bench.csv > $o/launch_share_8000.json 2>&1
python scripts/ncu_summary.py launches $o/launches_4000_bench.csv > $o/launch_share_4000.json 2>&1
rm -f $o/select_8000.ncu-rep $o/pass_4000.ncu-rep $o/small_64.ncu-rep
gzip -f $o/launches_*.csv
ls -la $o
du -sh $o
