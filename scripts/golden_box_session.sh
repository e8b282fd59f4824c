#!/bin/bash
# One ≤ 1-hour gpurun session of the 20000x40000 full-solve golden (scripts/make_golden_long.py):
# resumes from the checkpoint in /tmp on the box when the same box is reused (back-to-back calls),
# runs ~55 minutes on all host cores, checkpoints and pauses.  Goldens reached and the progress go
# to gpurun_out/golden/.  Calls only oracle/ and lpgen/.
export GOLDEN_OUT=gpurun_out/golden OMP_NUM_THREADS=$(nproc)
mkdir -p $GOLDEN_OUT
{ date; nproc; df -h /tmp | tail -1; ls -la /tmp/golden_ckpt_box 2>/dev/null; } > $GOLDEN_OUT/session_$(date +%s).txt
python -c "import oracle; oracle.build(parallel=True)" 
python scripts/make_golden_long.py 20000 40000 1 --chunk 512 --ckpt /tmp/golden_ckpt_box --ckpt-every 0 \
  --max-seconds ${MAX_SECONDS:-3150} --milestones 32768,65536,100000,120000 >> $GOLDEN_OUT/golden_long.log 2>&1
echo "exit $?" >> $GOLDEN_OUT/golden_long.log
tail -6 $GOLDEN_OUT/golden_long.log
cat $GOLDEN_OUT/dense_20000x40000_s1_progress.json
