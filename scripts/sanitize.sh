#!/bin/bash
# compute-sanitizer over every library path (scripts/sanitize_cases.py) at 64x64 and 1000x1000;
# logs under gpurun_out/sanitize/.  Usage: bash scripts/sanitize.sh [tools] [sizes]
out=gpurun_out/sanitize
mkdir -p $out
tools=${1:-"memcheck racecheck synccheck"}
sizes=${2:-"64 1000"}
for sz in $sizes; do
  piv=48; [ "$sz" -ge 1000 ] && piv=40
  for tool in $tools; do
    # (mblock2 — k_mblock on two virtual slabs — needs both slabs' clusters resident at once and
    #  polls the other's words; compute-sanitizer serialises kernels, so it cannot run under it:
    #  it times out as designed.  mlook3 runs the same mlook_step code one launch per pivot.)
    for case in small pass1 look16 look16serial pair32 slabs3 mlook3 phase1; do
      [ "$case" = small ] && [ "$sz" -gt 100 ] && continue
      m=$sz; n=$sz; [ "$case" = phase1 ] && [ "$sz" -ge 1000 ] && { m=300; n=400; }
      log=$out/${tool}_${case}_${sz}.log
      timeout 900 compute-sanitizer --tool $tool --print-limit 20 --error-exitcode 99 python scripts/sanitize_cases.py $case $m $n $piv > $log 2>&1
      rc=$?
      echo "$tool $case ${m}x${n}: rc=$rc $(grep -m1 -E 'ERROR SUMMARY|RACECHECK SUMMARY' $log) $(grep -m1 'sanitize case' $log)"
    done
  done
done
