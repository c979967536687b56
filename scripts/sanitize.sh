#!/bin/bash
# compute-sanitizer over the fused kernel's protocols (scripts/sanitize_cases.py):
# memcheck, racecheck (shared memory), synccheck, initcheck. bash scripts/sanitize.sh <tag>
TAG=${1:-san}
OUT=gpurun_out; mkdir -p $OUT
CS=/usr/local/cuda/bin/compute-sanitizer
for TOOL in memcheck racecheck synccheck initcheck; do
  EXTRA=""
  [ $TOOL = racecheck ] && EXTRA="--racecheck-report analysis"
  [ $TOOL = initcheck ] && EXTRA=""
  timeout 1200 $CS --tool $TOOL $EXTRA --print-limit 20 --error-exitcode 9 \
    python scripts/sanitize_cases.py > $OUT/sanitize_${TAG}_$TOOL.log 2>&1
  echo "$TOOL rc=$?" >> $OUT/sanitize_${TAG}_summary.txt
done
cat $OUT/sanitize_${TAG}_summary.txt
