#!/bin/bash
# build-level A/B on the box: bash scripts/ab_libs.sh <tag> "<ab_env args>" libA.so libB.so ...
TAG=$1; ARGS="$2"; shift 2
OUT=gpurun_out; mkdir -p $OUT
cp paper_2204_06666_b200/libehyb_b200.so /tmp/lib_orig.so
for R in 1 2; do
for L in "$@"; do
  cp $L paper_2204_06666_b200/libehyb_b200.so
  echo "== $L round $R" >> $OUT/ab_${TAG}.txt
  python scripts/ab_env.py $ARGS >> $OUT/ab_${TAG}.txt 2>> $OUT/ab_${TAG}.err
done
done
cp /tmp/lib_orig.so paper_2204_06666_b200/libehyb_b200.so
cat $OUT/ab_${TAG}.txt
