#!/bin/bash
# Experiment: ER-first warps x ELL layout x combine batch. bash scripts/exp_erw.sh <tag>
TAG=${1:-erw}
OUT=gpurun_out; mkdir -p $OUT
S=scripts/kernel_sweep.py
COMMON="--pool 0.95 --er-cost 5.0 --er-warps 8,12,16 --pf-ell 0 --pf-er 1 --reps 300 --vec 0,1"
for B in 1 4; do
  export EHYB_NVCC_FLAGS="-DEHYB_COMB_BATCH=$B"
  python paper_2204_06666_b200/build.py > $OUT/exp_${TAG}_build_$B.log 2>&1
  for C in cfg3f32 cfg2 cfg3f64; do
    AH=3; [ $C = cfg3f32 ] && AH=0,3
    timeout 900 python $S --config $C $COMMON --ahead $AH > $OUT/exp_${TAG}_b${B}_$C.jsonl 2> $OUT/exp_${TAG}_b${B}_$C.err
    echo "b$B $C rc=$?" >> $OUT/exp_${TAG}_summary.txt
  done
done
cat $OUT/exp_${TAG}_summary.txt
