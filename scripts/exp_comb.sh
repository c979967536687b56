#!/bin/bash
# Experiment: combine / pooled-sum batch size (EHYB_COMB_BATCH) x ELL layout,
# with ELL-alone / ER-alone phase times. bash scripts/exp_comb.sh <tag>
TAG=${1:-comb}
OUT=gpurun_out; mkdir -p $OUT
S=scripts/kernel_sweep.py
COMMON="--pool 0.95 --er-cost 5.0 --er-warps 8 --pf-ell 0 --pf-er 1 --reps 300 --phases"
for B in 4 1; do
  export EHYB_NVCC_FLAGS="-DEHYB_COMB_BATCH=$B"
  python paper_2204_06666_b200/build.py > $OUT/exp_${TAG}_build_$B.log 2>&1
  for C in cfg3f32 cfg2 cfg3f64; do
    AH=3; [ $C = cfg3f32 ] && AH=0
    timeout 600 python $S --config $C $COMMON --vec 0,1 --ahead $AH > $OUT/exp_${TAG}_b${B}_$C.jsonl 2> $OUT/exp_${TAG}_b${B}_$C.err
    echo "b$B $C rc=$?" >> $OUT/exp_${TAG}_summary.txt
  done
done
cat $OUT/exp_${TAG}_summary.txt
