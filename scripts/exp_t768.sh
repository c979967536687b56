#!/bin/bash
TAG=${1:-t768}
OUT=gpurun_out; mkdir -p $OUT
S=scripts/kernel_sweep.py
for T in 768; do
  export EHYB_NVCC_FLAGS="-DEHYB_MAX_THREADS=$T"; export EHYB_THREADS=$T
  python paper_2204_06666_b200/build.py > $OUT/exp_${TAG}_build.log 2>&1
  for C in cfg3f32 cfg2 cfg3f64 cfg5; do
    AH=3; [ $C = cfg3f32 ] && AH=0,3
    timeout 900 python $S --config $C --pool 0.95 --er-cost 5.0 --er-warps 4,6,8 --pf-ell 0 --pf-er 1 --reps 300 --vec 0,1 --ahead $AH > $OUT/exp_${TAG}_$C.jsonl 2> $OUT/exp_${TAG}_$C.err
    echo "$T $C rc=$?" >> $OUT/exp_${TAG}_summary.txt
  done
done
cat $OUT/exp_${TAG}_summary.txt
