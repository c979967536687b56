#!/bin/bash
TAG=${1:-f896}
OUT=gpurun_out; mkdir -p $OUT
S=scripts/kernel_sweep.py
for T in 896 1024; do
  export EHYB_NVCC_FLAGS="-DEHYB_MAX_THREADS_F32=$T"
  python paper_2204_06666_b200/build.py > $OUT/exp_${TAG}_build_$T.log 2>&1
  timeout 900 python $S --config cfg3f32 --pool 0.85,0.9 --er-cost 5.0 --er-warps 6,7,8 --pf-ell 0 --pf-er 1 --reps 300 --vec 1 --ahead 0 --phases > $OUT/exp_${TAG}_t${T}_cfg3f32.jsonl 2> $OUT/exp_${TAG}_t${T}.err
  echo "$T rc=$?" >> $OUT/exp_${TAG}_summary.txt
done
cat $OUT/exp_${TAG}_summary.txt
