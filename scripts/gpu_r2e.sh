#!/bin/bash
TAG=${1:-r2e}
OUT=gpurun_out; mkdir -p $OUT
python -c "import __graft_entry__ as g; g.build()" > /dev/null 2>&1
S=scripts/kernel_sweep.py
for C in cfg3f32 cfg2 cfg3f64 cfg5; do
  AH=3; [ $C = cfg3f32 ] && AH=0
  V=0; [ $C = cfg3f32 ] && V=1
  timeout 900 python $S --config $C --pool 0.95 --er-cost 5.0 --er-warps 8 --pf-ell 0 --pf-er 1 --reps 300 --vec $V --ahead $AH > $OUT/exp_${TAG}_$C.jsonl 2> $OUT/exp_${TAG}_$C.err
  echo "$C rc=$?" >> $OUT/summary_${TAG}.txt
done
timeout 1800 python -m pytest tests -m gpu -q -x > $OUT/pytest_gpu_$TAG.log 2>&1; echo "pytest rc=$?" >> $OUT/summary_${TAG}.txt
bash scripts/gpu_ncu.sh $TAG
cat $OUT/summary_${TAG}.txt; tail -3 $OUT/pytest_gpu_$TAG.log
