#!/bin/bash
TAG=${1:-own}
OUT=gpurun_out; mkdir -p $OUT
python -c "import __graft_entry__ as g; g.build()" > /dev/null 2>&1
S=scripts/kernel_sweep.py
for C in cfg3f32 cfg2 cfg3f64 cfg5; do
  AH=3; [ $C = cfg3f32 ] && AH=0
  V=0; [ $C = cfg3f32 ] && V=1; [ $C = cfg2 ] && V=1
  timeout 900 python $S --config $C --pool 0.9 --er-cost 5.0 --er-warps 6 --pf-ell 0 --pf-er 1 --reps 300 --vec $V --ahead $AH > $OUT/exp_${TAG}_$C.jsonl 2> $OUT/exp_${TAG}_$C.err
  echo "$C rc=$?" >> $OUT/exp_${TAG}_summary.txt
done
timeout 1800 python -m pytest tests -m gpu -q -x > $OUT/pytest_gpu_$TAG.log 2>&1; echo "pytest rc=$?" >> $OUT/exp_${TAG}_summary.txt
cat $OUT/exp_${TAG}_summary.txt; tail -2 $OUT/pytest_gpu_$TAG.log
