#!/bin/bash
# Experiment: 128-bit interleaved ELL stream (tail merged into the last batch)
# vs the SELL scalar stream, per config; then UB variants. bash scripts/exp_vec.sh <tag>
TAG=${1:-vec}
OUT=gpurun_out; mkdir -p $OUT
S=scripts/kernel_sweep.py
COMMON="--pool 0.95 --er-cost 5.0 --er-warps 8 --pf-ell 0 --pf-er 1 --vec 0,1 --reps 300"
python -c "import __graft_entry__ as g; g.build()" > $OUT/exp_${TAG}_build.log 2>&1
for C in cfg3f32 cfg2 cfg3f64 cfg5; do
  AH=3; [ $C = cfg3f32 ] && AH=0
  timeout 600 python $S --config $C $COMMON --ahead $AH > $OUT/exp_${TAG}_$C.jsonl 2> $OUT/exp_${TAG}_$C.err
  echo "$C rc=$?" >> $OUT/exp_${TAG}_summary.txt
done
export EHYB_NVCC_FLAGS="-DEHYB_VEC_UB_F64=3 -DEHYB_VEC_UB_F32=5"
python paper_2204_06666_b200/build.py >> $OUT/exp_${TAG}_build.log 2>&1
for C in cfg3f32 cfg2 cfg3f64; do
  AH=3; [ $C = cfg3f32 ] && AH=0
  timeout 600 python $S --config $C $COMMON --ahead $AH > $OUT/exp_${TAG}_ub_$C.jsonl 2> $OUT/exp_${TAG}_ub_$C.err
  echo "ub $C rc=$?" >> $OUT/exp_${TAG}_summary.txt
done
cat $OUT/exp_${TAG}_summary.txt
