#!/bin/bash
TAG=${1:-heavy}
OUT=gpurun_out; mkdir -p $OUT
python -c "import __graft_entry__ as g; g.build()" > /dev/null 2>&1
S=scripts/kernel_sweep.py
for H in 0 1.0 1.01 1.03; do
for C in cfg2 cfg3f32; do
  AH=3; [ $C = cfg3f32 ] && AH=0
  EHYB_POOL_HEAVY=$H timeout 900 python $S --config $C --pool 0.9,0.95,1.0 --er-cost 5.0 --er-warps 8 --pf-ell 0 --pf-er 1 --reps 300 --vec 1 --ahead $AH > $OUT/exp_${TAG}_h${H}_$C.jsonl 2> $OUT/exp_${TAG}_h${H}_$C.err
  echo "h $H $C rc=$?" >> $OUT/exp_${TAG}_summary.txt
done; done
timeout 600 python bench.py --config cfg1 --steps 500 --warmup 10 --no-cpu-baseline > $OUT/exp_${TAG}_cfg1.json 2> $OUT/exp_${TAG}_cfg1.err
cat $OUT/exp_${TAG}_summary.txt
