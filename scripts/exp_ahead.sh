#!/bin/bash
TAG=${1:-ahead}
OUT=gpurun_out; mkdir -p $OUT
python -c "import __graft_entry__ as g; g.build()" > /dev/null 2>&1
S=scripts/kernel_sweep.py
timeout 900 python $S --config cfg3f32 --pool 0.9 --er-cost 5.0 --er-warps 6,8 --pf-ell 0 --pf-er 0,1 --reps 300 --vec 1 --ahead 0,1,2,3 > $OUT/exp_${TAG}_cfg3f32.jsonl 2> $OUT/exp_${TAG}_cfg3f32.err
timeout 900 python $S --config cfg2 --pool 0.9 --er-cost 5.0 --er-warps 6,8 --pf-ell 0 --pf-er 0,1 --reps 300 --vec 1 --ahead 1,3 > $OUT/exp_${TAG}_cfg2.jsonl 2> $OUT/exp_${TAG}_cfg2.err
timeout 900 python $S --config cfg3f64 --pool 0.9 --er-cost 5.0 --er-warps 6,8 --pf-ell 0 --pf-er 1 --reps 300 --vec 0 --ahead 1,3 > $OUT/exp_${TAG}_cfg3f64.jsonl 2> $OUT/exp_${TAG}_cfg3f64.err
timeout 900 python $S --config cfg5 --pool 0.9 --er-cost 5.0 --er-warps 6,8 --pf-ell 0 --pf-er 1 --reps 100 --vec 0 --ahead 1,3 > $OUT/exp_${TAG}_cfg5.jsonl 2> $OUT/exp_${TAG}_cfg5.err
echo done
