#!/bin/bash
TAG=${1:-plast}
OUT=gpurun_out; mkdir -p $OUT
python -c "import __graft_entry__ as g; g.build()" > /dev/null 2>&1
S=scripts/kernel_sweep.py
for PL in 1 0; do
for C in cfg3f64 cfg5; do
  EHYB_POOL_LAST=$PL timeout 900 python $S --config $C --pool 0.9,1.0 --er-cost 5.0 --er-warps 6 --pf-ell 0 --pf-er 1 --reps 200 --vec 0 --ahead 3 > $OUT/exp_${TAG}_p${PL}_$C.jsonl 2> $OUT/exp_${TAG}_p${PL}_$C.err
done; done
for LS in 1; do
for C in cfg3f64 cfg5; do
  EHYB_POOL_LAST_SCRATCH=$LS timeout 900 python $S --config $C --pool 0.9 --er-cost 5.0 --er-warps 6 --pf-ell 0 --pf-er 1 --reps 200 --vec 0 --ahead 3 > $OUT/exp_${TAG}_ls${LS}_$C.jsonl 2> $OUT/exp_${TAG}_ls${LS}_$C.err
done; done
echo done
