#!/bin/bash
TAG=${1:-r2c}
OUT=gpurun_out; mkdir -p $OUT
python -c "import __graft_entry__ as g; g.build()" > /dev/null 2>&1
for C in cfg2 cfg3f32; do for V in 0 1; do
  timeout 600 python scripts/cta_balance.py --config $C --vec $V > $OUT/cta_balance_${TAG}_${C}_v$V.json 2> $OUT/cta_balance_${TAG}_${C}_v$V.err
done; done
bash scripts/sanitize.sh $TAG
timeout 1800 python -m pytest tests -m gpu -q > $OUT/pytest_gpu_$TAG.log 2>&1; echo "pytest rc=$?" >> $OUT/summary_$TAG.txt
cat $OUT/summary_$TAG.txt; tail -3 $OUT/pytest_gpu_$TAG.log
