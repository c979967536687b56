#!/bin/bash
# Bench every BASELINE config on one GPU: bash scripts/gpu_configs.sh <tag> [configs...]
TAG=${1:-rX}; shift
CFGS=${@:-cfg2 cfg1 cfg3f32 cfg3f64 cfg4 cfg5}
OUT=gpurun_out; mkdir -p $OUT
nproc > $OUT/host_$TAG.txt; free -g >> $OUT/host_$TAG.txt
python -c "import __graft_entry__ as g; g.build()"
timeout 600 python -m pytest tests/test_gpu_spmv.py -x -q -k host_many > $OUT/pytest_many_$TAG.log 2>&1; echo "pytest-many rc=$?" >> $OUT/summary_cfg_$TAG.txt
for C in $CFGS; do
  timeout 900 python bench.py --config $C --steps 500 --warmup 10 --cpu-seconds 5 > $OUT/bench_${TAG}_${C}.json 2> $OUT/bench_${TAG}_${C}.err
  echo "$C rc=$?" >> $OUT/summary_cfg_$TAG.txt
done
cat $OUT/summary_cfg_$TAG.txt
