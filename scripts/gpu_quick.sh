#!/bin/bash
# GPU tests + short benches: bash scripts/gpu_quick.sh <tag> "<pytest -k expr or empty>" cfgs...
TAG=$1; K="$2"; shift 2
OUT=gpurun_out; mkdir -p $OUT
python -c "import __graft_entry__ as g; g.build()" > $OUT/build_$TAG.log 2>&1
if [ -n "$K" ]; then
  timeout 1500 python -m pytest tests -m gpu -x -q -k "$K" > $OUT/pytest_$TAG.log 2>&1; echo "pytest rc=$?" >> $OUT/summary_$TAG.txt
fi
for C in "$@"; do
  timeout 900 python bench.py --config $C --steps 300 --warmup 10 --no-cpu-baseline > $OUT/bench_${TAG}_${C}.json 2> $OUT/bench_${TAG}_${C}.err
  echo "$C rc=$?" >> $OUT/summary_$TAG.txt
done
cat $OUT/summary_$TAG.txt
