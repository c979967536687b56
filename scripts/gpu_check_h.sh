#!/bin/bash
# HEAD check without rebuilding (the .so files travel): smoke, GPU tests, every config
TAG=${1:-h}; OUT=gpurun_out; mkdir -p $OUT
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > $OUT/smoke_$TAG.log 2>&1; echo "smoke rc=$?" >> $OUT/summary_$TAG.txt
timeout 1800 python -m pytest tests -m gpu -q -x > $OUT/pytest_gpu_$TAG.log 2>&1; echo "pytest rc=$?" >> $OUT/summary_$TAG.txt
for C in cfg2 cfg1 cfg3f32 cfg3f64 cfg4 cfg5; do
  timeout 900 python bench.py --config $C --steps 300 --warmup 10 --no-cpu-baseline > $OUT/bench_${TAG}_$C.json 2> $OUT/bench_${TAG}_$C.err; echo "$C rc=$?" >> $OUT/summary_$TAG.txt
done
cat $OUT/summary_$TAG.txt; tail -2 $OUT/pytest_gpu_$TAG.log
