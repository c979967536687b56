#!/bin/bash
TAG=${1:-r2f}
OUT=gpurun_out; mkdir -p $OUT
python -c "import __graft_entry__ as g; g.build(); g.smoke()" > $OUT/smoke_$TAG.log 2>&1; echo "smoke rc=$?" >> $OUT/summary_$TAG.txt
timeout 1800 python -m pytest tests -m gpu -q > $OUT/pytest_gpu_$TAG.log 2>&1; echo "pytest rc=$?" >> $OUT/summary_$TAG.txt
timeout 900 python bench.py > $OUT/bench_${TAG}_default.json 2> $OUT/bench_${TAG}_default.err; echo "bench rc=$?" >> $OUT/summary_$TAG.txt
for C in cfg3f32 cfg3f64 cfg5; do
  timeout 900 python bench.py --config $C --steps 300 --warmup 10 --cpu-seconds 5 > $OUT/bench_${TAG}_$C.json 2> $OUT/bench_${TAG}_$C.err; echo "$C rc=$?" >> $OUT/summary_$TAG.txt
done
cat $OUT/summary_$TAG.txt; tail -3 $OUT/pytest_gpu_$TAG.log
