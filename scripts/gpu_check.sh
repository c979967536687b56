#!/bin/bash
# Fresh-box check of HEAD: smoke, GPU tests, default bench. bash scripts/gpu_check.sh <tag>
TAG=${1:-check}
OUT=gpurun_out; mkdir -p $OUT
timeout 300 python -c "import __graft_entry__ as g; g.build(); g.smoke()" > $OUT/smoke_$TAG.log 2>&1; echo "smoke rc=$?" >> $OUT/summary_$TAG.txt
timeout 1500 python -m pytest tests -m gpu -x -q > $OUT/pytest_gpu_$TAG.log 2>&1; echo "pytest rc=$?" >> $OUT/summary_$TAG.txt
timeout 900 python bench.py > $OUT/bench_${TAG}_default.json 2> $OUT/bench_${TAG}_default.err; echo "bench rc=$?" >> $OUT/summary_$TAG.txt
cat $OUT/summary_$TAG.txt; tail -3 $OUT/pytest_gpu_$TAG.log
