#!/bin/bash
# r2b: GPU tests (hybrid mode), reference suite, sanitizer, cfg2 default bench,
# cfg4 in the three modes. bash scripts/gpu_r2b.sh <tag>
TAG=${1:-r2b}
OUT=gpurun_out; mkdir -p $OUT
python -c "import __graft_entry__ as g; g.build(); g.smoke()" > $OUT/smoke_$TAG.log 2>&1; echo "smoke rc=$?" >> $OUT/summary_$TAG.txt
timeout 600 python scripts/run_reference_tests.py > $OUT/reftests_$TAG.log 2>&1; echo "reftests rc=$?" >> $OUT/summary_$TAG.txt
timeout 1800 python -m pytest tests -m gpu -q -x > $OUT/pytest_gpu_$TAG.log 2>&1; echo "pytest rc=$?" >> $OUT/summary_$TAG.txt
timeout 600 python bench.py --steps 500 --warmup 10 --no-cpu-baseline > $OUT/bench_${TAG}_cfg2.json 2> $OUT/bench_${TAG}_cfg2.err; echo "bench cfg2 rc=$?" >> $OUT/summary_$TAG.txt
timeout 900 python bench.py --config cfg4 --steps 500 --warmup 10 --cpu-seconds 3 > $OUT/bench_${TAG}_cfg4.json 2> $OUT/bench_${TAG}_cfg4.err; echo "bench cfg4 rc=$?" >> $OUT/summary_$TAG.txt
bash scripts/sanitize.sh $TAG
cat $OUT/summary_$TAG.txt; tail -3 $OUT/pytest_gpu_$TAG.log; tail -2 $OUT/reftests_$TAG.log
