#!/bin/bash
# Fresh-box check of HEAD: smoke, GPU tests (incl. the reference's own suite),
# default bench, reference arm, ncu launch list. bash scripts/gpu_check.sh <tag>
TAG=${1:-check}
OUT=gpurun_out; mkdir -p $OUT
nvidia-smi > $OUT/nvidia_smi_$TAG.txt 2>&1
timeout 300 python -c "import __graft_entry__ as g; g.build(); g.smoke()" > $OUT/smoke_$TAG.log 2>&1; echo "smoke rc=$?" >> $OUT/summary_$TAG.txt
timeout 600 python scripts/run_reference_tests.py > $OUT/reftests_$TAG.log 2>&1; echo "reftests rc=$?" >> $OUT/summary_$TAG.txt
timeout 1800 python -m pytest tests -m gpu -q > $OUT/pytest_gpu_$TAG.log 2>&1; echo "pytest rc=$?" >> $OUT/summary_$TAG.txt
timeout 900 python bench.py > $OUT/bench_${TAG}_default.json 2> $OUT/bench_${TAG}_default.err; echo "bench rc=$?" >> $OUT/summary_$TAG.txt
timeout 900 python bench.py --impl reference --steps 5 --warmup 3 > $OUT/bench_ref_${TAG}.json 2> $OUT/bench_ref_${TAG}.err; echo "ref rc=$?" >> $OUT/summary_$TAG.txt
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file $OUT/launches_${TAG}_cfg2.csv python bench.py --steps 20 --warmup 3 --no-cpu-baseline --no-cusparse > /dev/null 2> $OUT/ncu_launch_$TAG.err; echo "ncu-launches rc=$?" >> $OUT/summary_$TAG.txt
cat $OUT/summary_$TAG.txt; tail -3 $OUT/pytest_gpu_$TAG.log; tail -3 $OUT/reftests_$TAG.log
