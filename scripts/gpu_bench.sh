#!/bin/bash
# bench + ncu evidence for one tag: bash scripts/gpu_bench.sh <tag> [config]
TAG=${1:-rX}; CFG=${2:-cfg2}
OUT=gpurun_out; mkdir -p $OUT
timeout 900 python bench.py --config $CFG --steps 2000 --warmup 20 > $OUT/bench_${TAG}_${CFG}.json 2> $OUT/bench_${TAG}_${CFG}.err; echo "bench rc=$?"
timeout 600 python bench.py --impl reference --config $CFG --steps 5 --warmup 3 > $OUT/bench_ref_${TAG}_${CFG}.json 2> $OUT/bench_ref_${TAG}_${CFG}.err; echo "ref rc=$?"
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -c 200 --csv --log-file $OUT/launches_${TAG}_${CFG}.csv python bench.py --config $CFG --steps 20 --warmup 3 --no-cpu-baseline --no-cusparse > /dev/null 2> $OUT/ncu_launch_${TAG}.err; echo "ncu-launches rc=$?"
timeout 900 ncu --set full --clock-control none --import-source on -k regex:spmv_fused -s 6 -c 1 -o $OUT/prof_${TAG}_${CFG} python bench.py --config $CFG --steps 8 --warmup 3 --no-cpu-baseline --no-cusparse > /dev/null 2> $OUT/ncu_full_${TAG}.err; echo "ncu-full rc=$?"
