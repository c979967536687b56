#!/bin/bash
# Round evidence: smoke, GPU tests, default bench + reference arm, every
# config, ncu launch list + full capture of the hot kernel. bash scripts/gpu_final.sh <tag>
TAG=${1:-final}
OUT=gpurun_out; mkdir -p $OUT
nvidia-smi > $OUT/nvidia_smi_$TAG.txt 2>&1
timeout 300 python -c "import __graft_entry__ as g; g.build(); g.smoke()" > $OUT/smoke_$TAG.log 2>&1; echo "smoke rc=$?" >> $OUT/summary_$TAG.txt
timeout 1500 python -m pytest tests -m gpu -x -q > $OUT/pytest_gpu_$TAG.log 2>&1; echo "pytest rc=$?" >> $OUT/summary_$TAG.txt
timeout 900 python bench.py > $OUT/bench_${TAG}_default.json 2> $OUT/bench_${TAG}_default.err; echo "bench rc=$?" >> $OUT/summary_$TAG.txt
timeout 900 python bench.py --impl reference --steps 5 --warmup 3 > $OUT/bench_ref_${TAG}.json 2> $OUT/bench_ref_${TAG}.err; echo "ref rc=$?" >> $OUT/summary_$TAG.txt
for C in cfg1 cfg3f32 cfg3f64 cfg4 cfg5; do
  timeout 900 python bench.py --config $C --steps 500 --warmup 10 --cpu-seconds 5 > $OUT/bench_${TAG}_$C.json 2> $OUT/bench_${TAG}_$C.err; echo "$C rc=$?" >> $OUT/summary_$TAG.txt
done
timeout 600 python bench.py --config cfg4 --fma --steps 500 --warmup 10 --no-cpu-baseline > $OUT/bench_${TAG}_cfg4_fma.json 2> $OUT/bench_${TAG}_cfg4_fma.err; echo "cfg4-fma rc=$?" >> $OUT/summary_$TAG.txt
timeout 900 python bench.py --dist --steps 300 --warmup 10 > $OUT/bench_${TAG}_dist.json 2> $OUT/bench_${TAG}_dist.err; echo "dist rc=$?" >> $OUT/summary_$TAG.txt
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file $OUT/launches_${TAG}_cfg2.csv python bench.py --steps 20 --warmup 3 --no-cpu-baseline --no-cusparse > /dev/null 2> $OUT/ncu_launch_$TAG.err; echo "ncu-launches rc=$?" >> $OUT/summary_$TAG.txt
timeout 900 ncu --set full --clock-control none --import-source on -k regex:spmv_fused -s 5 -c 1 -o $OUT/prof_${TAG}_cfg2 python bench.py --steps 8 --warmup 3 --no-cpu-baseline --no-cusparse > /dev/null 2> $OUT/ncu_full_$TAG.err; echo "ncu-full cfg2 rc=$?" >> $OUT/summary_$TAG.txt
timeout 900 ncu --set full --clock-control none --import-source on -k regex:spmv_fused -s 5 -c 1 -o $OUT/prof_${TAG}_cfg3f32 python bench.py --config cfg3f32 --steps 8 --warmup 3 --no-cpu-baseline --no-cusparse > /dev/null 2> $OUT/ncu_full3_$TAG.err; echo "ncu-full cfg3f32 rc=$?" >> $OUT/summary_$TAG.txt
cat $OUT/summary_$TAG.txt
