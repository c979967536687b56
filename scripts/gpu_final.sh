#!/bin/bash
# Round evidence: smoke, GPU tests, reference suite, default bench + reference
# arm, every config, the multi-rank flow, ncu launch list + full capture of the
# hot kernel. bash scripts/gpu_final.sh <tag>
TAG=${1:-final}
OUT=gpurun_out; mkdir -p $OUT
nvidia-smi > $OUT/nvidia_smi_$TAG.txt 2>&1
timeout 300 python -c "import __graft_entry__ as g; g.build(); g.smoke()" > $OUT/smoke_$TAG.log 2>&1; echo "smoke rc=$?" >> $OUT/summary_$TAG.txt
timeout 1800 python -m pytest tests -m gpu -q > $OUT/pytest_gpu_$TAG.log 2>&1; echo "pytest rc=$?" >> $OUT/summary_$TAG.txt
timeout 600 python scripts/run_reference_tests.py > $OUT/reftests_$TAG.log 2>&1; echo "reftests rc=$?" >> $OUT/summary_$TAG.txt
timeout 900 python bench.py > $OUT/bench_${TAG}_default.json 2> $OUT/bench_${TAG}_default.err; echo "bench rc=$?" >> $OUT/summary_$TAG.txt
timeout 900 python bench.py --impl reference --steps 5 --warmup 3 > $OUT/bench_ref_${TAG}.json 2> $OUT/bench_ref_${TAG}.err; echo "ref rc=$?" >> $OUT/summary_$TAG.txt
for C in cfg1 cfg3f32 cfg3f64 cfg4 cfg5; do
  timeout 900 python bench.py --config $C --steps 500 --warmup 10 --cpu-seconds 5 > $OUT/bench_${TAG}_$C.json 2> $OUT/bench_${TAG}_$C.err; echo "$C rc=$?" >> $OUT/summary_$TAG.txt
done
timeout 600 python bench.py --config cfg4 --exact --steps 100 --warmup 5 --no-cpu-baseline > $OUT/bench_${TAG}_cfg4_exact.json 2> $OUT/bench_${TAG}_cfg4_exact.err; echo "cfg4-exact rc=$?" >> $OUT/summary_$TAG.txt
timeout 900 python bench.py --dist --config cfg5 --steps 50 --warmup 5 > $OUT/bench_${TAG}_dist_cfg5.json 2> $OUT/bench_${TAG}_dist_cfg5.err; echo "dist cfg5 rc=$?" >> $OUT/summary_$TAG.txt
EHYB_DIST_BACKEND=gloo timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29541 bench.py --gpus 2 --config cfg5k4 --steps 10 --warmup 3 > $OUT/bench_${TAG}_gloo2_cfg5k4.json 2> $OUT/bench_${TAG}_gloo2_cfg5k4.err; echo "gloo2 rc=$?" >> $OUT/summary_$TAG.txt
EHYB_BENCH_PREP=host timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file $OUT/launches_${TAG}_cfg2.csv python bench.py --steps 20 --warmup 3 --no-cpu-baseline --no-cusparse > /dev/null 2> $OUT/ncu_launch_$TAG.err; echo "ncu-launches rc=$?" >> $OUT/summary_$TAG.txt
KEEP=none bash scripts/gpu_ncu.sh $TAG cfg2 cfg3f32 cfg3f64 cfg5 cfg1 cfg4 > /dev/null 2>&1; echo "ncu-full rc=$?" >> $OUT/summary_$TAG.txt
cat $OUT/summary_$TAG.txt; tail -2 $OUT/pytest_gpu_$TAG.log; tail -1 $OUT/reftests_$TAG.log
