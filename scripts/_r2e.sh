OUT=gpurun_out; TAG=r2e
python -c "import __graft_entry__ as g; g.build()" > $OUT/build_$TAG.log 2>&1
timeout 900 python bench.py --config cfg3f32 --steps 500 --warmup 10 --cpu-seconds 5 > $OUT/bench_${TAG}_cfg3f32.json 2> $OUT/bench_${TAG}_cfg3f32.err; echo "cfg3f32 rc=$?"
timeout 900 ncu --set full --clock-control none --import-source on -k regex:spmv_fused -s 5 -c 1 -o $OUT/prof_${TAG}_cfg3f32 python bench.py --config cfg3f32 --steps 8 --warmup 3 --no-cpu-baseline --no-cusparse > /dev/null 2> $OUT/ncu_full3_$TAG.err; echo "ncu rc=$?"
