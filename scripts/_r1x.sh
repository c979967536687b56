python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build_r1x.log 2>&1
timeout 900 python -m pytest tests -m gpu -x -q -k "shards or host_many or cg" > gpurun_out/pytest_r1x.log 2>&1; echo "pytest rc=$?"
timeout 600 python bench.py --steps 500 --warmup 10 --no-cpu-baseline --no-cusparse > gpurun_out/bench_r1x_cfg2.json 2> gpurun_out/bench_r1x_cfg2.err; echo "bench rc=$?"
bash scripts/gpu_sweep.sh r1x "--pool 0.95,0.6 --er-cost 5.0 --er-warps 0,4,8 --ahead 3 --pf-ell 0 --pf-er 1" cfg3f64 cfg5
