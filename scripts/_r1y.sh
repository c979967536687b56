python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build_r1y.log 2>&1
timeout 900 python -m pytest tests/test_gpu_spmv.py -x -q -k "persistent or config_bitwise or corpus" > gpurun_out/pytest_r1y.log 2>&1; echo "pytest rc=$?"
timeout 600 python bench.py --steps 2000 --warmup 20 --no-cpu-baseline --no-cusparse > gpurun_out/bench_r1y_cfg2.json 2> gpurun_out/bench_r1y_cfg2.err; echo "bench rc=$?"
bash scripts/gpu_sweep.sh r1y "--pool 0.95,0.5,0.2 --er-cost 5.0 --er-warps 4,8 --ahead 3 --pf-ell 0 --pf-er 1" cfg3f64 cfg5
