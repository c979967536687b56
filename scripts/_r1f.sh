bash scripts/gpu_sweep.sh r1f "--pool 0.95 --er-cost 5.0 --er-warps 0,4 --ahead 3 --pf-ell 0 --pf-er 1" cfg2 cfg3f32 cfg1
timeout 600 python -m pytest tests -m gpu -x -q -k "long_rows" > gpurun_out/pytest_r1f.log 2>&1; echo "pytest rc=$?"
timeout 600 python bench.py --config cfg4 --steps 100 --warmup 5 --no-cpu-baseline > gpurun_out/bench_r1f_cfg4.json 2> gpurun_out/bench_r1f_cfg4.err; echo "cfg4 rc=$?"
