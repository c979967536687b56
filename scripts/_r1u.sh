python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build_r1u.log 2>&1
timeout 900 python -m pytest tests -m gpu -x -q > gpurun_out/pytest_r1u.log 2>&1; echo "pytest rc=$?"
bash scripts/gpu_sweep.sh r1u "--pool 0.95,0.8 --er-cost 5.0 --er-warps 4,8,12 --ahead 3 --pf-ell 0 --pf-er 1" cfg3f32 cfg2
timeout 900 python bench.py --dist --steps 200 --warmup 10 > gpurun_out/bench_r1u_dist.json 2> gpurun_out/bench_r1u_dist.err; echo "dist rc=$?"
