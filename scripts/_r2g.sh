python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build_r2g.log 2>&1
timeout 1200 python -m pytest tests -m gpu -x -q > gpurun_out/pytest_r2g.log 2>&1; echo "pytest rc=$?"
bash scripts/gpu_sweep.sh r2g "--pool 0.95,0.8 --er-cost 5.0 --er-warps 4,8 --ahead 3 --pf-ell 0 --pf-er 1" cfg5 cfg3f64
