python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build_r2a.log 2>&1
timeout 900 python -m pytest tests/test_gpu_spmv.py -x -q -k "persistent or config_bitwise or corpus" > gpurun_out/pytest_r2a.log 2>&1; echo "pytest rc=$?"
bash scripts/gpu_sweep.sh r2a "--pool 0.95,0.7,0.5 --er-cost 5.0 --er-warps 4,8 --ahead 3 --pf-ell 0 --pf-er 1" cfg3f64 cfg5
bash scripts/gpu_sweep.sh r2a "--pool 0.95 --er-cost 5.0 --er-warps 8 --ahead 3 --pf-ell 0 --pf-er 1" cfg2
