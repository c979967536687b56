python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build_r2f.log 2>&1
timeout 900 python -m pytest tests/test_gpu_spmv.py -x -q -k "persistent or config_bitwise" > gpurun_out/pytest_r2f.log 2>&1; echo "pytest rc=$?"
bash scripts/gpu_sweep.sh r2f "--pool 0.95,0.6,0.3,0.05 --er-cost 5.0 --er-warps 4,8 --ahead 3 --pf-ell 0 --pf-er 1" cfg3f64 cfg5
