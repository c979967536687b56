python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build_r1n.log 2>&1
timeout 900 python -m pytest tests -m gpu -x -q > gpurun_out/pytest_r1n.log 2>&1; echo "pytest rc=$?"
bash scripts/gpu_sweep.sh r1n "--pool 0.95 --er-cost 5.0 --er-warps 4,8 --ahead 3 --pf-ell 0 --pf-er 1 --vec 0,1" cfg3f32 cfg2 cfg3f64
