python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build_r1i.log 2>&1
timeout 900 python -m pytest tests -m gpu -x -q -k "spmv or shards or cg" > gpurun_out/pytest_r1i.log 2>&1; echo "pytest rc=$?"
bash scripts/gpu_sweep.sh r1i "--pool 0.95,0.7 --er-cost 5.0 --er-warps 4,8,12 --ahead 3 --pf-ell 0 --pf-er 1 --ring 0,1" cfg3f32 cfg2 cfg1
