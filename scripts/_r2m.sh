python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build_r2m.log 2>&1
bash scripts/gpu_sweep.sh r2m "--pool 0.95,100 --er-cost 5.0 --er-warps 0,4,8,16 --ahead 0,3 --pf-ell 0 --pf-er 0,1" cfg1
