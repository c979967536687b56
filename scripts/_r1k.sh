python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build_r1k.log 2>&1
timeout 300 python -m pytest tests/test_gpu_spmv.py -x -q -k "corpus or small_bitwise or config_bitwise" > gpurun_out/pytest_r1k.log 2>&1; echo "pytest rc=$?"
bash scripts/gpu_sweep.sh r1k "--pool 0.95 --er-cost 5.0 --er-warps 4,8 --ahead 3 --pf-ell 0 --pf-er 1 --ring 0,1" cfg3f32 cfg2 cfg1
