python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build_r1z.log 2>&1
timeout 900 python -m pytest tests/test_gpu_spmv.py -x -q -k "persistent or config_bitwise or corpus or long" > gpurun_out/pytest_r1z.log 2>&1; echo "pytest rc=$?"
timeout 300 python scripts/pcie_probe.py > gpurun_out/pcie_r1z.json 2>&1; echo "pcie rc=$?"
bash scripts/gpu_sweep.sh r1z "--pool 0.95,0.7 --er-cost 5.0 --er-warps 4,8 --ahead 3 --pf-ell 0 --pf-er 1" cfg2 cfg3f32 cfg3f64 cfg5
