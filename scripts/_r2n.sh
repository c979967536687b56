python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build_r2n.log 2>&1
timeout 1200 python -m pytest tests -m gpu -x -q > gpurun_out/pytest_r2n.log 2>&1; echo "pytest rc=$?"
timeout 600 python bench.py --config cfg1 --steps 500 --warmup 10 --cpu-seconds 5 > gpurun_out/bench_r2n_cfg1.json 2> gpurun_out/bench_r2n_cfg1.err; echo "cfg1 rc=$?"
