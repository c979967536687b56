python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build_r1v.log 2>&1
timeout 900 python -m pytest tests -m gpu -x -q -k "cg or cli or shards" > gpurun_out/pytest_r1v.log 2>&1; echo "pytest rc=$?"
timeout 900 python bench.py --dist --steps 300 --warmup 10 > gpurun_out/bench_r1v_dist.json 2> gpurun_out/bench_r1v_dist.err; echo "dist rc=$?"
timeout 900 python bench.py --steps 2000 --warmup 20 > gpurun_out/bench_r1v_cfg2.json 2> gpurun_out/bench_r1v_cfg2.err; echo "bench rc=$?"
