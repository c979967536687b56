python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build_r2h.log 2>&1
timeout 1200 python -m pytest tests -m gpu -x -q > gpurun_out/pytest_r2h.log 2>&1; echo "pytest rc=$?"
