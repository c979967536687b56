python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build_r1o.log 2>&1
bash scripts/gpu_sweep.sh r1o "--pool 0.95 --er-cost 5.0 --er-warps 8 --ahead 3 --pf-ell 0 --pf-er 1 --vec 0" cfg3f32 cfg2
bash scripts/gpu_sweep.sh r1p "--pool 0.95 --er-cost 5.0 --er-warps 8 --ahead 3 --pf-ell 0 --pf-er 1 --vec 1" cfg3f32 cfg2
