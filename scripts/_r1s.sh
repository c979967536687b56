python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build_r1s.log 2>&1
timeout 600 python scripts/kernel_sweep.py --config cfg3f32 --pool 0.95 --er-cost 5.0 --er-warps 8 --ahead 3 --pf-ell 0 --pf-er 1 > gpurun_out/sweep_r1s_cfg3f32.txt 2>&1; echo "sweep rc=$?"
timeout 600 ncu --set full --import-source on --clock-control none -k regex:spmv_fused -s 3 -c 1 -o gpurun_out/prof_r1s_ell python scripts/launch_once.py --config cfg3f32 --mode ell > gpurun_out/ncu_r1s_ell.log 2>&1; echo "ncu ell rc=$?"
timeout 600 ncu --set full --import-source on --clock-control none -k regex:spmv_fused -s 3 -c 1 -o gpurun_out/prof_r1s_er python scripts/launch_once.py --config cfg3f32 --mode er > gpurun_out/ncu_r1s_er.log 2>&1; echo "ncu er rc=$?"
