python -c "import __graft_entry__ as g; g.build()"
for C in cfg2 cfg3f32 cfg1; do
timeout 900 python scripts/kernel_sweep.py --config $C --pool 0.95,0.5 --er-cost 5.0 --er-warps 4 --ahead 0,3 --pf-ell 0 --pf-er 0,1 --mix 0,1 > gpurun_out/sweep_r1d_$C.txt 2>gpurun_out/sweep_r1d_$C.err
echo "$C rc=$?"
done
