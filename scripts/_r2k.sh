for H in 0 1 2 3; do
  EHYB_NVCC_FLAGS="-DEHYB_LD_HINT=$H" python paper_2204_06666_b200/build.py > gpurun_out/build_r2k_$H.log 2>&1
  for C in cfg2 cfg3f32; do
    timeout 600 python scripts/kernel_sweep.py --config $C --pool 0.95 --er-cost 5.0 --er-warps 8 --ahead 3 --pf-ell 0 --pf-er 1 > gpurun_out/sweep_r2k_h${H}_$C.txt 2> gpurun_out/sweep_r2k_h${H}_$C.err
    echo "hint $H $C rc=$?"
  done
done
