run() { # flags config tag
  EHYB_NVCC_FLAGS="$1" python paper_2204_06666_b200/build.py > gpurun_out/build_r_$3.log 2>&1
  timeout 600 python scripts/kernel_sweep.py --config $2 --pool 0.95 --er-cost 5.0 --er-warps 8 --ahead 3 --pf-ell 0 --pf-er 1 --vec 0 > gpurun_out/sweep_r_$3.txt 2> gpurun_out/sweep_r_$3.err
  echo "$1 $2 rc=$?"
}
run "-DEHYB_UNROLL_F32=4" cfg3f32 f32u4
run "-DEHYB_UNROLL_F32=6" cfg3f32 f32u6
run "-DEHYB_UNROLL_F64=4" cfg2 f64u4
run "-DEHYB_UNROLL_F64=6" cfg2 f64u6
run "-DEHYB_UNROLL_F64=12" cfg2 f64u12
