run() { # flags threads tag extra-sweep-args
  EHYB_NVCC_FLAGS="$1" python paper_2204_06666_b200/build.py > gpurun_out/build_t_$3.log 2>&1
  EHYB_THREADS=$2 timeout 600 python scripts/kernel_sweep.py --config cfg3f32 --pool 0.95 --er-cost 5.0 --er-warps 8 --ahead 3 --pf-er 1 $4 > gpurun_out/sweep_t_$3.txt 2> gpurun_out/sweep_t_$3.err
  echo "$1 $2 rc=$?"
}
run "" 1024 base "--pf-ell 0,1"
run "-DEHYB_MAX_THREADS=768 -DEHYB_UNROLL_F32=16" 768 t768u16 "--pf-ell 0"
run "-DEHYB_MAX_THREADS=768 -DEHYB_UNROLL_F32=12" 768 t768u12 "--pf-ell 0"
run "-DEHYB_MAX_THREADS=512 -DEHYB_UNROLL_F32=16" 512 t512u16 "--pf-ell 0"
run "-DEHYB_MAX_THREADS=512 -DEHYB_UNROLL_F32=24" 512 t512u24 "--pf-ell 0"
