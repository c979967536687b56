for F in "" "-DEHYB_UNROLL_F32=8" "-DEHYB_UNROLL_F32=12" "-DEHYB_NO_PUBLISH_FENCE"; do
  T=$(echo "x$F" | tr -c 'a-zA-Z0-9' '_')
  EHYB_NVCC_FLAGS="$F" python paper_2204_06666_b200/build.py > gpurun_out/build_q_$T.log 2>&1
  timeout 600 python scripts/kernel_sweep.py --config cfg3f32 --pool 0.95 --er-cost 5.0 --er-warps 8 --ahead 3 --pf-ell 0 --pf-er 1 --vec 0 > gpurun_out/sweep_q_$T.txt 2> gpurun_out/sweep_q_$T.err
  echo "$F rc=$?"
done
