for F in "" "-DEHYB_F32_PIPE=0"; do
  T=$(echo "x$F" | tr -c 'a-zA-Z0-9' '_')
  EHYB_NVCC_FLAGS="$F" python paper_2204_06666_b200/build.py > gpurun_out/build_r2d_$T.log 2>&1
  if [ -z "$F" ]; then
    timeout 900 python -m pytest tests -m gpu -x -q -k "corpus or small or config_bitwise or long or shards" > gpurun_out/pytest_r2d.log 2>&1; echo "pytest rc=$?"
  fi
  timeout 600 python scripts/kernel_sweep.py --config cfg3f32 --pool 0.95 --er-cost 5.0 --er-warps 4,8 --ahead 3 --pf-ell 0 --pf-er 1 > gpurun_out/sweep_r2d_${T}_cfg3f32.txt 2> gpurun_out/sweep_r2d_${T}_cfg3f32.err
  echo "$F rc=$?"
done
