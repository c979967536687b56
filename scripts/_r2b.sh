for F in "" "-DEHYB_ER_PAIRS=0"; do
  T=$(echo "x$F" | tr -c 'a-zA-Z0-9' '_')
  EHYB_NVCC_FLAGS="$F" python paper_2204_06666_b200/build.py > gpurun_out/build_r2b_$T.log 2>&1
  if [ -z "$F" ]; then
    timeout 900 python -m pytest tests -m gpu -x -q -k "persistent or config_bitwise or corpus or long or shards or small" > gpurun_out/pytest_r2b.log 2>&1; echo "pytest rc=$?"
  fi
  for C in cfg2 cfg3f32 cfg3f64 cfg5; do
    timeout 600 python scripts/kernel_sweep.py --config $C --pool 0.95 --er-cost 5.0 --er-warps 4,8 --ahead 3 --pf-ell 0 --pf-er 1 > gpurun_out/sweep_r2b_${T}_$C.txt 2> gpurun_out/sweep_r2b_${T}_$C.err
    echo "$F $C rc=$?"
  done
done
