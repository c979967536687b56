#!/bin/bash
# fp32 ELL unroll sweep on cfg3f32: bash scripts/gpu_unroll.sh <tag> U...
TAG=$1; shift
OUT=gpurun_out; mkdir -p $OUT
for U in "$@"; do
  EHYB_NVCC_FLAGS="-DEHYB_UNROLL_F32=$U" python -m paper_2204_06666_b200.build --force > $OUT/build_${TAG}_u$U.log 2>&1
  for R in 1 2; do
    timeout 600 python bench.py --config cfg3f32 --steps 500 --warmup 10 --no-cpu-baseline --no-cusparse > $OUT/unroll_${TAG}_u${U}_$R.json 2> $OUT/unroll_${TAG}_u${U}_$R.err
    echo "U=$U run $R rc=$? $(python -c "import json,sys; d=json.load(open('$OUT/unroll_${TAG}_u${U}_$R.json')); print(round(d['ms_per_step']*1e3,1),'us', d.get('parity'))" 2>&1)"
  done
done
python -m paper_2204_06666_b200.build --force > /dev/null 2>&1
