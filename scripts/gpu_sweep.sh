#!/bin/bash
# knob sweep + per-CTA phase profile: bash scripts/gpu_sweep.sh <tag> "<sweep args>" cfgs...
TAG=$1; ARGS="$2"; shift 2
OUT=gpurun_out; mkdir -p $OUT
python -c "import __graft_entry__ as g; g.build()" > $OUT/build_$TAG.log 2>&1
for C in "$@"; do
  timeout 900 python scripts/kernel_sweep.py --config $C $ARGS > $OUT/sweep_${TAG}_$C.txt 2>$OUT/sweep_${TAG}_$C.err
  echo "$C rc=$?"
done
