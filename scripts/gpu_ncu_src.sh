#!/bin/bash
# ncu full capture of one fused launch per config, kept with its source page
# (per-line instruction counts / stalls): bash scripts/gpu_ncu_src.sh <tag> cfgs...
TAG=$1; shift
OUT=gpurun_out; mkdir -p $OUT
NCU="ncu --set full --clock-control none --import-source on -k regex:spmv_fused -s 5 -c 1"
for C in "$@"; do
  timeout 900 $NCU -o $OUT/prof_${TAG}_$C python scripts/launch_once.py --config $C --n 7 > $OUT/ncu_${TAG}_$C.log 2>&1
  echo "ncu $C rc=$?"
  ncu -i $OUT/prof_${TAG}_$C.ncu-rep --page raw --csv > $OUT/prof_${TAG}_$C.raw.csv 2>/dev/null
  ncu -i $OUT/prof_${TAG}_$C.ncu-rep --page source --csv --print-source cuda > $OUT/prof_${TAG}_$C.src.csv 2>/dev/null
  ncu -i $OUT/prof_${TAG}_$C.ncu-rep --page source --csv --print-source sass > $OUT/prof_${TAG}_$C.sass.csv 2>/dev/null
  rm -f $OUT/prof_${TAG}_$C.ncu-rep
done
du -sh $OUT
