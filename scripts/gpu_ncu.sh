#!/bin/bash
# ncu captures per config (full set, one fused launch) + the ER-only launch of
# cfg2 / cfg3f32 (spill-gather L2 hit rate) + the cfg2 launch list.
# bash scripts/gpu_ncu.sh <tag> [configs...]
TAG=${1:-r2}; shift
CONFIGS=${@:-cfg2 cfg3f32 cfg3f64 cfg5 cfg1 cfg4}
OUT=gpurun_out; mkdir -p $OUT
# the prebuilt .so files travel with the snapshot (no rebuild on the box)
NCU="ncu --set full --clock-control none --import-source on -k regex:spmv_fused -s 5 -c 1"
for C in $CONFIGS; do
  timeout 900 $NCU -o $OUT/prof_${TAG}_$C python scripts/launch_once.py --config $C --n 7 > $OUT/ncu_${TAG}_$C.log 2>&1
  echo "ncu $C rc=$?" >> $OUT/ncu_${TAG}_summary.txt
  ncu -i $OUT/prof_${TAG}_$C.ncu-rep --page raw --csv > $OUT/prof_${TAG}_$C.raw.csv 2>/dev/null
  ncu -i $OUT/prof_${TAG}_$C.ncu-rep --page details --csv > $OUT/prof_${TAG}_$C.details.csv 2>/dev/null
  [ "$C" = "${KEEP:-cfg2}" ] || rm -f $OUT/prof_${TAG}_$C.ncu-rep
done
for C in cfg2 cfg3f32; do
  timeout 900 $NCU -o $OUT/prof_${TAG}_${C}_er python scripts/launch_once.py --config $C --mode er --n 7 > $OUT/ncu_${TAG}_${C}_er.log 2>&1
  echo "ncu $C er rc=$?" >> $OUT/ncu_${TAG}_summary.txt
  ncu -i $OUT/prof_${TAG}_${C}_er.ncu-rep --page raw --csv > $OUT/prof_${TAG}_${C}_er.raw.csv 2>/dev/null
  rm -f $OUT/prof_${TAG}_${C}_er.ncu-rep
done
EHYB_BENCH_PREP=host timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file $OUT/launches_${TAG}_cfg2.csv python bench.py --steps 20 --warmup 3 --no-cpu-baseline --no-cusparse > /dev/null 2> $OUT/ncu_launch_$TAG.err; echo "launches rc=$?" >> $OUT/ncu_${TAG}_summary.txt
du -sh $OUT; cat $OUT/ncu_${TAG}_summary.txt
