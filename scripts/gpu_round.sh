#!/bin/bash
# One GPU session: smoke, GPU tests, bench, ncu launch list + full capture.
# Usage (from the repo root, under gpurun): bash scripts/gpu_round.sh [tag]
TAG=${1:-r01}
OUT=gpurun_out
mkdir -p $OUT
nvidia-smi > $OUT/nvidia_smi_$TAG.txt 2>&1
python -c "import torch;p=torch.cuda.get_device_properties(0);print(p, p.L2_cache_size if hasattr(p,'L2_cache_size') else '')" > $OUT/devprops_$TAG.txt 2>&1
timeout 300 python -c "import __graft_entry__ as g; g.build(); g.smoke()" > $OUT/smoke_$TAG.log 2>&1; echo "smoke rc=$?" >> $OUT/summary_$TAG.txt
timeout 1200 python -m pytest tests -m gpu -x -q > $OUT/pytest_gpu_$TAG.log 2>&1; echo "pytest rc=$?" >> $OUT/summary_$TAG.txt
timeout 900 python bench.py --steps 2000 --warmup 20 > $OUT/bench_$TAG.json 2> $OUT/bench_$TAG.err; echo "bench rc=$?" >> $OUT/summary_$TAG.txt
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -k regex:spmv_fused -c 30 --csv --log-file $OUT/launches_$TAG.csv python bench.py --steps 20 --warmup 3 --no-cpu-baseline --no-cusparse > /dev/null 2> $OUT/ncu_launch_$TAG.err; echo "ncu-launches rc=$?" >> $OUT/summary_$TAG.txt
timeout 900 ncu --set full --clock-control none --import-source on -k regex:spmv_fused -s 5 -c 1 -o $OUT/prof_$TAG python bench.py --steps 8 --warmup 3 --no-cpu-baseline --no-cusparse > /dev/null 2> $OUT/ncu_full_$TAG.err; echo "ncu-full rc=$?" >> $OUT/summary_$TAG.txt
cat $OUT/summary_$TAG.txt
