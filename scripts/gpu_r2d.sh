#!/bin/bash
# r2d: work-unit split correctness + cost, multi-rank bench flow (gloo, ranks
# sharing the GPU), cfg5 through the sharded path. bash scripts/gpu_r2d.sh <tag>
TAG=${1:-r2d}
OUT=gpurun_out; mkdir -p $OUT
python -c "import __graft_entry__ as g; g.build()" > /dev/null 2>&1
timeout 1800 python -m pytest tests -m gpu -q -x > $OUT/pytest_gpu_$TAG.log 2>&1; echo "pytest rc=$?" >> $OUT/summary_$TAG.txt
for SP in 1 2; do
  EHYB_SPLIT=$SP timeout 600 python scripts/kernel_sweep.py --config cfg2 --pool 0.95 --er-cost 5.0 --er-warps 8 --pf-ell 0 --pf-er 1 --reps 300 --ahead 3 > $OUT/exp_${TAG}_split$SP.jsonl 2>&1
  echo "split $SP rc=$?" >> $OUT/summary_$TAG.txt
done
EHYB_DIST_BACKEND=gloo timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29533 bench.py --gpus 2 --config cfg2s --steps 20 --warmup 3 > $OUT/dist_${TAG}_gloo2_cfg2s.json 2> $OUT/dist_${TAG}_gloo2_cfg2s.err; echo "dist gloo2 cfg2s rc=$?" >> $OUT/summary_$TAG.txt
EHYB_DIST_BACKEND=gloo timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29534 bench.py --gpus 2 --config cfg5k4 --steps 10 --warmup 3 > $OUT/dist_${TAG}_gloo2_cfg5k4.json 2> $OUT/dist_${TAG}_gloo2_cfg5k4.err; echo "dist gloo2 cfg5k4 rc=$?" >> $OUT/summary_$TAG.txt
timeout 900 python bench.py --dist --config cfg5 --steps 50 --warmup 5 > $OUT/dist_${TAG}_n1_cfg5.json 2> $OUT/dist_${TAG}_n1_cfg5.err; echo "dist n1 cfg5 rc=$?" >> $OUT/summary_$TAG.txt
cat $OUT/summary_$TAG.txt; tail -3 $OUT/pytest_gpu_$TAG.log
