#!/usr/bin/env python3
"""Dev tool for profilers: build a config, upload it, then launch the fused
kernel (or one phase of it) a few times — run under ncu with -k/-s/-c.

    python scripts/launch_once.py --config cfg3f32 [--mode full|ell|er] [--n 5]
"""
import argparse
import ctypes as C
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import torch  # noqa: E402

import bench  # noqa: E402
import paper_2204_06666_b200 as E  # noqa: E402
from paper_2204_06666_b200 import _lib as L  # noqa: E402
from paper_2204_06666_b200 import workloads as W  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--config", default="cfg3f32")
ap.add_argument("--mode", default="full", choices=("full", "ell", "er"))
ap.add_argument("--n", type=int, default=5)
args = ap.parse_args()
m, e, _ = bench.build_workload(args.config)
dm = E.device_matrix(e, 0)
xr = torch.from_numpy(E.permute_vector(W.deterministic_vector(e.dimension, 0), e.plan)).to(
    "cuda:0", dm.torch_dtype)
y = torch.empty_like(xr)
# ell / er: one phase alone (EHYB_TUNE_PHASES, measurement only): the ER-only
# launch isolates the spill path (its L2 hit rate is the ER x gathers')
dm.tune(phases={"full": 0, "ell": 1, "er": 2}[args.mode])
st = C.c_void_p(torch.cuda.current_stream().cuda_stream)
for _ in range(args.n):
    L.call("ehyb_dev_spmv", dm.handle, C.c_void_p(xr.data_ptr()), C.c_void_p(y.data_ptr()),
           L.MODE_DEFAULT, st)
torch.cuda.synchronize()
print("done", dm.info())
