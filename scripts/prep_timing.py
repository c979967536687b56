#!/usr/bin/env python3
"""Dev: stage times of the host and the GPU preprocessing on one config.
    EHYB_GPREP_TIMING=1 python scripts/prep_timing.py --config cfg2"""
import argparse
import os
import sys
import time

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import paper_2204_06666_b200 as E  # noqa: E402
from paper_2204_06666_b200 import workloads as W  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--config", default="cfg2")
ap.add_argument("--torch", action="store_true", help="initialise torch's CUDA context first (as bench.py)")
args = ap.parse_args()
if args.torch:
    import torch

    torch.cuda.set_device(0)
    torch.zeros(1, device="cuda:0")
n, r, c, v, tau = W.build_config(args.config)
m = E.CooMatrix(n, n, r, c, v)
prof = W.CONFIG_PROFILES.get(args.config)
prof = E.DeviceProfile(*prof) if prof else E.B200_PROFILE
params = E.compute_params(n, tau, prof)
for it in range(2):
    t0 = time.perf_counter(); g = E.build_graph(m); t1 = time.perf_counter()
    parts = E.partition_graph(g, params.n_parts, params.vec_cache_size); t2 = time.perf_counter()
    cls = E.classify_rows(m, parts); t3 = time.perf_counter()
    plan = E.build_reorder_plan(cls, params, parts); t4 = time.perf_counter()
    e = E.assemble_ehyb(m, plan, params, parts); t5 = time.perf_counter()
    print(f"host: build_graph {t1-t0:.3f} partition {t2-t1:.3f} classify {t3-t2:.3f} "
          f"plan {t4-t3:.3f} assemble {t5-t4:.3f} s", flush=True)
    t = {}
    t0 = time.perf_counter()
    e2 = E.build_ehyb_gpu(m, tau=tau, profile=prof, device=0, timings=t)
    import sys as _s
    print("gpu done", flush=True, file=_s.stderr)
    print("gpu:", {k: round(x, 3) for k, x in t.items()}, f"total {time.perf_counter()-t0:.3f} s",
          flush=True)
    del e, e2
