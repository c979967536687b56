#!/usr/bin/env python3
"""Dev tool: time the GPU preprocessing pieces of one config twice (first
call, steady state): upload, build_graph, host BFS, the assemble C call,
EhybMatrix.check, close. python scripts/prep_probe.py cfg5"""
import os
import sys
import time

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import paper_2204_06666_b200 as E  # noqa: E402
from paper_2204_06666_b200 import gpu_prep as G  # noqa: E402
from paper_2204_06666_b200 import workloads as W  # noqa: E402

cfg = sys.argv[1]
n, r, c, v, tau = W.build_config(cfg)
m = E.CooMatrix(n, n, r, c, v)
prof = W.CONFIG_PROFILES.get(cfg)
params = E.compute_params(n, tau, E.DeviceProfile(*prof) if prof else E.B200_PROFILE)
nw, rw, cw, vw = W.stencil27(8, 8, 8)
E.build_ehyb_gpu(E.CooMatrix(nw, nw, rw, cw, vw), tau=tau, profile=E.DeviceProfile(4, 32, 8192), device=0)
orig_check = E.EhybMatrix.check
for rep in range(2):
    t = {}
    t0 = time.perf_counter()
    gp = G.GpuPrep(m, 0)
    t["upload"] = time.perf_counter() - t0
    t0 = time.perf_counter()
    g = gp.build_graph()
    t["build_graph"] = time.perf_counter() - t0
    t0 = time.perf_counter()
    parts = E.partition_graph(g, params.n_parts, params.vec_cache_size, seed=0)
    t["partition_graph"] = time.perf_counter() - t0
    del g
    tc = {}

    def timed_check(self):
        t1 = time.perf_counter()
        orig_check(self)
        tc["check"] = time.perf_counter() - t1

    E.EhybMatrix.check = timed_check
    t0 = time.perf_counter()
    _, _, e = gp.assemble(parts, params)
    t["assemble_total"] = time.perf_counter() - t0
    t["of_which_check"] = tc.get("check")
    E.EhybMatrix.check = orig_check
    t0 = time.perf_counter()
    gp.close()
    t["close"] = time.perf_counter() - t0
    t0 = time.perf_counter()
    del e
    t["free_arrays"] = time.perf_counter() - t0
    print(cfg, "rep", rep, {k: round(x, 3) if x is not None else None for k, x in t.items()}, flush=True)
