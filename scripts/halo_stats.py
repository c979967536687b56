#!/usr/bin/env python3
"""Halo volume of the weak-scaling multi-GPU workload (bench.py --gpus N):
per-rank halo values and halo ER rows with contiguous partition-id blocks vs
quotient-graph grouping (distributed.group_partitions). CPU only.

    python scripts/halo_stats.py 2 4 8
"""
import json
import os
import sys
import time

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import numpy as np  # noqa: E402

import paper_2204_06666_b200 as E  # noqa: E402
from paper_2204_06666_b200 import distributed as D  # noqa: E402


def stats(e, world):
    vec = e.params.vec_cache_size
    out = []
    for g in range(world):
        p0, p1 = D.part_range(e.n_parts, world, g)
        halo = D.halo_columns(e, p0, p1)
        out.append({"halo_values": int(halo.size), "owned_rows": int((p1 - p0) * vec)})
    return {"max_halo_values": max(o["halo_values"] for o in out),
            "mean_halo_frac": float(np.mean([o["halo_values"] / o["owned_rows"] for o in out]))}


for world in [int(a) for a in sys.argv[1:]] or [2, 4, 8]:
    t0 = time.time()
    n, r, c, v = D.weak_config(world)
    m = E.CooMatrix(n, n, r, c, v)
    del r, c, v
    e = E.build_ehyb(m, tau=8, profile=E.b200_profile(world))
    t_build = time.time() - t0
    t0 = time.time()
    e2 = D.renumber_partitions(e, D.group_partitions(e, world))
    t_group = time.time() - t0
    print(json.dumps({"gpus": world, "n": n, "n_parts": e.n_parts,
                      "contiguous_ids": stats(e, world), "grouped": stats(e2, world),
                      "build_s": round(t_build, 1), "group_s": round(t_group, 1)}), flush=True)
