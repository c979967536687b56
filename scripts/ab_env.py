#!/usr/bin/env python3
"""Dev tool: A/B handle-creation env knobs on one config, same process, the
variants timed in alternation (CUDA events, median of rounds), y checked
against the golden digest.

    python scripts/ab_env.py cfg3f32 EHYB_META_SMEM=0,1 [EHYB_X=a,b ...]
"""
from __future__ import annotations

import itertools
import json
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
sys.path.insert(0, os.path.join(ROOT, "tests", "golden"))

import numpy as np  # noqa: E402
import torch  # noqa: E402

import bench  # noqa: E402
import paper_2204_06666_b200 as E  # noqa: E402
from golden_util import digest  # noqa: E402
from paper_2204_06666_b200 import workloads as W  # noqa: E402
from paper_2204_06666_b200.device import DeviceMatrix  # noqa: E402


def main():
    cfgs = [a for a in sys.argv[1:] if "=" not in a]
    knobs = [a.split("=", 1) for a in sys.argv[1:] if "=" in a]
    names = [k for k, _ in knobs]
    combos = list(itertools.product(*[v.split(",") for _, v in knobs]))
    reps = int(os.environ.get("AB_REPS", "100"))
    rounds = int(os.environ.get("AB_ROUNDS", "5"))
    for cfg in cfgs:
        m, e, _ = bench.build_workload(cfg)
        gold = bench.golden_y_digest(cfg)
        bmin = E.min_bytes(e)
        stream = torch.cuda.Stream(0)
        x = W.deterministic_vector(e.dimension, 0)
        handles = []
        for combo in combos:
            for k, v in zip(names, combo):
                os.environ[k] = v
            handles.append(DeviceMatrix(e, 0))
        with torch.cuda.stream(stream):
            xr = torch.from_numpy(E.permute_vector(x, e.plan)).to("cuda:0", handles[0].torch_dtype)
            y = torch.empty_like(xr)
        stream.synchronize()
        times = [[] for _ in combos]
        ok = [True] * len(combos)
        ev0, ev1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        for r in range(rounds):
            for i, h in enumerate(handles):
                for _ in range(5):
                    h.spmv(xr, y, stream=stream)
                ev0.record(stream)
                for _ in range(reps):
                    h.spmv(xr, y, stream=stream)
                ev1.record(stream)
                ev1.synchronize()
                times[i].append(ev0.elapsed_time(ev1) / reps * 1e3)
                if r == 0 and gold is not None:
                    ok[i] = digest(y.cpu().numpy()) == gold["y_reordered"]
        for i, combo in enumerate(combos):
            us = float(np.median(times[i]))
            print(json.dumps({"config": cfg, **dict(zip(names, combo)), "us": round(us, 2),
                              "min_us": round(min(times[i]), 2), "frac": round(bmin / us / 1e3 / 6555.2, 4),
                              "bitwise": ok[i], "info": {k: handles[i].info()[k] for k in ("smem_bytes", "threads_per_cta")}}),
                  flush=True)
        del handles


if __name__ == "__main__":
    main()
