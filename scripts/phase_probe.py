#!/usr/bin/env python3
"""Dev tool: per config, time the fused launch, ELL alone and ER alone
(EHYB_TUNE_PHASES, measurement-only launches), an ER-first-warp sweep and
the per-CTA end-time spread.

    python scripts/phase_probe.py cfg3f32 cfg4 ...
"""

from __future__ import annotations

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

REPS = int(os.environ.get("PROBE_REPS", "200"))


def timed(dm, xr, y, stream, reps=REPS, flush=None):
    ev = [torch.cuda.Event(enable_timing=True) for _ in range(2 * reps)]
    for _ in range(5):
        dm.spmv(xr, y, stream=stream)
    ts = []
    for i in range(reps):
        if flush is not None:
            with torch.cuda.stream(stream):
                flush.add_(1)
        ev[2 * i].record(stream)
        dm.spmv(xr, y, stream=stream)
        ev[2 * i + 1].record(stream)
    stream.synchronize()
    ts = [ev[2 * i].elapsed_time(ev[2 * i + 1]) * 1e3 for i in range(reps)]
    return round(float(np.median(ts)), 2)


def main():
    for cfg in sys.argv[1:]:
        m, e, _ = bench.build_workload(cfg)
        gold = bench.golden_y_digest(cfg)
        bmin = E.min_bytes(e)
        dm = E.device_matrix(e, 0)
        stream = torch.cuda.Stream(0)
        x = W.deterministic_vector(e.dimension, 0)
        with torch.cuda.stream(stream):
            xr = torch.from_numpy(E.permute_vector(x, e.plan)).to("cuda:0", dm.torch_dtype)
            y = torch.empty_like(xr)
            flush = torch.zeros(128 * 1024 * 1024, dtype=torch.float32, device="cuda:0")
        stream.synchronize()
        info = dm.info()
        out = {"config": cfg, "bmin": bmin, "info": {k: info[k] for k in ("threads_per_cta", "ctas", "er_slices", "pool_slices", "er_buf_slices", "long_rows")}}
        out["full_us"] = timed(dm, xr, y, stream, flush=flush)
        ok = gold is None or digest(y.cpu().numpy()) == gold["y_reordered"]
        out["bitwise"] = ok
        out["full_noflush_us"] = timed(dm, xr, y, stream)
        for ph, key in ((1, "ell_only_us"), (2, "er_only_us")):
            dm.tune(phases=ph)
            out[key] = timed(dm, xr, y, stream, flush=flush)
        dm.tune(phases=0)
        ew = {}
        for w in [int(v) for v in os.environ.get("PROBE_ERW", "2,4,6,10").split(",")]:
            dm.tune(er_warps=w)
            ew[w] = timed(dm, xr, y, stream, flush=flush)
        out["er_warps_us"] = ew
        dm.tune(er_warps=6)
        n_ctas = info["ctas"]
        t = torch.zeros(n_ctas * 8, dtype=torch.int64, device="cuda:0")
        dm.tune(timing=t)
        dm.spmv(xr, y, stream=stream)
        stream.synchronize()
        dm.tune(timing=None)
        a = t.cpu().numpy().reshape(n_ctas, 8).astype(np.float64)
        t0 = a[:, 0].min()
        names = ("start", "window", "ell_issued", "end", "own_er", "combine", "pool", "ell_published")
        prof = {}
        for i, nm in enumerate(names):
            col = a[:, i]
            col = col[col > 1e12]
            if col.size:
                rel = (col - t0) / 1e3
                prof[nm] = [round(float(v), 1) for v in np.percentile(rel, [0, 10, 50, 90, 100])]
        out["cta_stamps_pct_0_10_50_90_100"] = prof
        print(json.dumps(out), flush=True)
        del dm


if __name__ == "__main__":
    main()
