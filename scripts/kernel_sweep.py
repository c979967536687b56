#!/usr/bin/env python3
"""Dev tool: sweep the fused kernel's launch knobs on one config and print
per-variant device time, effective GB/s and per-CTA phase timings.

    python scripts/kernel_sweep.py [--config cfg2] [--reps 300]
"""

from __future__ import annotations

import argparse
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


def time_variant(dm, xr, y, reps, stream, fma=False):
    ev0 = torch.cuda.Event(enable_timing=True)
    ev1 = torch.cuda.Event(enable_timing=True)
    for _ in range(10):
        dm.spmv(xr, y, fma=fma, stream=stream)
    ev0.record(stream)
    for _ in range(reps):
        dm.spmv(xr, y, fma=fma, stream=stream)
    ev1.record(stream)
    ev1.synchronize()
    return ev0.elapsed_time(ev1) / reps * 1e3  # us


STAMPS = ("start", "window", "ell_issued", "end", "own_er", "combine", "pool", "ell_published")


def cta_profile(dm, xr, y, stream, n_ctas):
    """Per-CTA phase stamps (us from the first CTA start): min / median / max."""
    t = torch.zeros(n_ctas * 8, dtype=torch.int64, device=xr.device)
    dm.tune(timing=t)
    dm.spmv(xr, y, stream=stream)
    stream.synchronize()
    dm.tune(timing=None)
    a = t.cpu().numpy().reshape(n_ctas, 8).astype(np.float64)
    t0 = a[:, 0].min()
    out = {}
    for i, name in enumerate(STAMPS):
        col = a[:, i]
        col = col[col > 0]
        if col.size == 0:
            continue
        rel = (col - t0) / 1e3
        out[name] = [round(float(np.min(rel)), 2), round(float(np.median(rel)), 2),
                     round(float(np.max(rel)), 2)]
    out["raw_col5_col6_median"] = [float(np.median(a[:, 5])), float(np.median(a[:, 6]))]
    out["cta_duration_us"] = [round(float(v), 2) for v in
                              np.percentile((a[:, 3] - a[:, 0]) / 1e3, [0, 50, 90, 100])]
    return out


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--config", default="cfg2")
    ap.add_argument("--reps", type=int, default=300)
    ap.add_argument("--quick", action="store_true")
    ap.add_argument("--pool", default="0,0.9,1.0,1.1")
    ap.add_argument("--er-cost", default="2.0")
    ap.add_argument("--er-warps", default="0,4")
    ap.add_argument("--ahead", default="0,3")
    ap.add_argument("--pf-ell", default="0,1")
    ap.add_argument("--pf-er", default="0,1")
    ap.add_argument("--ring", default="0", help="EHYB_RING values (0 = register ELL path)")
    ap.add_argument("--stage-kb", default="16", help="EHYB_STAGE_KB values")
    ap.add_argument("--vec", default="0", help="EHYB_VEC values (0 = SELL layout, scalar loads)")
    ap.add_argument("--phases", action="store_true", help="also time ELL alone and ER alone")
    args = ap.parse_args()
    m, e, _ = bench.build_workload(args.config)
    gold = bench.golden_y_digest(args.config)
    bmin = E.min_bytes(e)
    dm = E.device_matrix(e, 0)
    stream = torch.cuda.Stream(0)
    x = W.deterministic_vector(e.dimension, 0)
    with torch.cuda.stream(stream):
        xr = torch.from_numpy(E.permute_vector(x, e.plan)).to("cuda:0", dm.torch_dtype)
        y = torch.empty_like(xr)
    stream.synchronize()
    n_ctas = dm.info()["ctas"]
    results = []
    from paper_2204_06666_b200.device import DeviceMatrix

    handles = {}
    for pool, ercost, ring, skb, vec in itertools.product(
            args.pool.split(","), args.er_cost.split(","), args.ring.split(","),
            args.stage_kb.split(","), args.vec.split(",")):
        if ring == "0" and skb != args.stage_kb.split(",")[0]:
            continue
        os.environ["EHYB_VEC"] = vec
        os.environ["EHYB_POOL_FACTOR"] = pool
        os.environ["EHYB_ER_COST"] = ercost
        os.environ["EHYB_RING"] = ring
        os.environ["EHYB_STAGE_KB"] = skb
        handles[(pool, ercost, ring, skb, vec)] = DeviceMatrix(e, 0)
    ewl = [int(v) for v in args.er_warps.split(",")]
    ahl = [int(v) for v in args.ahead.split(",")]
    pfl = [int(v) for v in args.pf_ell.split(",")]
    pfrl = [int(v) for v in args.pf_er.split(",")]
    for (pool, ercost, ring, skb, vec), h in handles.items():
        for pfer, ew, ah, pfe in itertools.product(pfrl, ewl, ahl, pfl):
            h.tune(prefetch_ell=pfe, prefetch_er=pfer, threads=int(os.environ.get('EHYB_THREADS', h.info()['threads_per_cta'])), er_warps=ew, claim_ahead=ah)
            us = time_variant(h, xr, y, args.reps, stream)
            ok = gold is None or digest(y.cpu().numpy()) == gold["y_reordered"]
            results.append(dict(pool=pool, er_cost=ercost, ring=ring, stage_kb=skb, vec=vec,
                                ring_kb=h.info()["ring_bytes"] // 1024, pf_ell=pfe, pf_er=pfer, er_warps=ew,
                                ahead=ah, us=round(us, 2), gbs=round(bmin / us / 1e3, 1),
                                bitwise=ok))
            if args.phases:  # each phase alone (measurement-only launches)
                for ph, key in ((1, "ell_only_us"), (2, "er_only_us")):
                    h.tune(phases=ph)
                    results[-1][key] = round(time_variant(h, xr, y, args.reps, stream), 2)
                h.tune(phases=0)
            print(json.dumps(results[-1]), flush=True)
    best = min(results, key=lambda r: r["us"])
    dm = handles[(best["pool"], best["er_cost"], best["ring"], best["stage_kb"], best["vec"])]
    dm.tune(prefetch_ell=best["pf_ell"], prefetch_er=best["pf_er"], threads=int(os.environ.get('EHYB_THREADS', dm.info()['threads_per_cta'])),
            er_warps=best["er_warps"], claim_ahead=best["ahead"])
    prof = cta_profile(dm, xr, y, stream, n_ctas)
    # the two phases on their own (split launches): what each costs in isolation
    import ctypes as C
    from paper_2204_06666_b200 import _lib as L

    def phase_us(name):
        ev0 = torch.cuda.Event(enable_timing=True)
        ev1 = torch.cuda.Event(enable_timing=True)
        st = C.c_void_p(stream.cuda_stream)
        xp, yp = C.c_void_p(xr.data_ptr()), C.c_void_p(y.data_ptr())
        for _ in range(10):
            L.call(name, dm.handle, xp, yp, L.MODE_STRICT, st)
        ev0.record(stream)
        for _ in range(args.reps):
            L.call(name, dm.handle, xp, yp, L.MODE_STRICT, st)
        ev1.record(stream)
        ev1.synchronize()
        return round(ev0.elapsed_time(ev1) / args.reps * 1e3, 2)

    dm.tune(phases=1)
    prof["ell_only_us"] = round(time_variant(dm, xr, y, args.reps, stream), 2)
    dm.tune(phases=2)
    prof["er_only_us"] = round(time_variant(dm, xr, y, args.reps, stream), 2)
    dm.tune(phases=0)
    us_fma = time_variant(dm, xr, y, args.reps, stream, fma=True)
    print(json.dumps({"config": args.config, "best": best, "cta_profile_best": prof,
                      "fma_us": round(us_fma, 2), "bmin": bmin}), flush=True)


if __name__ == "__main__":
    main()
