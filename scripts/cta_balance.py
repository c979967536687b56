#!/usr/bin/env python3
"""Dev tool: per-CTA phase stamps of one fused launch next to each
partition's work (ELL slots, own ER slices/entries, pooled slices), to see
whether the spread of CTA finish times is structural or dynamic.

    python scripts/cta_balance.py --config cfg2 [--vec 1] > profiles/cta_balance_<tag>.json
"""

from __future__ import annotations

import argparse
import json
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import numpy as np  # noqa: E402
import torch  # noqa: E402

import bench  # noqa: E402
import paper_2204_06666_b200 as E  # noqa: E402
from paper_2204_06666_b200 import workloads as W  # noqa: E402

STAMPS = ("start", "window", "ell_issued", "end", "own_er", "combine", "pool", "ell_published")


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--config", default="cfg2")
    ap.add_argument("--vec", default="0")
    ap.add_argument("--launches", type=int, default=5)
    args = ap.parse_args()
    os.environ["EHYB_VEC"] = args.vec
    m, e, _ = bench.build_workload(args.config)
    dm = E.device_matrix(e, 0)
    info = dm.info()
    x = W.deterministic_vector(e.dimension, 0)
    xr = torch.from_numpy(E.permute_vector(x, e.plan)).to("cuda:0", dm.torch_dtype)
    y = torch.empty_like(xr)
    for _ in range(20):
        dm.spmv(xr, y)
    torch.cuda.synchronize()
    n_ctas = info["ctas"]
    runs = []
    for _ in range(args.launches):
        t = torch.zeros(n_ctas * 8, dtype=torch.int64, device="cuda:0")
        dm.tune(timing=t)
        dm.spmv(xr, y)
        torch.cuda.synchronize()
        dm.tune(timing=None)
        a = t.cpu().numpy().reshape(n_ctas, 8).astype(np.float64)
        a = (a - a[:, 0].min()) / 1e3
        runs.append(a)
    a = np.median(np.stack(runs), axis=0)
    vec = e.params.vec_cache_size
    spp = vec // 32
    pos = e.position_ell.astype(np.int64)
    ell = np.array([pos[(p + 1) * spp] - pos[p * spp] for p in range(e.n_parts)], dtype=np.float64)
    er_rows_owner = e.plan.y_idx_er // vec
    er_ent = np.bincount(er_rows_owner, weights=e.er_row_widths, minlength=e.n_parts)
    out = {"config": args.config, "vec": args.vec, "info": info}
    if n_ctas == e.n_parts:
        pub = a[:, 7]
        end = a[:, 3]
        out["corr_ell_published_vs_ell_slots"] = float(np.corrcoef(pub, ell)[0, 1])
        out["corr_ell_published_vs_er_entries"] = float(np.corrcoef(pub, er_ent)[0, 1])
        out["corr_end_vs_er_entries"] = float(np.corrcoef(end, er_ent)[0, 1])
        # run-to-run: is the same CTA late every launch?
        pubs = np.stack([r[:, 7] for r in runs])
        out["corr_published_launch0_vs_launch1"] = float(np.corrcoef(pubs[0], pubs[1])[0, 1])
        order = np.argsort(pub)
        out["earliest"] = [dict(cta=int(i), ell_published=round(float(pub[i]), 2),
                                end=round(float(end[i]), 2), ell_slots=int(ell[i]),
                                er_entries=int(er_ent[i]), window=round(float(a[i, 1]), 2))
                           for i in order[:5]]
        out["latest"] = [dict(cta=int(i), ell_published=round(float(pub[i]), 2),
                              end=round(float(end[i]), 2), ell_slots=int(ell[i]),
                              er_entries=int(er_ent[i]), window=round(float(a[i, 1]), 2))
                         for i in order[-5:]]
        # SM placement: CTA i runs on SM smid(i) — unknown here; report the
        # finish time by CTA index parity / halves (die halves map to ids?)
        out["pub_by_cta_quartile"] = [round(float(np.median(pub[q::4])), 2) for q in range(4)]
    out["stamps_median_over_ctas"] = {nm: round(float(np.median(a[:, i][a[:, i] > 0])), 2)
                                      for i, nm in enumerate(STAMPS) if (a[:, i] > 0).any()}
    print(json.dumps(out, indent=1))


if __name__ == "__main__":
    main()
