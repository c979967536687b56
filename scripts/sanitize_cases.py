#!/usr/bin/env python3
"""Small fused-kernel cases for compute-sanitizer (memcheck / racecheck /
synccheck / initcheck): the cross-CTA ER pool (one partition per CTA),
persistent CTAs (several partitions per CTA, in-place pooled rows), long rows
in all three arithmetic modes, and the two-launch shard path. Each result is
checked against the C restatement of the reference engine.

    compute-sanitizer --tool racecheck python scripts/sanitize_cases.py
"""

import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import numpy as np  # noqa: E402
import torch  # noqa: E402

import paper_2204_06666_b200 as E  # noqa: E402
from oracle import c_oracle  # noqa: E402
from paper_2204_06666_b200 import distributed as D  # noqa: E402
from paper_2204_06666_b200 import workloads as W  # noqa: E402
from paper_2204_06666_b200.device import DeviceMatrix  # noqa: E402


def check(name, got, want):
    ok = got.tobytes() == want.tobytes()
    print(f"{name}: {'bitwise == oracle' if ok else 'MISMATCH'}", flush=True)
    return ok


def main():
    torch.cuda.set_device(0)
    ok = True
    # 1. pool: more ER than the per-CTA budget, one partition per CTA
    n, r, c, v = W.permute_symmetric(*W.stencil27(20, 20, 20), seed=1)
    e = E.build_ehyb(E.CooMatrix(n, n, r, c, v), tau=8, profile=E.DeviceProfile(16, 32, 8192))
    xr = E.permute_vector(W.deterministic_vector(n, 0), e.plan)
    y, _ = E.spmv_ehyb(e, xr)
    ok &= check("pool", y, c_oracle.spmv_ehyb(e, xr))
    # 2. persistent CTAs (more partitions than resident CTAs)
    n, r, c, v = W.permute_symmetric(*W.stencil27(24, 24, 24), seed=4)
    e = E.build_ehyb(E.CooMatrix(n, n, r, c, v), tau=8, profile=E.DeviceProfile(300, 32, 2048))
    xr = E.permute_vector(W.deterministic_vector(n, 6), e.plan)
    y, _ = E.spmv_ehyb(e, xr)
    ok &= check("persistent", y, c_oracle.spmv_ehyb(e, xr))
    # 2b. fp32 one-wave (chunk metadata in shared memory, paired ER slices)
    # and persistent CTAs in cost order (unit -> partition table)
    n, r, c, v = W.permute_symmetric(*W.stencil27(20, 20, 20), seed=3)
    e = E.build_ehyb(E.CooMatrix(n, n, r, c, v), tau=4, profile=E.DeviceProfile(16, 32, 8192))
    xr = E.permute_vector(W.deterministic_vector(n, 1), e.plan).astype(np.float32)
    y, _ = E.spmv_ehyb(e, xr)
    ok &= check("fp32 metadata in smem", y, c_oracle.spmv_ehyb(e, xr))
    os.environ["EHYB_ORDER_UNITS"] = "1"
    n, r, c, v = W.permute_symmetric(*W.stencil27(24, 24, 24), seed=5)
    e = E.build_ehyb(E.CooMatrix(n, n, r, c, v), tau=8, profile=E.DeviceProfile(300, 32, 2048))
    xr = E.permute_vector(W.deterministic_vector(n, 6), e.plan)
    y, _ = E.spmv_ehyb(e, xr)
    ok &= check("persistent, cost-ordered units", y, c_oracle.spmv_ehyb(e, xr))
    del os.environ["EHYB_ORDER_UNITS"]
    # 3. long rows, strict / default / fma
    n, r, c, v = W.heavy_tail(k=12, n_hubs=3, min_len=200, max_len=2000)
    e = E.build_ehyb(E.CooMatrix(n, n, r, c, v), tau=8, profile=E.DeviceProfile(16, 32, 8192))
    os.environ["EHYB_LONG_ROW"] = "48"
    dm = DeviceMatrix(e, 0)
    xr = E.permute_vector(W.deterministic_vector(n, 2), e.plan)
    xt = torch.from_numpy(xr).cuda()
    want = c_oracle.spmv_ehyb(e, xr)
    ok &= check("long rows strict", dm.spmv(xt, exact=True).cpu().numpy(), want)
    yd = dm.spmv(xt).cpu().numpy()
    yf = dm.spmv(xt, fma=True).cpu().numpy()
    err = max(float(np.max(np.abs(yd - want))), float(np.max(np.abs(yf - want)))) / float(
        np.max(np.abs(want)))
    print(f"long rows default/fma: rel. error {err:.1e}", flush=True)
    ok &= err <= 1e-12
    dm.close()
    del os.environ["EHYB_LONG_ROW"]
    # 4. shards: local launch then halo launch, two ranks' handles
    n, r, c, v = W.permute_symmetric(*W.stencil27(16, 16, 16), seed=2)
    e = E.build_ehyb(E.CooMatrix(n, n, r, c, v), tau=4, profile=E.DeviceProfile(8, 32, 4096))
    xr = E.permute_vector(W.deterministic_vector(n, 3), e.plan)
    want = c_oracle.spmv_ehyb(e, xr)
    for rank in range(2):
        plan = D.plan_for(e, rank, 2)
        A = D.DistributedEhyb(e, device=0, plan=plan)
        lo, hi = plan.p0 * plan.vec, plan.p1 * plan.vec
        x_ext = A.new_ext()
        x_ext[: plan.local_rows] = torch.from_numpy(xr[lo:hi])
        x_ext[plan.local_rows:] = torch.from_numpy(xr[plan.halo_cols])
        ys = torch.empty(plan.local_rows, dtype=torch.float32, device="cuda:0")
        A.spmv_local(x_ext, ys, exact=True)
        torch.cuda.synchronize()
        ok &= check(f"shard {rank}/2", ys.cpu().numpy(), want[lo:hi])
    print("ALL OK" if ok else "FAILURES", flush=True)
    return 0 if ok else 1


if __name__ == "__main__":
    sys.exit(main())
