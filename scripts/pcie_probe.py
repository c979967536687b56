#!/usr/bin/env python3
"""PCIe ceiling for the end-to-end path: pinned H2D alone, D2H alone, and
both at once on two streams, for the cfg2 vector size (16.7 MB). Prints one
JSON line (GB/s per direction)."""
import json
import time

import torch

nb = 2_097_152 * 8
reps = 100
h_src = torch.empty(nb, dtype=torch.uint8).pin_memory()
h_dst = torch.empty(nb, dtype=torch.uint8).pin_memory()
d_a = torch.empty(nb, dtype=torch.uint8, device="cuda")
d_b = torch.empty(nb, dtype=torch.uint8, device="cuda")
s_in, s_out = torch.cuda.Stream(), torch.cuda.Stream()


def run(h2d, d2h):
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    for _ in range(reps):
        if h2d:
            with torch.cuda.stream(s_in):
                d_a.copy_(h_src, non_blocking=True)
        if d2h:
            with torch.cuda.stream(s_out):
                h_dst.copy_(d_b, non_blocking=True)
    torch.cuda.synchronize()
    return nb * reps / (time.perf_counter() - t0) / 1e9


run(True, True)
out = {"bytes": nb, "h2d_gbs": run(True, False), "d2h_gbs": run(False, True),
       "both_gbs_each": run(True, True)}
out["e2e_floor_ms_per_vector"] = nb / 1e9 / out["both_gbs_each"] * 1e3
print(json.dumps(out))
