#!/usr/bin/env python3
"""HBM read ceiling for context (the roofline denominator is the measured
copy bandwidth in MEASURED_PEAKS.json): a 2 GiB fp32 tensor reduced with
torch.sum (read-only stream) and copied (read + write), CUDA-event timed,
best of 10. One JSON line."""
import json

import torch

n = 512 << 20  # 2 GiB of fp32
a = torch.ones(n, dtype=torch.float32, device="cuda")
b = torch.empty_like(a)


def best(fn, reps=10):
    fn()
    torch.cuda.synchronize()
    out = []
    for _ in range(reps):
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        fn()
        e1.record()
        e1.synchronize()
        out.append(e0.elapsed_time(e1) / 1e3)
    return min(out)


t_read = best(lambda: a.sum())
t_copy = best(lambda: b.copy_(a))
print(json.dumps({"read_gbs": 4 * n / t_read / 1e9, "copy_gbs": 8 * n / t_copy / 1e9,
                  "bytes": 4 * n}))
