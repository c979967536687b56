#!/usr/bin/env python3
"""Dev tool: time the device-matrix creation (upload + derived layout) of
one config, three times. python scripts/upload_probe.py cfg5"""
import os
import sys
import time

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import torch  # noqa: E402

import bench  # noqa: E402
import paper_2204_06666_b200 as E  # noqa: E402
from paper_2204_06666_b200.device import DeviceMatrix  # noqa: E402

cfg = sys.argv[1]
m, e, _ = bench.build_workload(cfg)
for i in range(3):
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    dm = DeviceMatrix(e, 0)
    torch.cuda.synchronize()
    dt = time.perf_counter() - t0
    print(cfg, "staged" if os.environ.get("EHYB_UPLOAD_STAGED", "1") != "0" else "plain",
          f"create {dt:.3f} s, {dm.info()['device_bytes'] / 1e9:.2f} GB", flush=True)
    dm.close()
