#!/usr/bin/env python3
"""Dev tool: build libehyb_b200.so with `ptxas -v` and print registers /
spills of the fused SpMV kernel variants (T, STRICT, C32, SMEM, RING, P2P).

    EHYB_NVCC_FLAGS="-DEHYB_VEC_UB_F64=3" python scripts/ptxas_report.py
"""
import os
import re
import subprocess
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
r = subprocess.run([sys.executable, os.path.join(ROOT, "paper_2204_06666_b200", "build.py"),
                    "--force", "-v"], capture_output=True, text=True)
cur = None
rows = []
for ln in (r.stdout + r.stderr).splitlines():
    m = re.search(r"Compiling entry function '(\S+)'", ln)
    if m:
        cur = m.group(1)
        continue
    if cur is None:
        continue
    m = re.search(r"(\d+) bytes spill stores, (\d+) bytes spill loads", ln)
    if m:
        spill = (int(m.group(1)), int(m.group(2)))
        continue
    m = re.search(r"Used (\d+) registers", ln)
    if m:
        rows.append((cur, int(m.group(1)), spill))
        cur = None
for name, regs, (ss, sl) in rows:
    m = re.match(r"_ZN4ehyb17spmv_fused_kernelI([fd])Li(\d)E(.*)EEvNS_10SpmvParams", name)
    if not m:
        continue
    flags = "".join("1" if b == "1" else "0" for b in re.findall(r"Lb(\d)E?", m.group(3)))
    mode = {"0": "strict", "1": "fma", "2": "default"}[m.group(2)]
    print(f"fused<{m.group(1)}, {mode:7s} C32 SMEM RING P2P={flags}> regs={regs} spill st/ld={ss}/{sl}")
