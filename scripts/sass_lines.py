#!/usr/bin/env python3
"""Dev tool: attribute an ncu SASS source-page export (per-instruction
executed counts and stall samples) to kernels.cuh lines via nvdisasm -g of the
built library. python scripts/sass_lines.py <prof.sass.csv> <mangled kernel> [top]"""
import csv
import os
import re
import subprocess
import sys
import tempfile
from collections import defaultdict

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
csv_path, kern = sys.argv[1], sys.argv[2]
top = int(sys.argv[3]) if len(sys.argv) > 3 else 40
if os.environ.get("SASS_FILE"):  # nvdisasm -g output of the library the profile ran
    sass = open(os.environ["SASS_FILE"]).read()
else:
    tmp = tempfile.mkdtemp()
    subprocess.run(["cuobjdump", "-xelf", "all", os.path.join(ROOT, "paper_2204_06666_b200", "libehyb_b200.so")],
                   cwd=tmp, capture_output=True)
    cub = [f for f in os.listdir(tmp) if f.startswith("device.") and f.endswith(".cubin")][0]
    sass = subprocess.run(["nvdisasm", "-g", os.path.join(tmp, cub)], capture_output=True, text=True).stdout
lines = sass.splitlines()
start = next(i for i, l in enumerate(lines) if l.startswith(".text." + kern + ":"))
off2line = {}
cur = None
for l in lines[start + 1:]:
    if l.startswith(".text.") or l.startswith(".nv."):
        break
    m = re.search(r'line (\d+)', l)
    if "//## File" in l and m:
        cur = int(m.group(1))
        continue
    m = re.match(r'\s*/\*([0-9a-f]{4,})\*/', l)
    if m:
        off2line[int(m.group(1), 16)] = cur
rows = list(csv.reader(open(csv_path)))
hdr = rows[1]
ia, ie, iss = hdr.index("Address"), hdr.index("Instructions Executed"), hdr.index("Warp Stall Sampling (All Samples)")
data = [r for r in rows[2:] if len(r) == len(hdr)]
base = int(data[0][ia], 16)
inst = defaultdict(int)
stall = defaultdict(int)
for r in data:
    ln = off2line.get(int(r[ia], 16) - base)
    inst[ln] += int(float(r[ie] or 0))
    stall[ln] += int(float(r[iss] or 0))
src = open(os.path.join(ROOT, "paper_2204_06666_b200", "csrc", "kernels.cuh")).read().splitlines()
ti, ts = sum(inst.values()), sum(stall.values())
print(f"total warp instructions {ti}, stall samples {ts}")
for key, name in ((inst, "instructions"), (stall, "stall samples")):
    print(f"== top lines by {name}")
    for ln, v in sorted(key.items(), key=lambda kv: -kv[1])[:top]:
        txt = src[ln - 1].strip()[:90] if ln else "?"
        print(f"{ln!s:>5} {100*inst[ln]/ti:5.1f}% inst {100*stall[ln]/max(ts,1):5.1f}% stall  {txt}")
