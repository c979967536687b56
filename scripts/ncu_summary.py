#!/usr/bin/env python3
"""Summarise ncu captures (run here, no GPU needed) into profiles/.

    python scripts/ncu_summary.py --rep gpurun_out/prof_r05.ncu-rep \
        --launches gpurun_out/launches_r05.csv --config cfg2 --tag r1_final

Writes profiles/<tag>_<config>.md (human summary) and merges the per-launch
DRAM traffic into profiles/ncu_traffic.json (read by bench.py for the
`roofline.traffic` field).
"""

from __future__ import annotations

import argparse
import csv
import io
import json
import os
import statistics
import subprocess

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
PROFILES = os.path.join(ROOT, "profiles")

METRICS = [
    ("gpu__time_duration.sum", "kernel duration"),
    ("dram__bytes_read.sum", "DRAM read"),
    ("dram__bytes_write.sum", "DRAM write"),
    ("dram__bytes.sum.per_second", "DRAM throughput"),
    ("gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed", "DRAM % of peak (ncu)"),
    ("lts__t_sector_hit_rate.pct", "L2 hit rate"),
    ("lts__t_sector_op_read_hit_rate.pct", "L2 read hit rate"),
    ("l1tex__t_sector_hit_rate.pct", "L1 hit rate"),
    ("sm__throughput.avg.pct_of_peak_sustained_elapsed", "SM throughput % of peak"),
    ("smsp__average_warps_issue_stalled_barrier_per_issue_active.ratio", "barrier stalls / issue"),
    ("smsp__average_warps_issue_stalled_membar_per_issue_active.ratio", "membar stalls / issue"),
    ("smsp__average_warps_issue_stalled_short_scoreboard_per_issue_active.ratio",
     "short-scoreboard stalls / issue"),
    ("smsp__average_warps_issue_stalled_lg_throttle_per_issue_active.ratio", "LG-throttle stalls / issue"),
    ("sm__warps_active.avg.pct_of_peak_sustained_active", "achieved occupancy"),
    ("smsp__issue_active.avg.pct_of_peak_sustained_active", "issue active"),
    ("smsp__average_warps_issue_stalled_long_scoreboard_per_issue_active.ratio",
     "long-scoreboard stalls / issue"),
    ("l1tex__data_bank_conflicts_pipe_lsu_mem_shared_op_ld.sum", "smem load bank conflicts"),
    ("l1tex__data_pipe_lsu_wavefronts_mem_shared_op_ld.sum", "smem load wavefronts"),
    ("launch__registers_per_thread", "registers / thread"),
    ("launch__shared_mem_per_block_dynamic", "dynamic smem / CTA"),
    ("launch__grid_size", "grid"),
    ("launch__block_size", "block"),
]


def raw_rows(rep):
    if rep.endswith(".csv"):  # `ncu -i <rep> --page raw --csv` exported on the GPU box
        with open(rep) as fh:
            out = fh.read()
    else:
        out = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True,
                             text=True, check=True).stdout
    rows = list(csv.reader(io.StringIO(out)))
    hdr, units = rows[0], rows[1]
    return [dict(zip(hdr, zip(r, units))) for r in rows[2:]]


def to_bytes(val, unit):
    scale = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9}.get(unit, 1)
    return float(val.replace(",", "")) * scale


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--rep", required=True)
    ap.add_argument("--launches")
    ap.add_argument("--config", default="cfg2")
    ap.add_argument("--tag", required=True)
    ap.add_argument("--bmin", type=float, default=None, help="algorithmic bytes per launch")
    args = ap.parse_args()
    os.makedirs(PROFILES, exist_ok=True)
    kernels = raw_rows(args.rep)
    lines = [f"# ncu summary — {args.tag} ({args.config})", "",
             f"source: `{os.path.basename(args.rep)}` (`ncu --set full --clock-control none "
             "--import-source on`, one launch of the fused kernel; cold-cache, serialised)", ""]
    traffic = None
    for k in kernels:
        name = k.get("Kernel Name", ("?",))[0]
        lines += [f"## {name}", "", "| metric | value | unit |", "|---|---|---|"]
        for key, label in METRICS:
            if key in k:
                v, u = k[key]
                lines.append(f"| {label} (`{key}`) | {v} | {u} |")
        rd = to_bytes(*k["dram__bytes_read.sum"]) if "dram__bytes_read.sum" in k else 0.0
        wr = to_bytes(*k["dram__bytes_write.sum"]) if "dram__bytes_write.sum" in k else 0.0
        traffic = rd + wr
        lines += ["", f"DRAM traffic per launch: {traffic / 1e6:.1f} MB"]
        if args.bmin:
            lines.append(f"algorithmic bytes per launch: {args.bmin / 1e6:.1f} MB "
                         f"(traffic / algorithmic = {traffic / args.bmin:.3f})")
        lines.append("")
    if args.launches and os.path.exists(args.launches):
        rows = list(csv.reader(open(args.launches)))
        hdr = next(i for i, r in enumerate(rows) if "Kernel Name" in r)
        h = rows[hdr]
        per = {}
        for r in rows[hdr + 1:]:
            if len(r) != len(h):
                continue
            d = dict(zip(h, r))
            if d.get("Metric Name") == "gpu__time_duration.sum":
                per.setdefault(d["Kernel Name"], []).append(float(d["Metric Value"].replace(",", "")))
        total = sum(sum(v) for v in per.values())
        lines += ["## launch list (`--metrics gpu__time_duration.sum`)", "",
                  "| kernel | launches | median ns | share of listed time |", "|---|---|---|---|"]
        for name, v in sorted(per.items(), key=lambda kv: -sum(kv[1])):
            lines.append(f"| {name} | {len(v)} | {statistics.median(v):.0f} | "
                         f"{sum(v) / total:.1%} |")
        lines.append("")
    md = os.path.join(PROFILES, f"{args.tag}_{args.config}.md")
    with open(md, "w") as fh:
        fh.write("\n".join(lines))
    tj = os.path.join(PROFILES, "ncu_traffic.json")
    data = json.load(open(tj)) if os.path.exists(tj) else {}
    if traffic is not None:
        data[args.config] = {"dram_bytes_per_launch": traffic, "source": os.path.basename(md)}
    with open(tj, "w") as fh:
        json.dump(data, fh, indent=1, sort_keys=True)
    print(md)


if __name__ == "__main__":
    main()
