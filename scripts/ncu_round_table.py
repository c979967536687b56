#!/usr/bin/env python3
"""Dev tool: profiles/<tag>_summary.md from a round's raw ncu CSVs
(profiles/ncu_<tag>/prof_<tag>_<cfg>.raw.csv) and bench lines.
    python scripts/ncu_round_table.py <tag> <final HEAD>"""
import csv
import json
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
tag, head = sys.argv[1], sys.argv[2]
P = os.path.join(ROOT, "profiles")


def raw(path):
    r = list(csv.reader(open(path)))
    return {k: (v, u) for k, u, v in zip(r[0], r[1], r[2])}


def num(d, k):
    return float(d[k][0].replace(",", ""))


def us(d):
    t = num(d, "gpu__time_duration.sum")
    return t if d["gpu__time_duration.sum"][1] == "us" else t / 1e3


def nbytes(d, k):
    v, u = d[k]
    return float(v.replace(",", "")) * {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9}.get(u, 1)


names = {"cfg2": "cfg2 (fp64, K=1)", "cfg3f32": "cfg3 fp32 (K=1)", "cfg3f64": "cfg3 fp64 (K=2, persistent)",
         "cfg5": "cfg5 (fp64, K=4, persistent)", "cfg1": "cfg1 (fp64, small)",
         "cfg4": "cfg4 (fp64, hub rows, default mode)"}
out = [f"# ncu captures {tag}: every config, one fused launch each", "",
       f"`bash scripts/gpu_final.sh {tag}` on one B200 at HEAD {head} (`ncu --set full --clock-control none "
       "--import-source on -k regex:spmv_fused -s 5 -c 1`, launches from `scripts/launch_once.py`, default "
       f"arithmetic mode). Per-config tables: `profiles/{tag}_<config>.md`; raw CSVs: `profiles/ncu_{tag}/`. "
       "ncu times are cold-cache and serialised; the DRAM traffic per launch is `bench.py`'s `roofline.traffic` "
       "(`profiles/ncu_traffic.json`).", "",
       "| config | ncu us | DRAM traffic / algorithmic bytes | DRAM % of ncu peak | L2 read hit | issue active | "
       "long-scoreboard stalls / issue | smem bank-conflict wavefronts / all |",
       "|---|---|---|---|---|---|---|---|"]
for c in ["cfg2", "cfg3f32", "cfg3f64", "cfg5", "cfg1", "cfg4"]:
    d = raw(os.path.join(P, f"ncu_{tag}", f"prof_{tag}_{c}.raw.csv"))
    j = os.path.join(P, f"bench_{tag}_{'default' if c == 'cfg2' else c}.json")
    jd = json.loads([l for l in open(j).read().splitlines() if l.startswith("{")][-1])
    bmin = jd["roofline"]["algorithmic_bytes_per_launch"]
    tr = nbytes(d, "dram__bytes_read.sum") + nbytes(d, "dram__bytes_write.sum")
    out.append(f"| {names[c]} | {us(d):.1f} | {tr / 1e6:.1f} / {bmin / 1e6:.1f} MB = {tr / bmin:.3f} | "
               f"{num(d, 'gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed'):.1f} | "
               f"{num(d, 'lts__t_sector_op_read_hit_rate.pct'):.1f}% | "
               f"{num(d, 'smsp__issue_active.avg.pct_of_peak_sustained_active'):.1f}% | "
               f"{num(d, 'smsp__average_warps_issue_stalled_long_scoreboard_per_issue_active.ratio'):.1f} | "
               f"{num(d, 'l1tex__data_bank_conflicts_pipe_lsu_mem_shared_op_ld.sum') / 1e6:.2f}M / "
               f"{num(d, 'l1tex__data_pipe_lsu_wavefronts_mem_shared_op_ld.sum') / 1e6:.2f}M |")
out += ["", "ER-only launches (`launch_once.py --mode er`: the spill path alone, its L2 traffic is the ER "
        "slices and their x gathers):", "",
        "| config | ER-only us | L2 read hit rate | DRAM % of peak | long-scoreboard stalls / issue |",
        "|---|---|---|---|---|"]
for c in ["cfg2", "cfg3f32"]:
    d = raw(os.path.join(P, f"ncu_{tag}", f"prof_{tag}_{c}_er.raw.csv"))
    out.append(f"| {c} | {us(d):.1f} | {num(d, 'lts__t_sector_op_read_hit_rate.pct'):.1f}% | "
               f"{num(d, 'gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed'):.1f} | "
               f"{num(d, 'smsp__average_warps_issue_stalled_long_scoreboard_per_issue_active.ratio'):.1f} |")
open(os.path.join(P, f"{tag}_summary.md"), "w").write("\n".join(out) + "\n")
print("\n".join(out))
