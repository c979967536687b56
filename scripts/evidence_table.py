#!/usr/bin/env python3
"""Dev tool: DESIGN.md §4 rows from a round's bench JSON lines.
    python scripts/evidence_table.py <tag>   (reads profiles/bench_<tag>_*.json)"""
import json
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
tag = sys.argv[1]
order = ["default", "cfg1", "cfg3f32", "cfg3f64", "cfg4", "cfg4_exact", "cfg5", "dist_cfg5"]
for c in order:
    f = os.path.join(ROOT, "profiles", f"bench_{tag}_{c}.json")
    if not os.path.exists(f):
        continue
    lines = [l for l in open(f).read().splitlines() if l.startswith("{")]
    if not lines:
        print(c, "no JSON line")
        continue
    d = json.loads(lines[-1])
    k, r, e = d.get("kernel", {}), d["roofline"], d.get("e2e", {})
    g = (k.get("cuda_graph") or {}).get("us_per_spmv")
    cus = (d.get("cusparse") or {}).get("ehyb_speedup_vs_best")
    cpu = (d.get("cpu_baseline") or {}).get("value")
    pre = d.get("preprocessing") or {}
    print(f"{c}: {d['ms_per_step']*1e3:.1f} us (graph {g and round(g, 1)}, L2-res {k.get('l2_resident_avg_us') and round(k['l2_resident_avg_us'], 1)}) "
          f"{d['value']:.0f} GF/s, {r['achieved']:.0f} GB/s, frac {r['frac']:.3f} (peak {r['peak']}), traffic {r.get('traffic')}, "
          f"cuSPARSE x{cus and round(cus, 2)}, e2e {e.get('value') and round(e['value'], 1)} (sync {((e.get('sync_call') or {}).get('value') or 0):.0f}), "
          f"cpu {cpu and round(cpu, 1)}, prep {pre.get('partition_s') and round(pre['partition_s'], 2)} + {pre.get('reorder_assemble_s') and round(pre['reorder_assemble_s'], 2)} s "
          f"({d.get('prep_to_spmv_ratio') or pre.get('spmv_equivalents')}), clocks {d.get('clocks', {}).get('sm_mhz')} {d.get('clocks', {}).get('reasons')}, parity {str(d.get('parity'))[:60]}")
