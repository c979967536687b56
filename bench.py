#!/usr/bin/env python3
"""EHYB SpMV benchmark (BASELINE.json metric: SpMV GFLOP/s = 2*nnz/t and
achieved HBM GB/s vs peak).

    python bench.py [--gpus N] [--steps K] [--warmup W] [--config cfg2]
    python bench.py --impl reference ...      # the reference CPU engine arm

One step = one EHYB SpMV y = A x over the whole matrix (one fused kernel
launch). N=1 workload: BASELINE configs[1] (cfg2: 27-point 128^3 stencil,
random symmetric permutation, fp64). Prints ONE JSON line (rank 0).
"""

from __future__ import annotations

import argparse
import json
import os
import statistics
import subprocess
import sys
import threading
import time

import numpy as np

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

METRIC = "SpMV GFLOP/s (2*nnz/t) and achieved HBM GB/s vs peak"
UNIT = "GFLOP/s"
FALLBACK_HBM_GBS = 6650.0
SPEC_HBM_GBS = 8000.0  # B200 HBM3e datasheet (SURVEY.md 8d secondary denominator)


def log(*a):
    print(*a, file=sys.stderr, flush=True)


def measured_peak():
    path = os.path.join(ROOT, "MEASURED_PEAKS.json")
    try:
        with open(path) as fh:
            return float(json.load(fh)["hbm_gbs"]), "measured (MEASURED_PEAKS.json hbm_gbs)"
    except Exception:
        return FALLBACK_HBM_GBS, "fallback (B200_PROFILING.md)"


class ClockSampler:
    """nvidia-smi clocks / throttle reasons sampled during the timed region."""

    FIELDS = ("clocks.sm,clocks.max.sm,clocks_event_reasons.active,"
              "clocks_event_reasons.hw_slowdown,clocks_event_reasons.hw_thermal_slowdown,"
              "clocks_event_reasons.sw_thermal_slowdown,clocks_event_reasons.sw_power_cap")

    def __init__(self, index: int):
        self.index = index
        self.proc = None
        self.lines = []

    def __enter__(self):
        try:
            self.proc = subprocess.Popen(
                ["nvidia-smi", "-i", str(self.index), f"--query-gpu={self.FIELDS}",
                 "--format=csv,noheader,nounits", "-lms", "20"],
                stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
            self.t = threading.Thread(target=self._read, daemon=True)
            self.t.start()
        except Exception:
            self.proc = None
        return self

    def _read(self):
        for line in self.proc.stdout:
            self.lines.append(line.strip())

    def __exit__(self, *exc):
        if self.proc:
            self.proc.terminate()
            try:
                self.proc.wait(timeout=5)
            except Exception:
                self.proc.kill()
            self.t.join(timeout=2)

    def summary(self):
        sm, mx, reasons = [], None, set()
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        for ln in self.lines:
            parts = [p.strip() for p in ln.split(",")]
            if len(parts) < 7:
                continue
            try:
                sm.append(float(parts[0]))
                mx = float(parts[1])
            except ValueError:
                continue
            for nm, flag in zip(names, parts[3:7]):
                if flag.lower() == "active":
                    reasons.add(nm)
        if not sm:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": [], "samples": 0}
        return {"sm_mhz": statistics.median(sm), "sm_max_mhz": mx, "reasons": sorted(reasons),
                "samples": len(sm)}


def build_workload(name: str):
    """Matrix + native preprocessing (timed like cli.py:199-219)."""
    import paper_2204_06666_b200 as E
    from paper_2204_06666_b200 import workloads as W

    t0 = time.perf_counter()
    n, r, c, v, tau = W.build_config(name)
    t_gen = time.perf_counter() - t0
    m = E.CooMatrix(n, n, r, c, v)
    del r, c, v
    prof = W.CONFIG_PROFILES.get(name)
    params = E.compute_params(n, tau, E.DeviceProfile(*prof) if prof else E.B200_PROFILE)
    if os.environ.get("EHYB_BENCH_PREP", "gpu") == "host":  # e.g. launch lists: no prep kernels
        t0 = time.perf_counter()
        g = E.build_graph(m)
        tg = time.perf_counter()
        parts = E.partition_graph(g, params.n_parts, params.vec_cache_size, seed=0)
        t1 = time.perf_counter()
        cls = E.classify_rows(m, parts)
        plan = E.build_reorder_plan(cls, params, parts)
        e = E.assemble_ehyb(m, plan, params, parts)
        t2 = time.perf_counter()
        return m, e, dict(generate_s=t_gen, partition_s=t1 - t0, reorder_assemble_s=t2 - t1,
                          build_graph_s=tg - t0, partition_graph_s=t1 - tg, where="host")
    # GPU preprocessing (build_graph, classify / reorder / assemble on the
    # device, the BFS partitioner on the host); byte-identical to the host path.
    # A tiny matrix first loads the preprocessing kernels' modules (a one-time
    # per-process cost of CUDA lazy loading, ~0.4 s), so the timing below is
    # the steady-state pipeline
    nw, rw, cw, vw = W.stencil27(8, 8, 8)
    E.build_ehyb_gpu(E.CooMatrix(nw, nw, rw, cw, vw), tau=tau, profile=E.DeviceProfile(4, 32, 8192),
                     device=0)
    # the first build of a large matrix also pays one-time allocations
    # (process-wide pinned staging, device scratch): reported as first_call;
    # the timings are of a second, steady-state build of the same matrix
    t, first = {}, None
    for rep in range(2 if os.environ.get("EHYB_BENCH_PREP_REPEAT", "1") != "0" else 1):
        t = {}
        t0 = time.perf_counter()
        e = E.build_ehyb_gpu(m, tau=tau, profile=E.DeviceProfile(*prof) if prof else E.B200_PROFILE,
                             device=0, timings=t)
        total = time.perf_counter() - t0
        if rep == 0:
            first = dict(t, total_s=total)
    assert e.params == params
    return m, e, dict(generate_s=t_gen, first_call=first,
                      partition_s=t["upload_s"] + t["build_graph_s"] + t["partition_graph_s"],
                      reorder_assemble_s=t["reorder_assemble_s"], upload_s=t["upload_s"],
                      build_graph_s=t["build_graph_s"], partition_graph_s=t["partition_graph_s"],
                      total_s=total, where="GPU (build_graph, classify/reorder/assemble) + host "
                                           "(BFS partition_graph); kernel modules loaded "
                                           "beforehand (one-time lazy-loading cost excluded); "
                                           "steady state = the second build of the matrix")


def golden_y_digest(name: str):
    path = os.path.join(ROOT, "tests", "golden", f"config_{name}.json")
    if not os.path.exists(path):
        return None
    with open(path) as fh:
        return json.load(fh)


def cpu_engine_sample(e, xr, budget_s: float, threads: int):
    """Time the C restatement of the reference engine (oracle/) on a bounded
    sample: whole product if it fits the budget, else the first partitions /
    ER slices. Returns (gflops, seconds per sample, flops per sample, desc)."""
    from oracle import c_oracle

    prep = c_oracle.Prepared(e)
    y = np.empty(e.padded_dimension, prep.dt)
    t0 = time.perf_counter()
    prep.spmv(xr, threads, out=y)
    t_full = time.perf_counter() - t0
    nnz_full = e.nnz
    if t_full <= budget_s:
        parts, er = (0, e.n_parts), (0, prep.n_er_slices)
        flops = 2 * nnz_full
        desc = "full product"
    else:
        frac = max(budget_s / t_full, 1.0 / e.n_parts)
        p_hi = max(1, int(e.n_parts * frac))
        s_hi = int(prep.n_er_slices * frac)
        parts, er = (0, p_hi), (0, s_hi)
        vec = e.params.vec_cache_size
        nnz_ell = int(e.ell_row_widths[: p_hi * vec].sum())
        nnz_er = int(e.er_row_widths[: s_hi * e.params.warp_size].sum())
        flops = 2 * (nnz_ell + nnz_er)
        desc = f"partitions [0,{p_hi}) of {e.n_parts} + ER slices [0,{s_hi}) of {prep.n_er_slices}"
    return prep, parts, er, y, flops, desc


def reference_workload(args):
    """The workload our arm runs for this N (config name, profile), built by
    the ORACLE's C restatement of the reference preprocessing — no product
    code or library on this path."""
    from paper_2204_06666_b200 import workloads as W

    world = int(os.environ.get("WORLD_SIZE", "1"))
    g = max(world, args.gpus)
    name = args.config if g <= 1 else dist_config_name(args, g)
    n, r, c, v, tau = W.build_config(name) if name in W.CONFIGS else _weak_matrix(g)
    profile = W.CONFIG_PROFILES.get(name) or dist_profile(args, g)
    return name, n, r, c, v, tau, profile


def run_reference(args):
    """--impl reference: the reference's CPU SpMV path (engine.py:108-216) on
    the box's host cores. The reference is pure Python (nothing to compile),
    so per the tier rules the arm times the oracle port: the EHYB arrays come
    from oracle/ehyb_prep_oracle.c (the C restatement of the reference
    preprocessing, checked against the reference's own digests), the SpMV
    from oracle/ehyb_oracle.c with all host threads. Rank 0 only."""
    rank = int(os.environ.get("RANK", "0"))
    if rank != 0:
        return 0
    from golden_util import digest
    from oracle import c_oracle, c_prep
    from paper_2204_06666_b200 import workloads as W

    name, n, r, c, v, tau, profile = reference_workload(args)
    args.config = name
    prep_t = {}
    t0 = time.perf_counter()
    e = c_prep.build_ehyb(n, r, c, v, tau, tuple(profile), timings=prep_t)
    prep_t["total_s"] = time.perf_counter() - t0
    nnz = int(r.size)
    del r, c, v
    gold = golden_y_digest(name)
    parity = "no golden record for this config"
    if gold is not None:
        if digest(e.val_ell) != gold["digests"]["val_ell"] or \
                digest(e.col_er) != gold["digests"]["col_er"]:
            raise SystemExit("reference arm: EHYB arrays differ from the reference's digests")
        parity = "EHYB arrays == the reference's digests"
    x = W.deterministic_vector(n, 0)
    xr = np.zeros(e.padded_dimension, np.float32 if tau == 4 else np.float64)
    xr[e.plan.reorder_table[:n]] = x
    threads = len(os.sched_getaffinity(0))
    per_step_budget = max(0.05, 120.0 / max(1, args.steps + args.warmup))
    prep, parts, er, y, flops, desc = cpu_engine_sample(e, xr, per_step_budget, threads)
    if gold is not None and desc == "full product":
        ok = digest(y) == gold["y_reordered"]
        parity += "; y == the reference's y digest" if ok else "; y MISMATCH"
    for _ in range(args.warmup):
        prep.spmv(xr, threads, out=y, parts=parts, er_slices=er)
    t0 = time.perf_counter()
    for _ in range(args.steps):
        prep.spmv(xr, threads, out=y, parts=parts, er_slices=er)
    dt = (time.perf_counter() - t0) / args.steps
    value = flops / dt / 1e9
    desc_full = (f"{desc} per step ({flops} flops); SpMV = oracle/ehyb_oracle.c (C restatement "
                 f"of engine.py spmv_ehyb, OpenMP), arrays = oracle/ehyb_prep_oracle.c")
    ref_py = (reference_python_engine(e, xr, name)
              if not args.no_ref_python and e.dimension <= 6_000_000 else None)
    out = {
        "impl": "reference", "metric": METRIC, "value": value, "unit": UNIT,
        "n_gpus": args.gpus, "steps": args.steps, "warmup": args.warmup,
        "ms_per_step": dt * 1e3, "higher_is_better": True, "scaling": "weak",
        "vs_baseline": None, "dtype": "f64" if tau == 8 else "f32",
        "data": "synthetic", "config": config_block(args, None, e, nnz=nnz),
        "cpu_baseline": {"value": value, "unit": UNIT, "cores": threads, "kind": "port",
                         "sample": desc_full},
        "e2e": {"value": value, "unit": UNIT, "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
        "parity": parity,
        "preprocessing_s": dict(prep_t, source="oracle/ehyb_prep_oracle.c (C restatement of the "
                                               "reference preprocessing), host threads"),
        "reference_python_preprocessing_s": (gold or {}).get("timings"),
        "reference_python_engine": ref_py,
        "repo_libraries_mapped": repo_libraries_mapped(),
    }
    print(json.dumps(out), flush=True)
    return 0


def repo_libraries_mapped():
    """Shared objects from this repo mapped into the process (the reference
    arm must show only oracle/ libraries)."""
    try:
        with open("/proc/self/maps") as fh:
            libs = {ln.split()[-1] for ln in fh if ln.rstrip().endswith(".so")}
    except OSError:
        return None
    return sorted(os.path.relpath(p, ROOT) for p in libs if p.startswith(ROOT))


def reference_python_engine(e, xr, name):
    """One call of the UNMODIFIED reference engine (`ehyb.spmv_ehyb`, the
    pure-Python simulator installed into baseline/_ref) on the same arrays:
    how the reference itself runs this path (GIL-bound, ~1 core)."""
    ref = os.path.join(ROOT, "baseline", "_ref")
    if not os.path.isdir(os.path.join(ref, "ehyb")):
        return {"unavailable": "baseline/_ref not installed"}
    code = r"""
import json, sys, time, numpy as np
sys.path.insert(0, sys.argv[1])
import ehyb
d = np.load(sys.argv[2], allow_pickle=False)
p = ehyb.EhybParams(k=int(d['k']), n_parts=int(d['n_parts']), vec_cache_size=int(d['vec']),
                    tau=int(d['tau']), warp_size=int(d['warp']))
plan = ehyb.ReorderPlan(reorder_table=d['reorder'], inverse_table=d['inverse'],
                        arrange_table=d['arrange'], y_idx_er=d['y_idx_er'],
                        n_er_rows=int(d['n_er']), dimension=int(d['n']),
                        padded_dimension=int(d['padded']))
e = ehyb.EhybMatrix(params=p, plan=plan, dimension=int(d['n']), padded_dimension=int(d['padded']),
                    val_ell=d['val_ell'], col_ell=d['col_ell'], position_ell=d['position_ell'],
                    width_ell=d['width_ell'], part_boundary=d['part_boundary'],
                    ell_row_widths=d['ell_row_widths'], val_er=d['val_er'], col_er=d['col_er'],
                    position_er=d['position_er'], width_er=d['width_er'],
                    er_row_widths=d['er_row_widths'])
t0 = time.perf_counter()
y, st = ehyb.spmv_ehyb(e, d['xr'], ehyb.ExecutionConfig(worker_count=1))
dt = time.perf_counter() - t0
np.save(sys.argv[3], y)
print(json.dumps({"s": dt, "flops": int(st.flops)}))
"""
    import tempfile

    with tempfile.TemporaryDirectory() as td:
        arrs = os.path.join(td, "e.npz")
        p = e.params
        np.savez(arrs, k=p.k, n_parts=p.n_parts, vec=p.vec_cache_size, tau=p.tau, warp=p.warp_size,
                 n=e.dimension, padded=e.padded_dimension, n_er=e.plan.n_er_rows,
                 reorder=e.plan.reorder_table, inverse=e.plan.inverse_table,
                 arrange=e.plan.arrange_table, y_idx_er=e.plan.y_idx_er, xr=xr,
                 **{k: getattr(e, k) for k in ("val_ell", "col_ell", "position_ell", "width_ell",
                                                "part_boundary", "ell_row_widths", "val_er",
                                                "col_er", "position_er", "width_er",
                                                "er_row_widths")})
        yout = os.path.join(td, "y.npy")
        r = subprocess.run([sys.executable, "-c", code, ref, arrs, yout], capture_output=True,
                           text=True, timeout=900, env={**os.environ, "PYTHONPATH": ""})
        if r.returncode != 0:
            return {"unavailable": r.stderr.strip().splitlines()[-1][:200] if r.stderr else "failed"}
        res = json.loads(r.stdout.strip().splitlines()[-1])
        from golden_util import digest

        gold = golden_y_digest(name)
        y = np.load(yout)
        return {"value": res["flops"] / res["s"] / 1e9, "unit": UNIT, "s_per_spmv": res["s"],
                "cores": 1, "api": "ehyb.spmv_ehyb(e, x_r, ExecutionConfig(worker_count=1)) "
                                   "from baseline/_ref (unmodified reference)",
                "y_matches_reference_digest": None if gold is None
                else digest(y) == gold["y_reordered"]}


B200_PROFILE = (148, 32, 231424)


def dist_config_name(args, g: int) -> str:
    """The N > 1 workload: cfg5 (BASELINE configs[4], the 27-point 256^3
    stencil the north star's 8-GPU target is quoted on) unless --config
    names another; "weak" = the 128*N x 128 x 128 weak-scaling stencil."""
    return "cfg5" if args.config is None else args.config


def dist_profile(args, g: int):
    """G-independent structure (SURVEY.md 8e option i): every N uses the
    1-GPU B200 profile, so T_1 and T_N stream identical bytes; only the
    weak-scaling workload grows its partitions with N."""
    name = dist_config_name(args, g)
    if name == "weak":
        return (148 * g, 32, B200_PROFILE[2])
    from paper_2204_06666_b200 import workloads as W

    return W.CONFIG_PROFILES.get(name, B200_PROFILE)


def _weak_matrix(g: int):
    from paper_2204_06666_b200 import workloads as W

    n, r, c, v = W.permute_symmetric(*W.stencil27(128 * g, 128, 128), seed=1)
    return n, r, c, v, 8


def min_bytes_of(e) -> int:
    """SURVEY.md 8d minimum-bytes model: nnz_ell*(tau+2) + nnz_er*(tau+4) + 2*n*tau."""
    t = e.params.tau
    return int(e.nnz_ell * (t + 2) + e.nnz_er * (t + 4) + 2 * e.dimension * t)


L2_FLUSH_POLICY = ("L2 flushed before every timed step (a 512 MB write, then a 192 MB read so the "
                   "flush's dirty lines are written back outside the timed step); L2-resident "
                   "time reported separately")


def needs_l2_flush(e) -> bool:
    """A step whose minimum bytes are under 2x L2 would stay cache resident
    between back-to-back launches."""
    import torch

    l2 = torch.cuda.get_device_properties(torch.cuda.current_device()).L2_cache_size \
        if torch.cuda.is_available() else 126 << 20
    return min_bytes_of(e) < 2 * l2


class L2Flush:
    """Per-step L2 flush: write 512 MB (evicts every line the step could
    reuse), then read 192 MB of another buffer so the L2 holds clean lines —
    otherwise the ~126 MB of dirty lines the write leaves behind are written
    back DURING the timed step and charged to it (cfg4: ~10 us)."""

    def __init__(self, dev):
        import torch

        self.w = torch.empty(512 << 20, dtype=torch.uint8, device=f"cuda:{dev}")
        self.r = torch.ones(48 << 20, dtype=torch.float32, device=f"cuda:{dev}")
        self.out = torch.empty((), dtype=torch.float32, device=f"cuda:{dev}")

    def __call__(self, stream):
        import torch

        with torch.cuda.stream(stream):
            self.w.fill_(1)
            torch.sum(self.r, dim=0, out=self.out)


def config_block(args, m, e, nnz=None):
    from paper_2204_06666_b200 import workloads as W

    desc = (W.CONFIGS[args.config][0] if args.config in W.CONFIGS else
            f"27-point stencil {e.dimension // (128 * 128)}x128x128, random symmetric "
            f"permutation (the weak-scaling workload)")
    p = e.params
    prof = W.CONFIG_PROFILES.get(args.config, (p.n_parts // max(1, p.k), p.warp_size,
                                               B200_PROFILE[2]))
    return {
        "workload": f"{args.config}: {desc}",
        "n": int(e.dimension), "nnz": int(m.nnz if m is not None else nnz), "tau": int(p.tau),
        "profile": f"DeviceProfile{tuple(prof)}", "k": int(p.k),
        "n_parts": int(e.n_parts), "vec_cache_size": int(p.vec_cache_size),
        "nnz_ell": int(e.nnz_ell), "nnz_er": int(e.nnz_er),
        "l2_policy": ("inputs larger than L2 (matrix stream per step >= 2x L2)"
                      if not needs_l2_flush(e) else L2_FLUSH_POLICY),
        "parallelism": f"one CTA per partition x{e.n_parts}",
    }


def run_gpu(args):
    import torch

    import paper_2204_06666_b200 as E
    from paper_2204_06666_b200 import workloads as W
    from golden_util import digest

    world = int(os.environ.get("WORLD_SIZE", "1"))
    if world > 1 or args.gpus > 1 or args.dist:
        from paper_2204_06666_b200 import distributed as D

        return D.bench_main(args, ClockSampler)

    dev = 0
    torch.cuda.set_device(dev)
    m, e, prep_t = build_workload(args.config)
    nnz = m.nnz
    flops = 2 * nnz
    bmin = E.min_bytes(e)
    gold = golden_y_digest(args.config)

    t0 = time.perf_counter()
    dm = E.device_matrix(e, dev)  # upload + derived device layout (ehyb_dev_create)
    torch.cuda.synchronize(dev)
    prep_t["device_matrix_s"] = time.perf_counter() - t0
    prep_t["device_matrix_gbytes"] = dm.info()["device_bytes"] / 1e9
    info = dm.info()
    stream = torch.cuda.Stream(dev)
    x = W.deterministic_vector(e.dimension, 0)
    xr_host = E.permute_vector(x, e.plan)
    dt_t = dm.torch_dtype
    with torch.cuda.stream(stream):
        xr = torch.from_numpy(xr_host).to(f"cuda:{dev}", dt_t)
        y = torch.empty_like(xr)
    stream.synchronize()

    mode = dict(fma=args.fma, exact=args.exact)
    mode_name = "fma" if args.fma else ("strict" if args.exact else "default")
    tol = 1e-12 if e.params.tau == 8 else 1e-5
    n_long = dm.info()["long_rows"]
    # correctness gate: the exact mode bitwise against the reference's own y
    # (golden digest); the default mode is that same y unless the matrix has
    # long rows (segmented sums: within the north-star tolerance of it)
    dm.spmv(xr, y, exact=True, stream=stream)
    stream.synchronize()
    y_exact = y.cpu().numpy()
    dm.spmv(xr, y, **mode, stream=stream)
    stream.synchronize()
    parity = "unchecked"
    if gold is not None:
        ok = digest(y_exact) == gold["y_reordered"]
        if not ok:
            log("WARNING: GPU y differs from the reference digest")
            parity = "MISMATCH"
        elif mode_name == "strict" or (mode_name == "default" and n_long == 0):
            parity = "bitwise == reference y (sha256)"
            if y.cpu().numpy().tobytes() != y_exact.tobytes():
                parity = "MISMATCH (default mode differs from exact without long rows)"
        else:
            ym = y.cpu().numpy().astype(np.float64)
            err = float(np.max(np.abs(ym - y_exact))) / max(float(np.max(np.abs(y_exact))), 1e-300)
            parity = (f"rel. error {err:.1e} <= {tol:g} vs the reference y ({mode_name} mode; "
                      f"exact mode bitwise == reference y (sha256))" if err <= tol
                      else f"FAIL: rel. error {err:.1e} vs the reference y")

    # ---- device-resident timed region (value)
    for _ in range(args.warmup):
        dm.spmv(xr, y, **mode, stream=stream)
    stream.synchronize()
    ev0 = torch.cuda.Event(enable_timing=True)
    ev1 = torch.cuda.Event(enable_timing=True)
    # a step's matrix stream smaller than ~2x L2 would stay cache resident
    # between back-to-back launches: flush L2 (write 512 MB) between steps and
    # time each step on its own events
    flush_l2 = needs_l2_flush(e)
    t_resident = None
    with ClockSampler(dev) as clocks:
        torch.cuda.synchronize()
        # sustained load window (untimed) so the 20 ms nvidia-smi samples see
        # the kernel running: the timed region alone can be a few ms
        t_load = time.perf_counter()
        n_load = 0
        while time.perf_counter() - t_load < 1.5:
            for _ in range(64):
                dm.spmv(xr, y, **mode, stream=stream)
            n_load += 64
            stream.synchronize()
        if flush_l2:
            scratch = L2Flush(dev)
            evs = [(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True))
                   for _ in range(args.steps)]
            for a, b in evs:
                scratch(stream)
                a.record(stream)
                dm.spmv(xr, y, **mode, stream=stream)
                b.record(stream)
            stream.synchronize()
            t_step = sum(a.elapsed_time(b) for a, b in evs) / 1e3 / args.steps
            ev0.record(stream)
            for _ in range(args.steps):
                dm.spmv(xr, y, **mode, stream=stream)
            ev1.record(stream)
            ev1.synchronize()
            t_resident = ev0.elapsed_time(ev1) / 1e3 / args.steps
            del scratch
        else:
            ev0.record(stream)
            for _ in range(args.steps):
                dm.spmv(xr, y, **mode, stream=stream)
            ev1.record(stream)
            ev1.synchronize()
            t_step = ev0.elapsed_time(ev1) / 1e3 / args.steps
        torch.cuda.synchronize()
    value = flops / t_step / 1e9
    achieved = bmin / t_step / 1e9
    peak, peak_src = measured_peak()

    # SURVEY.md 8d protocol: a CUDA graph of R=100 SpMVs (launch overhead
    # removed), median of 5 replays; L2-resident for matrices below 2x L2
    graph = None
    y_main_bytes = y.cpu().numpy().tobytes()
    try:
        R = 100
        g = torch.cuda.CUDAGraph()
        with torch.cuda.stream(stream):
            for _ in range(3):
                dm.spmv(xr, y, **mode, stream=stream)
            stream.synchronize()
            with torch.cuda.graph(g, stream=stream):
                for _ in range(R):
                    dm.spmv(xr, y, **mode, stream=stream)
        times = []
        for _ in range(6):
            a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            with torch.cuda.stream(stream):  # replay runs on the current stream
                a.record(stream)
                g.replay()
                b.record(stream)
            b.synchronize()
            times.append(a.elapsed_time(b) / 1e3 / R)
        t_graph = statistics.median(times[1:])
        graph = {"us_per_spmv": t_graph * 1e6, "gflops": flops / t_graph / 1e9,
                 "spmv_per_graph": R, "replays": 5,
                 "bitwise_after_replay": (y.cpu().numpy().tobytes() == y_main_bytes)}
        del g
    except Exception as ex:  # graph capture unsupported here: report why
        graph = {"error": str(ex)[:200]}

    # the other arithmetic modes on the same protocol (include/ehyb_b200.h):
    # strict (every row bitwise), default (long rows in segments), fma
    y_main = y.clone()
    other_modes = []
    scratch = L2Flush(dev) if flush_l2 else None
    for name, kw in (("strict", dict(exact=True)), ("default", {}), ("fma", dict(fma=True))):
        if name == mode_name:
            continue
        evs = [(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True))
               for _ in range(min(args.steps, 200))]
        for _ in range(3):
            dm.spmv(xr, y, **kw, stream=stream)
        for a, b in evs:
            if scratch is not None:
                scratch(stream)
            a.record(stream)
            dm.spmv(xr, y, **kw, stream=stream)
            b.record(stream)
        stream.synchronize()
        t_other = sum(a.elapsed_time(b) for a, b in evs) / 1e3 / len(evs)
        yo = y.cpu().numpy().astype(np.float64)
        other_modes.append({"mode": name, "avg_us": t_other * 1e6,
                            "gflops": flops / t_other / 1e9, "effective_gbs": bmin / t_other / 1e9,
                            "rel_err_vs_reference_y": float(np.max(np.abs(yo - y_exact)))
                            / (float(np.max(np.abs(y_exact))) or 1.0)})
    del scratch
    y.copy_(y_main)

    # ---- cuSPARSE CSR comparator, same protocol
    cus = {}
    if not args.no_cusparse:
        csr = E.coo_to_csr(m)
        from paper_2204_06666_b200.device import DeviceCsr

        dcsr = DeviceCsr(csr.n_rows, csr.n_cols, csr.row_ptr, csr.col_idx, csr.values,
                         tau=e.params.tau, device=dev)
        xu = torch.from_numpy(x).to(f"cuda:{dev}", dt_t)
        yu = torch.empty_like(xu)
        flusher = L2Flush(dev) if flush_l2 else None
        for alg in (1, 2):
            for _ in range(max(3, args.warmup)):
                dcsr.spmv(xu, yu, alg, stream)
            stream.synchronize()
            k = max(10, min(args.steps, 200))
            ev0.record(stream)
            for _ in range(k):
                dcsr.spmv(xu, yu, alg, stream)
            ev1.record(stream)
            ev1.synchronize()
            t = ev0.elapsed_time(ev1) / 1e3 / k
            if flusher is not None:  # same protocol as the EHYB value: flushed steps
                cus[f"csr_alg{alg}_l2_resident_ms"] = t * 1e3
                evs = [(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True))
                       for _ in range(k)]
                for a, b in evs:
                    flusher(stream)
                    a.record(stream)
                    dcsr.spmv(xu, yu, alg, stream)
                    b.record(stream)
                stream.synchronize()
                t = sum(a.elapsed_time(b) for a, b in evs) / 1e3 / k
            cus[f"csr_alg{alg}_gflops"] = flops / t / 1e9
            cus[f"csr_alg{alg}_ms"] = t * 1e3
        cus["ehyb_speedup_vs_best"] = value / max(cus["csr_alg1_gflops"], cus["csr_alg2_gflops"])
        del dcsr, xu, yu, csr

    # ---- end-to-end through the public API with pinned host buffers: every
    # step copies its own x in (H2D), multiplies, and copies its y out (D2H)
    n_buf = 4
    xs_pin = [torch.from_numpy(W.deterministic_vector(e.dimension, s).astype(dm.dtype))
              .pin_memory() for s in range(n_buf)]
    ys_pin = [torch.empty(e.dimension, dtype=dt_t).pin_memory() for _ in range(n_buf)]
    xs_np = [t.numpy() for t in xs_pin]
    ys_np = [t.numpy() for t in ys_pin]
    k_e2e = max(8, min(args.steps, 200))
    for _ in range(max(3, min(args.warmup, 10))):
        dm.spmv_host(xs_np[0], user_order=True, **mode, out=ys_np[0])
    # (a) one synchronous call per vector (spmv_ehyb_user's host path)
    t0 = time.perf_counter()
    for i in range(k_e2e):
        dm.spmv_host(xs_np[i % n_buf], user_order=True, **mode, out=ys_np[i % n_buf])
    t_sync = (time.perf_counter() - t0) / k_e2e
    # (b) the same K products through spmv_host_many: copy-in of step i+1 and
    # copy-out of step i-1 overlap step i
    seq_x = [xs_np[i % n_buf] for i in range(k_e2e)]
    seq_y = [ys_np[i % n_buf] for i in range(k_e2e)]
    dm.spmv_host_many(seq_x[:4], user_order=True, **mode, out=seq_y[:4])
    t0 = time.perf_counter()
    dm.spmv_host_many(seq_x, user_order=True, **mode, out=seq_y)
    t_e2e = (time.perf_counter() - t0) / k_e2e
    # every host output equals the device-resident product of its input
    e2e_ok = True
    for j in range(n_buf):
        yd = dm.spmv_user(xs_pin[j].to(f"cuda:{dev}"), **mode).cpu().numpy()
        e2e_ok &= yd.tobytes() == ys_np[j].tobytes()
    if not e2e_ok:
        log("WARNING: spmv_host_many output differs from the device product")
    tb = e.params.tau

    # ---- CPU baseline: C restatement of the reference engine, host cores
    cpu = None
    if not args.no_cpu_baseline:
        threads = len(os.sched_getaffinity(0))
        prep, parts, er, yc, cflops, desc = cpu_engine_sample(e, xr_host, 2.0, threads)
        reps = []
        t_end = time.perf_counter() + args.cpu_seconds
        while time.perf_counter() < t_end or len(reps) < 3:
            t0 = time.perf_counter()
            prep.spmv(xr_host, threads, out=yc, parts=parts, er_slices=er)
            reps.append(time.perf_counter() - t0)
        tc = statistics.median(reps)
        cpu = {"value": cflops / tc / 1e9, "unit": UNIT, "cores": threads, "kind": "port",
               "sample": f"{desc}, median of {len(reps)} reps (oracle/ehyb_oracle.c, "
                         f"C restatement of engine.py spmv_ehyb, OpenMP)"}
        if desc == "full product" and parity == "unchecked":
            # no golden record for this config (the reference is too slow to
            # run at its size): check against the pinned C restatement instead
            # (exact mode bitwise; the run's own mode within the tolerance)
            ok = yc.tobytes() == y_exact.tobytes()
            ym = y_main.cpu().numpy().astype(np.float64)
            yr = yc.astype(np.float64)
            err = float(np.max(np.abs(ym - yr))) / max(float(np.max(np.abs(yr))), 1e-300)
            if not ok:
                parity = "MISMATCH: exact mode vs C restatement"
            elif ym.tobytes() == yr.tobytes():
                parity = ("bitwise == C restatement of the reference engine (pinned on the "
                          "golden configs)")
            else:
                parity = (f"rel. error {err:.1e} <= {tol:g} vs the C restatement of the reference "
                          f"engine ({mode_name} mode; exact mode bitwise)" if err <= tol
                          else f"FAIL: rel. error {err:.1e}")

    traffic = None
    prof_path = os.path.join(ROOT, "profiles", "ncu_traffic.json")
    if os.path.exists(prof_path):
        with open(prof_path) as fh:
            traffic = json.load(fh).get(args.config, {}).get("dram_bytes_per_launch")

    out = {
        "metric": METRIC, "value": value, "unit": UNIT, "n_gpus": 1, "steps": args.steps,
        "warmup": args.warmup, "ms_per_step": t_step * 1e3, "higher_is_better": True,
        "scaling": "weak", "vs_baseline": None, "dtype": "f64" if tb == 8 else "f32",
        "data": "synthetic", "config": config_block(args, m, e),
        "roofline": {"bound": "hbm", "achieved": achieved, "peak": peak, "unit": "GB/s",
                     "frac": achieved / peak, "traffic": traffic,
                     "peak_source": peak_src,
                     "peak_spec": SPEC_HBM_GBS, "frac_spec": achieved / SPEC_HBM_GBS,
                     "algorithmic_bytes_per_launch": bmin,
                     "model": "nnz_ell*(tau+2) + nnz_er*(tau+4) + 2*n*tau (SURVEY.md 8d)"},
        "cpu_baseline": cpu,
        "e2e": {"value": flops / t_e2e / 1e9, "unit": UNIT,
                "h2d_bytes_per_step": int(e.dimension * tb),
                "d2h_bytes_per_step": int(e.dimension * tb),
                "ms_per_step": t_e2e * 1e3, "steps": k_e2e,
                "api": "DeviceMatrix.spmv_host_many(xs, user_order=True): per step pinned "
                       "H2D of x_i, permute, fused SpMV, unpermute, D2H of y_i; copies of "
                       "neighbouring steps overlap the product (PCIe full duplex)",
                "parity": "bitwise == device product" if e2e_ok else "MISMATCH",
                "sync_call": {"value": flops / t_sync / 1e9, "ms_per_step": t_sync * 1e3,
                              "api": "DeviceMatrix.spmv_host(x, user_order=True) per step "
                                     "(spmv_ehyb_user host path), synchronous"}},
        "e2e_single_call": {"value": flops / t_sync / 1e9, "unit": UNIT,
                            "ms_per_step": t_sync * 1e3,
                            "h2d_bytes_per_step": int(e.dimension * tb),
                            "d2h_bytes_per_step": int(e.dimension * tb),
                            "api": "spmv_ehyb_user host path (DeviceMatrix.spmv_host), one "
                                   "synchronous call per vector"},
        "gpu_launches": args.steps,
        "clocks": dict(clocks.summary(), window=f"{n_load} untimed load steps (>= 1.5 s) "
                                                f"then the timed steps"),
        "parity": parity,
        "cusparse": cus,
        "kernel": {"avg_us": t_step * 1e6, "effective_gbs": achieved,
                   "mode": mode_name, "long_rows": n_long, "other_modes": other_modes,
                   "cuda_graph": graph,
                   "l2_resident_avg_us": None if t_resident is None else t_resident * 1e6,
                   "traffic_model_bytes": E.traffic_model(e), "device_info": info},
        "preprocessing": dict(prep_t, prep_to_spmv_ratio=(prep_t["partition_s"]
                                                          + prep_t["reorder_assemble_s"]) / t_step),
    }
    print(json.dumps(out), flush=True)
    return 0


def main(argv=None):
    ap = argparse.ArgumentParser(description=__doc__)
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=2000)
    ap.add_argument("--warmup", type=int, default=20)
    ap.add_argument("--impl", choices=("ours", "reference"), default="ours")
    ap.add_argument("--config", default=None,
                    help="workload (default: cfg2 at N=1, cfg5 at N>1; 'weak' = weak scaling)")
    ap.add_argument("--no-ref-python", action="store_true",
                    help="reference arm: skip the one timed call of the unmodified reference "
                         "engine from baseline/_ref (~6 s per cfg2 SpMV; skipped above 6M rows)")
    ap.add_argument("--fma", action="store_true", help="fused multiply-add mode")
    ap.add_argument("--exact", action="store_true",
                    help="strict mode: every row bitwise (default: long rows in segments)")
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--no-cusparse", action="store_true")
    ap.add_argument("--cpu-seconds", type=float, default=10.0)
    ap.add_argument("--dist", action="store_true",
                    help="run the row-sharded (NCCL) path even on one GPU")
    args = ap.parse_args(argv)
    if args.warmup < 3:
        log("warmup raised to 3 (timing rule)")
        args.warmup = 3
    sys.path.insert(0, os.path.join(ROOT, "tests", "golden"))
    world = int(os.environ.get("WORLD_SIZE", "1"))
    if args.config is None and max(world, args.gpus) <= 1 and not args.dist:
        args.config = "cfg2"
    if args.impl == "reference":
        return run_reference(args)
    return run_gpu(args)


if __name__ == "__main__":
    sys.exit(main())
