#!/usr/bin/env python3
"""Generate the golden fixtures by running the REAL reference package.

The reference (`ehyb` 0.1.0, /root/reference/pkg, pure Python + numpy) is
imported from a temporary copy; its outputs are the ground truth that pins
both the oracle (oracle/) and the product (paper_2204_06666_b200/). This script
only runs where /root/reference exists (the dev container); the fixtures it
writes are committed and travel to the GPU box.

    python tests/golden/make_golden.py small            -> small_cases.npz / small_cases.json
    python tests/golden/make_golden.py corpus           -> corpus_digests.json
    python tests/golden/make_golden.py container        -> container_digests.json
    python tests/golden/make_golden.py config cfg1 ...  -> config_<name>.json

Fixtures hold full arrays for small cases and golden digests (golden_util.digest:
sha256 of dtype|shape|bytes) for the corpus and the BASELINE configs.
"""

from __future__ import annotations

import json
import os
import shutil
import sys
import tempfile
import time

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(os.path.dirname(HERE))
sys.path.insert(0, ROOT)
sys.path.insert(0, HERE)

from golden_util import collect, digest, digests  # noqa: E402
from paper_2204_06666_b200 import workloads as W  # noqa: E402

REFERENCE = "/root/reference/pkg/src"

# B200 profile used for every BASELINE config: 148 SMs, 32-lane slices,
# 227 KB opt-in shared memory minus 1 KB kept for the kernel's own words.
B200_PROFILE_ARGS = (148, 32, 232448 - 1024)


def load_reference():
    tmp = tempfile.mkdtemp(prefix="ehyb_ref_")
    shutil.copytree(REFERENCE, os.path.join(tmp, "src"))
    sys.path.insert(0, os.path.join(tmp, "src"))
    import ehyb  # noqa: F401
    import ehyb.cli  # noqa: F401

    return sys.modules["ehyb"]


def run_pipeline(ehyb, n, rows, cols, vals, tau, profile_args, assignment=None,
                 n_parts_hint=None, seed=0, rebalance=False, timings=None):
    """The reference pipeline step by step (helpers.pipeline, tests/helpers.py:117-125;
    with rebalance=True, build_ehyb's external-partition branch format.py:425-439)."""
    m = ehyb.CooMatrix(n, n, rows, cols, vals)
    profile = ehyb.DeviceProfile(*profile_args)
    params = ehyb.compute_params(n, tau, profile)
    t0 = time.perf_counter()
    g = ehyb.build_graph(m)
    t1 = time.perf_counter()
    if assignment is None:
        parts = ehyb.partition_graph(g, params.n_parts, params.vec_cache_size, seed=seed)
    elif rebalance:
        parts = ehyb.PartitionMap.from_assignment(assignment, n_parts=n_parts_hint)
        if parts.n_parts < params.n_parts:
            parts = ehyb.PartitionMap.from_assignment(parts.assignment, n_parts=params.n_parts)
        if int(parts.part_sizes.max(initial=0)) > params.vec_cache_size:
            parts = ehyb.rebalance_partition(g, parts, params.vec_cache_size)
    else:
        parts = ehyb.PartitionMap.from_assignment(assignment, n_parts=n_parts_hint)
    t2 = time.perf_counter()
    cls = ehyb.classify_rows(m, parts)
    plan = ehyb.build_reorder_plan(cls, params, parts)
    e = ehyb.assemble_ehyb(m, plan, params, parts)
    t3 = time.perf_counter()
    if timings is not None:
        timings.update(build_graph_s=t1 - t0, partition_s=t2 - t1, reorder_assemble_s=t3 - t2)
    return m, params, g, parts, cls, plan, e


def small_case_specs():
    tiny = (2, 4, 64)
    yield "tridiag8_kat", W.tridiagonal(8), 8, tiny, np.array([0] * 4 + [1] * 4), 2, False
    yield "identity16", (16, np.arange(16), np.arange(16), np.ones(16)), 8, tiny, None, None, False
    nb = 8
    r = np.repeat(np.arange(nb), 4)
    blocks = np.concatenate([np.repeat(np.arange(4) + 4 * b, 4) for b in range(2)])
    bcols = np.concatenate([np.tile(np.arange(4) + 4 * b, 4) for b in range(2)])
    del r
    yield "blockdiag2x4", (8, blocks, bcols, 1.0 + 0.01 * np.arange(32)), 8, tiny, None, None, False
    yield "empty5", (5, np.zeros(0, np.int64), np.zeros(0, np.int64), np.zeros(0)), 8, tiny, None, None, False
    yield "desc_sort_w1", (3, np.array([0, 1, 1, 1, 2, 2]), np.array([0, 0, 1, 2, 1, 2]),
                           np.ones(6)), 8, (1, 1, 64), np.zeros(3, np.int64), 1, False
    for s in range(6):
        rng = np.random.default_rng(s)
        tau = 4 if s % 3 == 2 else 8
        procs = [1, 2, 4][s % 3]
        yield (f"random64_s{s}", W.random_coo(64, float(rng.uniform(0.02, 0.15)), seed=s), tau,
               (procs, 8, 512 if tau == 8 else 256), None, None, False)
    yield "random128_f32", W.random_coo(128, 0.08, seed=42), 4, (2, 8, 2048), None, None, False
    yield "poisson32", W.laplacian_2d(32, 32), 8, (4, 32, 2048), None, None, False
    yield "default80_64x64", W.laplacian_2d(64, 64), 8, (80, 32, 48 * 1024), None, None, False
    n = 64
    pr, pc, pv = [], [], []
    for i in range(n):
        pr += [i, i]
        pc += [i, (i + n // 2) % n]
        pv += [2.0, 1.0]
    yield ("phase_barrier", (n, np.array(pr), np.array(pc), np.array(pv, float)), 8, (4, 4, 128),
           np.arange(n) // 16, 4, False)
    yield ("rebalance_tridiag16", W.tridiagonal(16), 8, (2, 8, 64), np.zeros(16, np.int64), 1, True)
    yield ("rebalance_random40", W.random_coo(40, 0.1, seed=6), 8, (4, 8, 80),
           np.zeros(40, np.int64), 4, True)
    yield "chain4096", W.tridiagonal(4096), 8, (4, 32, 48 * 1024), None, None, False
    yield "grid3d16", W.laplacian_3d7(16, 16, 16), 8, (4, 32, 48 * 1024), None, None, False
    yield "grid3d16_w4_f32", W.laplacian_3d7(16, 16, 16), 4, (16, 4, 1024), None, None, False
    yield "heavy_small", W.heavy_tail(k=16, n_hubs=4, min_len=100, max_len=2000), 8, (8, 32, 8192), None, None, False
    yield "stencil27_12", W.permute_symmetric(*W.stencil27(12, 12, 12), seed=1), 8, (6, 32, 4096), None, None, False


def cmd_small(ehyb):
    arrays = {}
    meta = {}
    for name, (n, r, c, v), tau, prof, assign, nph, reb in small_case_specs():
        m, params, g, parts, cls, plan, e = run_pipeline(
            ehyb, n, r, c, v, tau, prof, assignment=assign, n_parts_hint=nph, rebalance=reb)
        got = collect(parts, cls, plan, e, graph=g)
        x = W.deterministic_vector(n, 0)
        xr = ehyb.permute_vector(x, plan)
        y, st = ehyb.spmv_ehyb(e, xr)
        yu = ehyb.spmv_ehyb_user(e, x)
        ycsr = ehyb.spmv_csr(ehyb.coo_to_csr(m), x)
        got.update(rows=m.rows, cols=m.cols, vals=m.values, x=x, y_reordered=y, y_user=yu,
                   y_csr=ycsr)
        if assign is not None:
            got["assignment_in"] = np.asarray(assign, np.int64)
        for k, a in got.items():
            arrays[f"{name}/{k}"] = np.asarray(a)
        if reb:
            eb = ehyb.build_ehyb(m, tau=tau, profile=ehyb.DeviceProfile(*prof),
                                 partition=ehyb.PartitionMap.from_assignment(assign, n_parts=nph))
            assert digest(eb.val_ell) == digest(e.val_ell)
            assert digest(eb.plan.reorder_table) == digest(plan.reorder_table)
        meta[name] = dict(
            n=n, tau=tau, profile=list(prof), external=assign is not None, rebalance=reb,
            n_parts_hint=nph, k=params.k, n_parts=params.n_parts, vec=params.vec_cache_size,
            n_er=plan.n_er_rows, nnz_ell=e.nnz_ell, nnz_er=e.nnz_er,
            cached_loads=st.cached_loads, uncached_loads=st.uncached_loads, flops=st.flops,
            bytes_touched_model=st.bytes_touched_model,
            traffic_model=ehyb.traffic_model(e),
            footprint=ehyb.footprint_stats(e).__dict__,
        )
    np.savez_compressed(os.path.join(HERE, "small_cases.npz"), **arrays)
    with open(os.path.join(HERE, "small_cases.json"), "w") as fh:
        json.dump(meta, fh, indent=1, sort_keys=True)
    print(f"small: {len(meta)} cases, {len(arrays)} arrays")


def cmd_corpus(ehyb):
    out = []
    t0 = time.perf_counter()
    for i, d in enumerate(W.corpus_specs()):
        m, params, g, parts, cls, plan, e = run_pipeline(
            ehyb, d["n"], d["rows"], d["cols"], d["vals"], d["tau"], d["profile"],
            assignment=d["assignment"], n_parts_hint=d["n_parts_hint"], seed=d["seed"])
        x = W.deterministic_vector(d["n"], i)
        xr = ehyb.permute_vector(x, plan)
        y, _ = ehyb.spmv_ehyb(e, xr)
        rec = dict(name=d["name"], n_parts=params.n_parts, vec=params.vec_cache_size,
                   nnz_ell=e.nnz_ell, nnz_er=e.nnz_er, traffic_model=ehyb.traffic_model(e),
                   digests=digests(collect(parts, cls, plan, e, graph=g)),
                   y_reordered=digest(y))
        out.append(rec)
    with open(os.path.join(HERE, "corpus_digests.json"), "w") as fh:
        json.dump(out, fh, indent=0)
    print(f"corpus: {len(out)} cases in {time.perf_counter() - t0:.1f}s")


def cmd_config(ehyb, names):
    for name in names:
        t0 = time.perf_counter()
        n, r, c, v, tau = W.build_config(name)
        tgen = time.perf_counter() - t0
        tm = {}
        prof = tuple(W.CONFIG_PROFILES.get(name, B200_PROFILE_ARGS))
        m, params, g, parts, cls, plan, e = run_pipeline(
            ehyb, n, r, c, v, tau, prof, timings=tm)
        arr = collect(parts, cls, plan, e, graph=g)
        x = W.deterministic_vector(n, 0)
        xr = ehyb.permute_vector(x, plan)
        t1 = time.perf_counter()
        y, st = ehyb.spmv_ehyb(e, xr)
        tm["spmv_ehyb_s"] = time.perf_counter() - t1
        yu = ehyb.spmv_ehyb_user(e, x)
        csr = ehyb.coo_to_csr(m)
        t1 = time.perf_counter()
        ycsr = ehyb.spmv_csr(csr, x)
        tm["spmv_csr_s"] = time.perf_counter() - t1
        cm = ehyb.cut_metrics(m, parts)
        fp = ehyb.footprint_stats(e)
        den = float(np.max(np.abs(ycsr))) if ycsr.size else 1.0
        rec = dict(
            name=name, description=W.CONFIGS[name][0], n=n, nnz=m.nnz, tau=tau,
            profile=list(prof), k=params.k, n_parts=params.n_parts,
            vec=params.vec_cache_size, padded=e.padded_dimension, n_er=plan.n_er_rows,
            nnz_ell=e.nnz_ell, nnz_er=e.nnz_er, slots_ell=int(e.val_ell.size),
            slots_er=int(e.val_er.size), inner_fraction=cm.inner_fraction,
            traffic_model=ehyb.traffic_model(e), footprint_total=fp.total_bytes,
            bytes_touched_model=st.bytes_touched_model,
            digests=digests(arr),
            y_reordered=digest(y), y_user=digest(yu),
            y_user_sum=float(np.sum(yu, dtype=np.float64)), y_user_head=[float(a) for a in yu[:8]],
            rel_err_vs_csr=float(np.max(np.abs(yu.astype(np.float64) - ycsr)) / den),
            timings=dict(generate_s=tgen, **tm), host=dict(cpus=os.cpu_count()),
        )
        with open(os.path.join(HERE, f"config_{name}.json"), "w") as fh:
            json.dump(rec, fh, indent=1, sort_keys=True)
        print(f"config {name}: n={n} nnz={m.nnz} parts={params.n_parts} vec={params.vec_cache_size} "
              f"inner={cm.inner_fraction:.4f} total {time.perf_counter() - t0:.1f}s {tm}", flush=True)
        del m, g, parts, cls, plan, e, arr, r, c, v, y, yu, csr, ycsr


def cmd_container(ehyb):
    """Digests of the reference's .ehyb container bytes (matrix_io.py:337-377)
    for every small case."""
    import hashlib
    import io

    out = {}
    for name, (n, r, c, v), tau, prof, assign, nph, reb in small_case_specs():
        *_, e = run_pipeline(ehyb, n, r, c, v, tau, prof, assignment=assign,
                             n_parts_hint=nph, rebalance=reb)
        buf = io.BytesIO()
        ehyb.write_ehyb_container(e, buf)
        out[name] = hashlib.sha256(buf.getvalue()).hexdigest()
    with open(os.path.join(HERE, "container_digests.json"), "w") as fh:
        json.dump(out, fh, indent=1, sort_keys=True)
    print(f"container: {len(out)} digests")


def main(argv):
    ehyb = load_reference()
    if argv[0] == "small":
        cmd_small(ehyb)
    elif argv[0] == "corpus":
        cmd_corpus(ehyb)
    elif argv[0] == "container":
        cmd_container(ehyb)
    elif argv[0] == "config":
        cmd_config(ehyb, argv[1:])
    else:
        raise SystemExit(__doc__)


if __name__ == "__main__":
    main(sys.argv[1:])
