"""GPU preprocessing (gpu_prep.py, csrc/prep_gpu.cu) against the host path,
which is pinned to the reference: build_graph's adjacency and every array of
classify_rows / build_reorder_plan / assemble_ehyb byte for byte, on the
golden small cases, reference-corpus structures, heavy-tailed hubs, duplicate
coordinates, fp32 and fp64, slice heights 1/4/8/32, and external partitions
(the rebalance path)."""

import numpy as np
import pytest

import paper_2204_06666_b200 as E
from paper_2204_06666_b200 import workloads as W
from golden_data import small_case, small_meta

pytestmark = pytest.mark.gpu
torch = pytest.importorskip("torch")

ARRAYS = ("val_ell", "col_ell", "position_ell", "width_ell", "part_boundary", "ell_row_widths",
          "val_er", "col_er", "position_er", "width_er", "er_row_widths")
PLAN = ("reorder_table", "inverse_table", "arrange_table", "y_idx_er")


def same(a, b):
    a, b = np.asarray(a), np.asarray(b)
    return a.dtype == b.dtype and a.shape == b.shape and a.tobytes() == b.tobytes()


def check_matrix(m, tau, profile, partition=None):
    try:
        host = E.build_ehyb(m, tau=tau, profile=profile, partition=partition)
    except ValueError as ex:  # the host path rejects it: the GPU path must too
        with pytest.raises(ValueError):
            E.build_ehyb_gpu(m, tau=tau, profile=profile, partition=partition, device=0)
        return str(ex)
    t = {}
    gpu = E.build_ehyb_gpu(m, tau=tau, profile=profile, partition=partition, device=0, timings=t)
    for k in ARRAYS:
        assert same(getattr(gpu, k), getattr(host, k)), k
    for k in PLAN:
        assert same(getattr(gpu.plan, k), getattr(host.plan, k)), k
    assert gpu.plan.n_er_rows == host.plan.n_er_rows
    assert set(t) == {"upload_s", "build_graph_s", "partition_graph_s", "reorder_assemble_s"}
    return host


def test_build_graph_matches_host():
    from paper_2204_06666_b200.gpu_prep import GpuPrep

    for n, r, c, v in (W.permute_symmetric(*W.stencil27(12, 12, 12), seed=3),
                       W.heavy_tail(k=10, n_hubs=3, min_len=50, max_len=400)):
        m = E.CooMatrix(n, n, r, c, v)
        g = E.build_graph(m)
        gp = GpuPrep(m, 0)
        gg = gp.build_graph()
        gp.close()
        assert same(gg.adj_ptr, g.adj_ptr) and same(gg.adj, g.adj)


@pytest.mark.parametrize("name", sorted(small_meta()))
def test_small_golden_cases(name):
    meta = small_meta()[name]
    g = small_case(name)
    m = E.CooMatrix(meta["n"], meta["n"], g["rows"], g["cols"], g["vals"])
    prof = E.DeviceProfile(*meta["profile"])
    part = None
    if g.get("assignment_in") is not None:
        part = E.PartitionMap.from_assignment(g["assignment_in"], n_parts=meta["n_parts_hint"])
    check_matrix(m, meta["tau"], prof, part)


@pytest.mark.parametrize("tau", [4, 8])
@pytest.mark.parametrize("kind", ["stencil", "rgg", "heavy", "dups"])
def test_structures(kind, tau):
    rng = np.random.default_rng(7)
    if kind == "stencil":
        n, r, c, v = W.permute_symmetric(*W.stencil27(20, 20, 20), seed=1)
        prof = E.DeviceProfile(16, 32, 8192)
    elif kind == "rgg":
        n, r, c, v = W.rgg3d(30_000)
        prof = E.DeviceProfile(24, 8, 4096)
    elif kind == "heavy":
        n, r, c, v = W.heavy_tail(k=16, n_hubs=4, min_len=200, max_len=3000)
        prof = E.DeviceProfile(12, 4, 8192)
    else:  # duplicate coordinates: entry order decides the rank within the row
        n = 3000
        r = rng.integers(0, n, 40_000)
        c = rng.integers(0, n, 40_000)
        v = rng.standard_normal(40_000)
        r = np.concatenate([r, r[:5000]])
        c = np.concatenate([c, c[:5000]])
        v = np.concatenate([v, -v[:5000] * 0.5])
        prof = E.DeviceProfile(6, 1, 4096)
    check_matrix(E.CooMatrix(n, n, r, c, v), tau, prof)


def test_external_partition_rebalanced():
    n, r, c, v = W.permute_symmetric(*W.stencil27(16, 16, 16), seed=2)
    m = E.CooMatrix(n, n, r, c, v)
    part = E.PartitionMap.from_assignment(np.arange(n) % 3, n_parts=3)
    check_matrix(m, 8, E.DeviceProfile(8, 32, 8192), part)


def test_config_scale_cfg2_digests():
    # the bench workload: every parity array equal to the reference's digests
    import json
    import os

    from golden_util import digest

    path = os.path.join(os.path.dirname(__file__), "golden", "config_cfg2.json")
    rec = json.load(open(path))
    n, r, c, v, tau = W.build_config("cfg2")
    e = E.build_ehyb_gpu(E.CooMatrix(n, n, r, c, v), tau=tau, profile=E.B200_PROFILE, device=0)
    for k, want in rec["digests"].items():
        obj = e.plan if hasattr(e.plan, k) and not hasattr(e, k) else e
        if hasattr(obj, k):
            assert digest(getattr(obj, k)) == want, k
