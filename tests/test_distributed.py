"""Multi-GPU layer (distributed.py): halo plans, the halo exchange over a real
torch.distributed process group (gloo, world_size 2 and 3 on CPU), shard
products on one GPU, and CG."""

import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

import paper_2204_06666_b200 as E
from oracle import c_oracle
from paper_2204_06666_b200 import distributed as D
from paper_2204_06666_b200 import workloads as W


def matrix(tau=8):
    n, r, c, v = W.permute_symmetric(*W.stencil27(14, 14, 14), seed=1)
    m = E.CooMatrix(n, n, r, c, v)
    return m, E.build_ehyb(m, tau=tau, profile=E.DeviceProfile(12, 32, 8192))


def shard_product_host(e, plan, x_ext):
    """Test-side float64 product of the owned rows from x_ext through the
    plan's column remap (owned -> c - lo, remote -> local_rows + halo slot)."""
    vec, warp = e.params.vec_cache_size, e.params.warp_size
    lo, hi = plan.p0 * vec, plan.p1 * vec
    coo_r, coo_c, coo_v = [], [], []
    w = e.ell_row_widths.astype(np.int64)
    rows = np.repeat(np.arange(e.padded_dimension), w)
    k = np.arange(rows.size) - np.repeat(np.cumsum(w) - w, w)
    idx = e.position_ell[rows // warp] + rows % warp + k * warp
    coo_r.append(rows)
    coo_c.append(e.col_ell[idx].astype(np.int64) + (rows // vec) * vec)
    coo_v.append(e.val_ell[idx])
    w2 = e.er_row_widths.astype(np.int64)
    slots = np.repeat(np.arange(e.plan.n_er_rows), w2)
    k2 = np.arange(slots.size) - np.repeat(np.cumsum(w2) - w2, w2)
    idx2 = e.position_er[slots // warp] + slots % warp + k2 * warp
    coo_r.append(e.plan.y_idx_er[slots])
    coo_c.append(e.col_er[idx2].astype(np.int64))
    coo_v.append(e.val_er[idx2])
    r = np.concatenate(coo_r)
    c = np.concatenate(coo_c)
    v = np.concatenate(coo_v).astype(np.float64)
    keep = (r >= lo) & (r < hi)
    r, c, v = r[keep] - lo, c[keep], v[keep]
    own = (c >= lo) & (c < hi)
    ext = np.where(own, c - lo, plan.local_rows + np.searchsorted(plan.halo_cols, c))
    assert np.all(plan.halo_cols[np.searchsorted(plan.halo_cols, c[~own])] == c[~own])
    y = np.zeros(plan.local_rows)
    np.add.at(y, r, v * x_ext[ext])
    return y


def _free_port():
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


def _worker(rank, world, port):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        m, e = matrix()
        plan = D.build_halo_plan(e)
        assert plan.world == world and plan.rank == rank
        xr = E.permute_vector(W.deterministic_vector(e.dimension, 0), e.plan)
        lo, hi = plan.p0 * plan.vec, plan.p1 * plan.vec
        x_ext = torch.zeros(plan.local_rows + plan.n_halo, dtype=torch.float64)
        x_ext[: plan.local_rows] = torch.from_numpy(xr[lo:hi])
        D.halo_exchange(x_ext, plan)
        got = x_ext.numpy()
        assert np.array_equal(got[plan.local_rows:], xr[plan.halo_cols]), "halo values"
        y_loc = shard_product_host(e, plan, got)
        y_full = c_oracle.spmv_ehyb(e, xr, 1)
        den = np.max(np.abs(y_full))
        assert np.max(np.abs(y_loc - y_full[lo:hi])) / den < 1e-12, "shard product"
        # every rank's rows together cover the padded space exactly once
        sizes = [torch.zeros(1, dtype=torch.int64) for _ in range(world)]
        dist.all_gather(sizes, torch.tensor([plan.local_rows]))
        assert sum(int(s) for s in sizes) == e.padded_dimension
    finally:
        dist.destroy_process_group()


@pytest.mark.parametrize("world", [2, 3])
def test_halo_exchange_gloo(world):
    mp.spawn(_worker, args=(world, _free_port()), nprocs=world, join=True)


def test_plans_are_consistent():
    m, e = matrix()
    for world in (2, 4):
        plans = [D.plan_for(e, r, world) for r in range(world)]
        for g, pg in enumerate(plans):
            for q, pq in enumerate(plans):
                # what q sends to g == g's halo entries owned by q
                seg = np.cumsum([0] + pq.send_splits)
                sent = pq.send_idx[seg[g]:seg[g + 1]] + pq.p0 * pq.vec
                rseg = np.cumsum([0] + pg.recv_splits)
                assert np.array_equal(sent, pg.halo_cols[rseg[q]:rseg[q + 1]])
        assert sum(p.local_rows for p in plans) == e.padded_dimension
        # plans key the device index cache (identity hash), one tensor per plan
        t = D._idx_tensor(plans[0], torch.device("cpu"))
        assert D._idx_tensor(plans[0], torch.device("cpu")) is t
        assert np.array_equal(t.numpy(), plans[0].send_idx)


def heavy_matrix(tau=8):
    n, r, c, v = W.heavy_tail(k=14, n_hubs=4, min_len=100, max_len=1500)
    m = E.CooMatrix(n, n, r, c, v)
    return m, E.build_ehyb(m, tau=tau, profile=E.DeviceProfile(12, 32, 8192))


@pytest.mark.gpu
@pytest.mark.parametrize("world", [1, 2, 3])
@pytest.mark.parametrize("tau", [4, 8])
@pytest.mark.parametrize("kind", ["stencil", "heavy"])
def test_shards_on_one_gpu_bitwise(world, tau, kind, monkeypatch):
    # local launch (ELL + ER rows with owned columns) then halo launch (ER
    # rows with a halo column, long rows), and the single fused launch:
    # both bitwise equal to the full product
    if kind == "heavy":
        monkeypatch.setenv("EHYB_LONG_ROW", "40")
        m, e = heavy_matrix(tau)
    else:
        m, e = matrix(tau)
    xr = E.permute_vector(W.deterministic_vector(e.dimension, 0), e.plan)
    y_full, _ = E.spmv_ehyb(e, xr, E.ExecutionConfig(exact=True))
    dt = torch.float32 if tau == 4 else torch.float64
    for rank in range(world):
        plan = D.plan_for(e, rank, world)
        A = D.DistributedEhyb(e, device=0, plan=plan)
        lo, hi = plan.p0 * plan.vec, plan.p1 * plan.vec
        x_ext = A.new_ext()
        x_ext[: plan.local_rows] = torch.from_numpy(xr[lo:hi]).to(dt)
        x_ext[plan.local_rows:] = torch.from_numpy(xr[plan.halo_cols]).to(dt)
        y = torch.empty(plan.local_rows, dtype=dt, device="cuda:0")
        A.spmv_local(x_ext, y, exact=True)
        torch.cuda.synchronize()
        assert y.cpu().numpy().tobytes() == y_full[lo:hi].tobytes()
        y2 = torch.empty_like(y)
        import ctypes as C
        from paper_2204_06666_b200 import _lib as L
        L.call("ehyb_dev_spmv", A._h, C.c_void_p(x_ext.data_ptr()), C.c_void_p(y2.data_ptr()),
               L.MODE_STRICT, C.c_void_p(torch.cuda.current_stream().cuda_stream))
        torch.cuda.synchronize()
        assert y2.cpu().numpy().tobytes() == y_full[lo:hi].tobytes()


@pytest.mark.gpu
@pytest.mark.parametrize("method", ["chronopoulos-gear", "classic"])
def test_cg_converges_single_gpu(method):
    m, e = matrix()
    plan = D.plan_for(e, 0, 1)
    A = D.DistributedEhyb(e, device=0, plan=plan)
    ones = A.new_ext()
    ones[: A.local_rows].fill_(1.0)
    # padding rows of b stay 0 (empty rows), so the solution there is 0
    b = torch.empty(A.local_rows, dtype=torch.float64, device="cuda:0")
    A.spmv_local(ones, b)
    x, info = D.cg(A, b, maxiter=200, tol=1e-10, method=method)
    assert info["method"] == method
    torch.cuda.synchronize()
    real = np.zeros(A.local_rows, bool)
    real[e.plan.reorder_table[: e.dimension]] = True
    xs = x.cpu().numpy()
    assert info["rel_residual"] < 1e-9
    assert np.max(np.abs(xs[real] - 1.0)) < 1e-7
    assert np.all(xs[~real] == 0.0)


def test_partition_grouping_cuts_halo_and_keeps_results():
    # renumbering partitions so each rank's contiguous block is compact in the
    # quotient graph: same products (bitwise, C oracle), smaller halos
    n, r, c, v = W.permute_symmetric(*W.stencil27(20, 20, 40), seed=1)
    m = E.CooMatrix(n, n, r, c, v)
    e = E.build_ehyb(m, tau=8, profile=E.DeviceProfile(24, 32, 8192))
    x = W.deterministic_vector(n, 0)
    y = E.unpermute_vector(c_oracle.spmv_ehyb(e, E.permute_vector(x, e.plan)), e.plan)
    for world in (2, 4, 8):
        order = D.group_partitions(e, world)
        assert sorted(order.tolist()) == list(range(e.n_parts))
        e2 = D.renumber_partitions(e, order)
        e2.check()
        y2 = E.unpermute_vector(c_oracle.spmv_ehyb(e2, E.permute_vector(x, e2.plan)), e2.plan)
        assert y2.tobytes() == y.tobytes()

        def total_halo(ee):
            return sum(D.halo_columns(ee, *D.part_range(ee.n_parts, world, g)).size
                       for g in range(world))

        assert total_halo(e2) < total_halo(e)
    with pytest.raises(ValueError, match="permutation"):
        D.renumber_partitions(e, np.zeros(e.n_parts, np.int64))


@pytest.mark.gpu
@pytest.mark.parametrize("world", [2, 3])
def test_grouped_shards_on_one_gpu_match_the_original(world):
    # the multi-GPU bench path: renumber partitions by quotient-graph groups,
    # shard the renumbered matrix, and get the original matrix's y
    m, e = matrix(8)
    e2 = D.renumber_partitions(e, D.group_partitions(e, world))
    x = W.deterministic_vector(e.dimension, 0)
    y_ref = E.spmv_ehyb_user(e, x)
    xr2 = E.permute_vector(x, e2.plan)
    y2 = np.empty(e2.padded_dimension)
    for rank in range(world):
        plan = D.plan_for(e2, rank, world)
        A = D.DistributedEhyb(e2, device=0, plan=plan)
        lo, hi = plan.p0 * plan.vec, plan.p1 * plan.vec
        x_ext = A.new_ext()
        x_ext[: plan.local_rows] = torch.from_numpy(xr2[lo:hi])
        x_ext[plan.local_rows:] = torch.from_numpy(xr2[plan.halo_cols])
        y = torch.empty(plan.local_rows, dtype=torch.float64, device="cuda:0")
        A.spmv_local(x_ext, y)
        torch.cuda.synchronize()
        y2[lo:hi] = y.cpu().numpy()
    assert E.unpermute_vector(y2, e2.plan).tobytes() == y_ref.tobytes()


def _p2p_worker(rank, world, port, q):
    # ranks share cuda:0; handles exchanged over gloo, halo pulled in-kernel
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        torch.cuda.set_device(0)
        for kind, tau in (("stencil", 8), ("heavy", 4)):
            m, e = matrix(tau) if kind == "stencil" else heavy_matrix(tau)
            A = D.DistributedEhyb(e, device=0, exchange="p2p")
            xr = E.permute_vector(W.deterministic_vector(e.dimension, 0), e.plan)
            lo, hi = A.plan.p0 * A.plan.vec, A.plan.p1 * A.plan.vec
            # zero-copy handle-owned buffer, or a user buffer copied in by spmv
            x_ext = A.ext_buffer() if kind == "stencil" else A.new_ext()
            y = torch.empty(A.local_rows, dtype=A.dtype, device="cuda:0")
            for it in range(3):  # the sequence numbers advance, x is rewritten each time
                x_ext[: A.local_rows] = torch.from_numpy(xr[lo:hi] * (it + 1)).to(A.dtype)
                A.spmv(x_ext, y, exact=True)
                torch.cuda.synchronize()
                got = y.cpu().numpy()
                ref = c_oracle.spmv_ehyb(e, (xr * (it + 1)).astype(xr.dtype))[lo:hi]
                ok = got.tobytes() == ref.tobytes()  # the sign of zero included
                q.put((rank, kind, it, ok))
            del A
        # CG on the p2p operator converges like the single-GPU one
        m, e = matrix(8)
        A = D.DistributedEhyb(e, device=0, exchange="p2p")
        ones = A.new_ext()
        ones[: A.local_rows].fill_(1.0)
        b = torch.empty(A.local_rows, dtype=torch.float64, device="cuda:0")
        A.spmv(ones, b)
        x, info = D.cg(A, b.clone(), maxiter=200, tol=1e-10)
        q.put((rank, "cg", info["iterations"], info["rel_residual"] < 1e-9))
    finally:
        dist.destroy_process_group()


@pytest.mark.gpu
@pytest.mark.parametrize("world", [2, 3])
def test_p2p_fused_exchange_multi_process_one_gpu(world):
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_p2p_worker, args=(r, world, port, q)) for r in range(world)]
    for p in procs:
        p.start()
    for p in procs:
        p.join(timeout=240)
    alive = [p for p in procs if p.is_alive()]
    for p in alive:
        p.kill()
    assert not alive, "p2p ranks did not finish"
    assert all(p.exitcode == 0 for p in procs)
    res = [q.get() for _ in range(world * 7)]
    assert all(r[3] for r in res), res
