"""Seeded randomized parity sweep of the fused kernel against the C
restatement of the reference engine (itself pinned to the reference's golden
vectors): random structures (uniform, banded + hubs, permuted stencils),
both precisions, slice heights 32/8/4/1, profiles from one partition to more
partitions than resident CTAs, long-row thresholds, and 1-3 shards. Strict
mode must be bitwise; FMA mode within the north-star tolerance."""

import ctypes as C

import numpy as np
import pytest

import paper_2204_06666_b200 as E
from oracle import c_oracle
from paper_2204_06666_b200 import distributed as D
from paper_2204_06666_b200 import workloads as W
from paper_2204_06666_b200 import _lib as L

pytestmark = pytest.mark.gpu

torch = pytest.importorskip("torch")


def _matrix(kind, rng):
    if kind == "uniform":
        n = int(rng.integers(50, 3000))
        return W.random_coo(n, float(rng.uniform(0.5, 8.0)) / n, int(rng.integers(1 << 30)))
    if kind == "hubs":
        k = int(rng.integers(8, 16))
        return W.heavy_tail(k=k, n_hubs=int(rng.integers(1, 5)), seed=int(rng.integers(1 << 30)),
                            min_len=20, max_len=int(rng.integers(100, 1500)))
    k = int(rng.integers(6, 20))
    return W.permute_symmetric(*W.stencil27(k, k, int(rng.integers(4, 24))),
                               seed=int(rng.integers(1 << 30)))


CASES = [(seed, kind) for seed in range(30) for kind in ("uniform", "hubs", "stencil")]


@pytest.mark.parametrize("seed,kind", CASES)
def test_random_structures_bitwise(seed, kind, monkeypatch):
    rng = np.random.default_rng(1000 + seed)
    n, r, c, v = _matrix(kind, rng)
    m = E.CooMatrix(n, n, r, c, v)
    tau = int(rng.choice([4, 8]))
    warp = int(rng.choice([32, 32, 8, 4, 1]))
    procs = int(rng.choice([1, 3, 16, 64, 300]))
    shm = int(rng.choice([2048, 8192, 65536]))
    try:
        e = E.build_ehyb(m, tau=tau, profile=E.DeviceProfile(procs, warp, shm))
    except ValueError:
        pytest.skip("infeasible profile for this draw")
    monkeypatch.setenv("EHYB_LONG_ROW", str(int(rng.choice([8, 32, 128, 100000]))))
    from paper_2204_06666_b200.device import DeviceMatrix

    dm = DeviceMatrix(e, 0)
    x = W.deterministic_vector(n, seed)
    xr = E.permute_vector(x, e.plan)
    want = c_oracle.spmv_ehyb(e, xr)
    xt = torch.from_numpy(xr).to("cuda:0", dm.torch_dtype)
    y = dm.spmv(xt, exact=True)
    y2 = dm.spmv(xt, exact=True)
    torch.cuda.synchronize()
    assert y.cpu().numpy().tobytes() == want.tobytes()
    assert y2.cpu().numpy().tobytes() == want.tobytes()
    yf = dm.spmv(xt, fma=True).cpu().numpy().astype(np.float64)
    den = max(float(np.max(np.abs(want))), 1e-300)
    tol = 1e-12 if tau == 8 else 1e-5
    assert float(np.max(np.abs(yf - want))) / den <= tol
    # default mode: bitwise without long rows, else within the tolerance
    yd = dm.spmv(xt).cpu().numpy()
    if dm.info()["long_rows"] == 0:
        assert yd.tobytes() == want.tobytes()
    else:
        assert float(np.max(np.abs(yd.astype(np.float64) - want))) / den <= tol
    # the sharded path: local + halo launches per shard
    world = int(rng.integers(1, 4))
    if e.n_parts >= world:
        st = C.c_void_p(torch.cuda.current_stream().cuda_stream)
        for rank in range(world):
            plan = D.plan_for(e, rank, world)
            A = D.DistributedEhyb(e, device=0, plan=plan)
            lo, hi = plan.p0 * plan.vec, plan.p1 * plan.vec
            x_ext = A.new_ext()
            x_ext[: plan.local_rows] = torch.from_numpy(xr[lo:hi]).to(A.dtype)
            x_ext[plan.local_rows:] = torch.from_numpy(xr[plan.halo_cols]).to(A.dtype)
            ys = torch.empty(plan.local_rows, dtype=A.dtype, device="cuda:0")
            A.spmv_local(x_ext, ys, exact=True)
            torch.cuda.synchronize()
            got = ys.cpu().numpy()
            # byte-identical, the sign of zero included: shards reproduce the
            # reference's ER padding products (inline, or after the exchange
            # when another rank owns the padding column)
            ref = want[lo:hi]
            assert got.tobytes() == ref.tobytes()
            L.call("ehyb_dev_spmv", A._h, C.c_void_p(x_ext.data_ptr()),
                   C.c_void_p(ys.data_ptr()), L.MODE_STRICT, st)
            torch.cuda.synchronize()
            assert ys.cpu().numpy().tobytes() == ref.tobytes()
    dm.close()


def _same_modulo_nan_payload(got, want):
    nan = np.isnan(want)
    return np.array_equal(np.isnan(got), nan) and got[~nan].tobytes() == want[~nan].tobytes()


@pytest.mark.parametrize("tau", [8, 4])
@pytest.mark.parametrize("bad", [np.inf, -np.inf, np.nan, -0.0, 0.0, -3.0])
def test_shards_reproduce_padding_products(tau, bad):
    """x[pad column] non-finite or a signed zero, and -0.0 row sums: every
    shard's y equals the reference engine's byte for byte (NaN payloads
    aside), also on shards that do not own the padding column."""
    n, r, c, v = W.permute_symmetric(*W.stencil27(14, 14, 10), seed=5)
    # rows whose products cancel to -0.0: negative-zero values on a few rows
    v = v.copy()
    v[r % 97 == 3] = -0.0
    m = E.CooMatrix(n, n, r, c, v)
    e = E.build_ehyb(m, tau=tau, profile=E.DeviceProfile(12, 32, 4096 * tau // 8))
    assert e.nnz_er > 0
    xr = E.permute_vector(W.deterministic_vector(n, 3), e.plan)
    xr[np.arange(xr.size) % 53 == 1] = -0.0
    xr[D.er_pad_column(e)] = bad
    want = c_oracle.spmv_ehyb(e, xr)
    st = C.c_void_p(torch.cuda.current_stream().cuda_stream)
    for world in (2, 3):
        for rank in range(world):
            plan = D.plan_for(e, rank, world)
            A = D.DistributedEhyb(e, device=0, plan=plan)
            lo, hi = plan.p0 * plan.vec, plan.p1 * plan.vec
            x_ext = A.new_ext()
            x_ext[: plan.local_rows] = torch.from_numpy(xr[lo:hi]).to(A.dtype)
            x_ext[plan.local_rows:] = torch.from_numpy(xr[plan.halo_cols]).to(A.dtype)
            ys = torch.empty(plan.local_rows, dtype=A.dtype, device="cuda:0")
            A.spmv_local(x_ext, ys)
            torch.cuda.synchronize()
            assert _same_modulo_nan_payload(ys.cpu().numpy(), want[lo:hi]), (world, rank)
            L.call("ehyb_dev_spmv", A._h, C.c_void_p(x_ext.data_ptr()),
                   C.c_void_p(ys.data_ptr()), L.MODE_STRICT, st)
            torch.cuda.synchronize()
            assert _same_modulo_nan_payload(ys.cpu().numpy(), want[lo:hi]), (world, rank)
