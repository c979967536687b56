"""GPU parity of the fused sm_100a SpMV (through the C ABI) against the
reference: bitwise y (strict mode) on the golden small cases, the 512-case
corpus digests and the config-scale digests the reference itself produced;
tolerance checks for FMA mode and the cuSPARSE comparator; edge cases."""

import numpy as np
import pytest

import paper_2204_06666_b200 as E
from golden_data import config_record, corpus_digests, small_case, small_meta
from golden_util import digest
from oracle import c_oracle
from oracle import ehyb_oracle as O
from paper_2204_06666_b200 import workloads as W
from pipeline_util import product_pipeline

pytestmark = pytest.mark.gpu

torch = pytest.importorskip("torch")


def rel_error(y, y_ref):
    y = np.asarray(y, np.float64)
    y_ref = np.asarray(y_ref, np.float64)
    den = float(np.max(np.abs(y_ref))) if y_ref.size else 0.0
    diff = float(np.max(np.abs(y - y_ref))) if y_ref.size else 0.0
    return diff / den if den > 0 else diff


def small_e(name):
    meta = small_meta()[name]
    g = small_case(name)
    m, params, graph, parts, cls, plan, e = product_pipeline(
        meta["n"], g["rows"], g["cols"], g["vals"], meta["tau"], meta["profile"],
        assignment=g.get("assignment_in"), n_parts_hint=meta["n_parts_hint"],
        rebalance=meta["rebalance"])
    return meta, g, m, plan, e


@pytest.mark.parametrize("name", sorted(small_meta()))
def test_small_bitwise_numpy_path(name):
    meta, g, m, plan, e = small_e(name)
    exact = E.ExecutionConfig(exact=True)
    y, stats = E.spmv_ehyb(e, E.permute_vector(g["x"], plan), exact)
    assert y.dtype == g["y_reordered"].dtype
    assert y.tobytes() == g["y_reordered"].tobytes()
    assert stats.cached_loads == meta["cached_loads"]
    assert stats.uncached_loads == meta["uncached_loads"]
    assert stats.bytes_touched_model == meta["bytes_touched_model"]
    yu = E.spmv_ehyb_user(e, g["x"], exact)
    assert yu.tobytes() == g["y_user"].tobytes()
    # default mode: bitwise unless a row is wider than the long-row threshold
    yd, _ = E.spmv_ehyb(e, E.permute_vector(g["x"], plan))
    if E.device_matrix(e).info()["long_rows"] == 0:
        assert yd.tobytes() == y.tobytes()
    else:
        assert rel_error(yd, y) <= (1e-12 if meta["tau"] == 8 else 1e-5)


@pytest.mark.parametrize("name", sorted(small_meta()))
def test_small_torch_path_and_fma(name):
    meta, g, m, plan, e = small_e(name)
    dt = torch.float32 if meta["tau"] == 4 else torch.float64
    x = torch.from_numpy(g["x"]).to("cuda:0", dt)
    dm = E.device_matrix(e, 0)
    xr = dm.permute(x)
    assert np.array_equal(xr.cpu().numpy(), E.permute_vector(g["x"], plan).astype(xr.cpu().numpy().dtype))
    y = dm.spmv(xr, exact=True)
    torch.cuda.synchronize()
    assert y.cpu().numpy().tobytes() == g["y_reordered"].tobytes()
    yu = E.unpermute_vector(y, plan)
    assert yu.cpu().numpy().tobytes() == g["y_user"].tobytes()
    yf = dm.spmv_user(x, fma=True)
    tol = 1e-12 if meta["tau"] == 8 else 1e-5
    assert rel_error(yf.cpu().numpy(), g["y_csr"]) <= tol


def test_corpus_bitwise():
    recs = corpus_digests()
    for i, (rec, d) in enumerate(zip(recs, W.corpus_specs())):
        *_, plan, e = product_pipeline(d["n"], d["rows"], d["cols"], d["vals"], d["tau"],
                                       d["profile"], assignment=d["assignment"],
                                       n_parts_hint=d["n_parts_hint"], seed=d["seed"])
        xr = E.permute_vector(W.deterministic_vector(d["n"], i), plan)
        y, _ = E.spmv_ehyb(e, xr)
        assert digest(y) == rec["y_reordered"], d["name"]


_RGG_CACHE = {}


def _config_matrix(name):
    """cfg3f32 / cfg3f64 share one 5M-row matrix: generate it once."""
    if name.startswith("cfg3f"):
        if "m" not in _RGG_CACHE:
            _RGG_CACHE["m"] = W.rgg3d(5_000_000)
        n, r, c, v = _RGG_CACHE["m"]
        return n, r, c, v, 4 if name == "cfg3f32" else 8
    return W.build_config(name)


@pytest.mark.parametrize("name", ["cfg1", "cfg2s", "cfg3s", "cfg4s", "cfg2", "cfg4", "cfg5k4",
                                  "cfg3f32", "cfg3f64"])
def test_config_bitwise(name):
    rec = config_record(name)
    if rec is None:
        pytest.skip("golden record missing")
    n, r, c, v, tau = _config_matrix(name)
    m, params, graph, parts, cls, plan, e = product_pipeline(n, r, c, v, tau, tuple(rec["profile"]))
    assert digest(e.val_ell) == rec["digests"]["val_ell"]
    x = W.deterministic_vector(n, 0)
    exact = E.ExecutionConfig(exact=True)
    y, _ = E.spmv_ehyb(e, E.permute_vector(x, plan), exact)
    assert digest(y) == rec["y_reordered"]
    yu = E.spmv_ehyb_user(e, x, exact)
    assert digest(yu) == rec["y_user"]
    tol = 1e-12 if tau == 8 else 1e-5
    # FMA mode within the north-star tolerance of the strict result
    dm = E.device_matrix(e, 0)
    yt = dm.spmv_user(torch.from_numpy(x).to("cuda:0", dm.torch_dtype), fma=True)
    assert rel_error(yt.cpu().numpy(), yu) <= tol
    # the default mode: bitwise unless the matrix has rows wider than the
    # long-row threshold, whose segmented sums are within the tolerance
    yd, _ = E.spmv_ehyb(e, E.permute_vector(x, plan))
    if dm.info()["long_rows"] == 0:
        assert yd.tobytes() == y.tobytes()
    else:
        assert rel_error(yd, y) <= tol
    # repeated launches are bit-identical (no atomics in the data path)
    y2, _ = E.spmv_ehyb(e, E.permute_vector(x, plan), exact)
    assert y2.tobytes() == y.tobytes()
    yd2, _ = E.spmv_ehyb(e, E.permute_vector(x, plan))
    assert yd2.tobytes() == yd.tobytes()


def test_spmv_csr_is_bitwise_the_reference_oracle():
    """engine.py:56-69: np.add.reduceat order (first product + numpy pairwise
    sum), reproduced on the GPU — rows of 0..~2000 entries, empty rows,
    signed zeros, non-finite x."""
    n, r, c, v = W.permute_symmetric(*W.stencil27(20, 20, 20), seed=3)
    m = E.CooMatrix(n, n, r, c, v)
    x = W.deterministic_vector(n, 5)
    y = E.spmv_csr(E.coo_to_csr(m), x)
    assert y.tobytes() == O.spmv_csr(n, r, c, v, x).tobytes()
    rng = np.random.default_rng(11)
    n, nc = 3000, 12000  # rectangular: rows up to 9999 entries need that many columns
    lens = np.concatenate([np.arange(0, 300), rng.integers(0, 40, n - 310),
                           [1000, 1001, 1024, 1031, 1500, 2047, 2048, 2049, 4097, 9999]])
    rows = np.repeat(np.arange(n), lens)
    cols = np.concatenate([np.sort(rng.choice(nc, size=L, replace=False)) for L in lens])
    vals = rng.standard_normal(rows.size) * np.exp(rng.uniform(-30, 30, rows.size))
    vals[rng.integers(0, rows.size, 50)] = -0.0
    m = E.CooMatrix(n, nc, rows, cols, vals)
    csr = E.coo_to_csr(m)
    for xs in (rng.standard_normal(nc),
               np.where(rng.random(nc) < 0.01, np.inf, rng.standard_normal(nc)), -np.zeros(nc)):
        got = E.spmv_csr(csr, xs)
        want = O.spmv_csr(n, rows, cols, vals, xs)
        # bitwise, except that a NaN's payload is the hardware's
        nan = np.isnan(want)
        assert np.array_equal(np.isnan(got), nan)
        assert got[~nan].tobytes() == want[~nan].tobytes()


def test_cusparse_comparator_matches_oracle():
    from paper_2204_06666_b200.device import DeviceCsr

    n, r, c, v = W.permute_symmetric(*W.stencil27(20, 20, 20), seed=3)
    m = E.CooMatrix(n, n, r, c, v)
    csr = E.coo_to_csr(m)
    x = W.deterministic_vector(n, 5)
    dc = DeviceCsr(csr.n_rows, csr.n_cols, csr.row_ptr, csr.col_idx, csr.values, tau=8)
    xt = torch.from_numpy(x).cuda()
    want = O.spmv_csr(n, r, c, v, x)
    for alg in (1, 2):
        yt = torch.empty_like(xt)
        dc.spmv(xt, yt, alg=alg)
        assert rel_error(yt.cpu().numpy(), want) <= 1e-14


def test_window_in_global_memory_path():
    # window of 40,000 fp64 values (320 KB) exceeds shared memory: the kernel
    # gathers the window from global memory instead
    n, r, c, v = W.permute_symmetric(*W.stencil27(40, 40, 25), seed=2)
    m = E.CooMatrix(n, n, r, c, v)
    e = E.build_ehyb(m, tau=8, profile=E.DeviceProfile(1, 32, 1 << 20))
    dm = E.device_matrix(e, 0)
    assert dm.info()["window_in_smem"] == 0
    x = W.deterministic_vector(n, 1)
    xr = E.permute_vector(x, e.plan)
    y, _ = E.spmv_ehyb(e, xr)
    assert y.tobytes() == c_oracle.spmv_ehyb(e, xr).tobytes()


@pytest.mark.parametrize("tau", [4, 8])
def test_non_finite_x_matches_reference_engine(tau):
    # NaN/inf propagation including the reference's 0*x[0] padding products
    n, r, c, v = W.heavy_tail(k=12, n_hubs=3, min_len=50, max_len=400)
    m = E.CooMatrix(n, n, r, c, v)
    e = E.build_ehyb(m, tau=tau, profile=E.DeviceProfile(16, 32, 4096))
    x = W.deterministic_vector(n, 2)
    xr = E.permute_vector(x, e.plan)
    for bad in (np.inf, -np.inf, np.nan):
        xb = xr.copy()
        xb[0] = bad
        xb[7] = -np.inf
        y, _ = E.spmv_ehyb(e, xb, E.ExecutionConfig(exact=True))
        want = c_oracle.spmv_ehyb(e, xb)
        assert np.array_equal(np.isnan(y), np.isnan(want))
        fin = ~np.isnan(want)
        assert y[fin].tobytes() == want[fin].tobytes()


def test_edge_cases():
    # empty matrix, identity, every entry outer (ER only)
    e = E.build_ehyb(E.CooMatrix(6, 6, [], [], []), tau=8, profile=E.DeviceProfile(2, 4, 64))
    y, _ = E.spmv_ehyb(e, np.ones(e.padded_dimension))
    assert np.array_equal(y, np.zeros(e.padded_dimension))
    e = E.build_ehyb(E.CooMatrix(5, 5, np.arange(5), np.arange(5), np.arange(5.0)),
                     tau=4, profile=E.DeviceProfile(2, 4, 64))
    x = np.arange(5.0) + 1
    assert np.array_equal(E.spmv_ehyb_user(e, x), (np.arange(5.0) * x).astype(np.float32))
    n = 64
    rows = np.arange(n)
    cols = (rows + n // 2) % n
    m = E.CooMatrix(n, n, rows, cols, np.linspace(1, 2, n))
    parts = E.PartitionMap.from_assignment(np.arange(n) // 16, n_parts=4)
    e = E.build_ehyb(m, tau=8, profile=E.DeviceProfile(4, 4, 128), partition=parts)
    assert e.nnz_ell == 0 and e.nnz_er == n
    x = W.deterministic_vector(n, 3)
    xr = E.permute_vector(x, e.plan)
    y, _ = E.spmv_ehyb(e, xr)
    assert y.tobytes() == c_oracle.spmv_ehyb(e, xr).tobytes()
    with pytest.raises(ValueError, match="length mismatch"):
        E.spmv_ehyb(e, np.zeros(3))
    with pytest.raises(ValueError, match="length mismatch"):
        E.spmv_ehyb_user(e, np.zeros(n + 1))


@pytest.mark.parametrize("user_order", [True, False])
def test_host_many_pipeline_matches_single_calls(user_order):
    # the pipelined host path (copy-in / product / copy-out of neighbouring
    # vectors overlapped) gives each vector exactly the single-call result
    n, r, c, v = W.permute_symmetric(*W.stencil27(24, 24, 24), seed=5)
    m = E.CooMatrix(n, n, r, c, v)
    e = E.build_ehyb(m, tau=8, profile=E.DeviceProfile(12, 32, 16384))
    dm = E.device_matrix(e, 0)
    length = n if user_order else e.padded_dimension
    xs = [torch.from_numpy(W.deterministic_vector(length, s)).pin_memory().numpy()
          for s in range(7)]
    ys = [torch.empty(length, dtype=torch.float64).pin_memory().numpy() for _ in xs]
    out = dm.spmv_host_many(xs, user_order=user_order, out=ys)
    assert out is ys
    for x, y in zip(xs, ys):
        want = dm.spmv_host(x, user_order=user_order)
        assert y.tobytes() == want.tobytes()
    # pageable inputs, a 2-D batch, and the empty batch
    X = np.stack([W.deterministic_vector(length, 9 + s) for s in range(3)])
    Y = dm.spmv_host_many(X, user_order=user_order)
    for x, y in zip(X, Y):
        assert y.tobytes() == dm.spmv_host(x, user_order=user_order).tobytes()
    assert dm.spmv_host_many([], user_order=user_order) == []
    with pytest.raises(ValueError, match="length mismatch"):
        dm.spmv_host_many([np.zeros(3)], user_order=user_order)


def _fresh_handle(e, monkeypatch, long_row):
    from paper_2204_06666_b200.device import DeviceMatrix

    monkeypatch.setenv("EHYB_LONG_ROW", str(long_row))
    return DeviceMatrix(e, 0)


@pytest.mark.parametrize("tau", [4, 8])
@pytest.mark.parametrize("case", ["hubs", "many", "warp4"])
def test_long_rows_bitwise_strict_and_fma_tolerance(monkeypatch, tau, case):
    # rows wider than EHYB_LONG_ROW leave the slice paths and run as whole-warp
    # serial chains (strict) or reassociated segments (FMA mode)
    if case == "hubs":
        n, r, c, v = W.heavy_tail(k=16, n_hubs=4, min_len=200, max_len=3000)
        prof, long_row = E.DeviceProfile(16, 32, 8192), 48
    elif case == "many":  # most 27-point rows become long rows
        n, r, c, v = W.permute_symmetric(*W.stencil27(16, 16, 16), seed=2)
        prof, long_row = E.DeviceProfile(8, 32, 8192), 12
    else:  # generic slice height
        n, r, c, v = W.heavy_tail(k=10, n_hubs=3, min_len=50, max_len=400)
        prof, long_row = E.DeviceProfile(8, 4, 8192), 16
    m = E.CooMatrix(n, n, r, c, v)
    e = E.build_ehyb(m, tau=tau, profile=prof)
    dm = _fresh_handle(e, monkeypatch, long_row)
    assert dm.info()["long_rows"] > 0
    dt = dm.torch_dtype
    for seed in (0, 1):
        x = W.deterministic_vector(n, seed)
        xr = E.permute_vector(x, e.plan)
        want = c_oracle.spmv_ehyb(e, xr)
        xt = torch.from_numpy(xr).to("cuda:0", dt)
        for _ in range(3):  # repeated launches: per-launch counters reset
            y = dm.spmv(xt, exact=True)
            torch.cuda.synchronize()
            assert y.cpu().numpy().tobytes() == want.tobytes()
        yf = dm.spmv(xt, fma=True)
        yf2 = dm.spmv(xt, fma=True)
        torch.cuda.synchronize()
        assert yf.cpu().numpy().tobytes() == yf2.cpu().numpy().tobytes()  # deterministic
        tol = 1e-12 if tau == 8 else 1e-5
        assert rel_error(yf.cpu().numpy(), want) <= tol
        # default mode: slice rows bitwise strict, long rows the segmented sums
        # (the same code as FMA mode's long rows), deterministic
        yd = dm.spmv(xt).cpu().numpy()
        assert dm.spmv(xt).cpu().numpy().tobytes() == yd.tobytes()
        assert rel_error(yd, want) <= tol
        yfn = yf.cpu().numpy()
        same = (yd.view(np.uint8).reshape(-1, yd.itemsize) == want.view(np.uint8).reshape(
            -1, yd.itemsize)).all(1)
        same |= (yd.view(np.uint8).reshape(-1, yd.itemsize) == yfn.view(np.uint8).reshape(
            -1, yd.itemsize)).all(1)
        assert same.all()
    # non-finite x: the reference's padding products propagate NaN/inf
    xb = E.permute_vector(W.deterministic_vector(n, 3), e.plan)
    xb[0] = np.nan
    xb[e.params.vec_cache_size] = np.inf
    want = c_oracle.spmv_ehyb(e, xb)
    y = dm.spmv(torch.from_numpy(xb).to("cuda:0", dt), exact=True).cpu().numpy()
    assert np.array_equal(np.isnan(y), np.isnan(want))
    fin = ~np.isnan(want)
    assert y[fin].tobytes() == want[fin].tobytes()
    dm.close()


def test_persistent_ctas_multiple_partitions_per_cta():
    # more partitions than resident CTAs (148 x 1 per SM): every CTA loops
    # over several partitions, re-staging its window each time
    n, r, c, v = W.permute_symmetric(*W.stencil27(40, 40, 40), seed=4)
    m = E.CooMatrix(n, n, r, c, v)
    e = E.build_ehyb(m, tau=8, profile=E.DeviceProfile(600, 32, 4096))
    assert e.n_parts >= 600
    dm = E.device_matrix(e, 0)
    assert dm.info()["ctas"] < e.n_parts
    x = W.deterministic_vector(n, 6)
    xr = E.permute_vector(x, e.plan)
    want = c_oracle.spmv_ehyb(e, xr)
    for _ in range(3):
        y, _ = E.spmv_ehyb(e, xr)
        assert y.tobytes() == want.tobytes()
    # the split launches of the sharded path (local phase, then halo phase)
    # with several partitions per CTA, two shards
    from paper_2204_06666_b200 import distributed as D

    for world in (1, 2):
        for rank in range(world):
            plan = D.plan_for(e, rank, world)
            A = D.DistributedEhyb(e, device=0, plan=plan)
            lo, hi = plan.p0 * plan.vec, plan.p1 * plan.vec
            x_ext = A.new_ext()
            x_ext[: plan.local_rows] = torch.from_numpy(xr[lo:hi])
            x_ext[plan.local_rows:] = torch.from_numpy(xr[plan.halo_cols])
            ys = torch.empty(plan.local_rows, dtype=torch.float64, device="cuda:0")
            for _ in range(2):
                A.spmv_local(x_ext, ys)
                torch.cuda.synchronize()
                assert ys.cpu().numpy().tobytes() == want[lo:hi].tobytes()


def test_launch_kind_sequences_keep_per_launch_counters():
    # any interleaving of full / local / halo launches must reset the
    # per-launch counters of the next launch (they alternate by epoch parity)
    import ctypes as C
    from paper_2204_06666_b200 import _lib as L
    from paper_2204_06666_b200 import distributed as D

    for prof in (E.DeviceProfile(600, 32, 4096), E.DeviceProfile(24, 32, 8192)):
        n, r, c, v = W.permute_symmetric(*W.stencil27(40, 40, 40), seed=4)
        e = E.build_ehyb(E.CooMatrix(n, n, r, c, v), tau=8, profile=prof)
        xr = E.permute_vector(W.deterministic_vector(n, 6), e.plan)
        want = c_oracle.spmv_ehyb(e, xr)
        plan = D.plan_for(e, 0, 1)
        A = D.DistributedEhyb(e, device=0, plan=plan)
        x_ext = A.new_ext()
        x_ext[: plan.local_rows] = torch.from_numpy(xr)
        st = C.c_void_p(torch.cuda.current_stream().cuda_stream)
        seqs = [["ehyb_dev_spmv"], ["ehyb_dev_spmv_ell", "ehyb_dev_spmv_er"],
                ["ehyb_dev_spmv_ell", "ehyb_dev_spmv_er"], ["ehyb_dev_spmv"],
                ["ehyb_dev_spmv_ell", "ehyb_dev_spmv_er"], ["ehyb_dev_spmv"], ["ehyb_dev_spmv"]]
        for seq in seqs:
            y = torch.zeros(plan.local_rows, dtype=torch.float64, device="cuda:0")
            for name in seq:
                L.call(name, A._h, C.c_void_p(x_ext.data_ptr()), C.c_void_p(y.data_ptr()),
                       L.MODE_STRICT, st)
            torch.cuda.synchronize()
            assert y.cpu().numpy().tobytes() == want.tobytes(), seq


def test_fused_launch_beside_busy_kernels():
    # the fused kernel's pool / persistent-CTA protocols spin on flags other
    # CTAs write; the cooperative launch keeps the whole grid co-resident
    # while another stream keeps the SMs busy (GEMMs issued just before)
    busy, work = torch.cuda.Stream(), torch.cuda.Stream()
    a = torch.randn(4096, 4096, device="cuda:0")
    b = torch.randn(4096, 4096, device="cuda:0")
    c = torch.empty_like(a)
    for prof in (E.DeviceProfile(16, 32, 8192), E.DeviceProfile(600, 32, 4096)):
        n, r, cc, v = W.permute_symmetric(*W.stencil27(24, 24, 24), seed=5)
        e = E.build_ehyb(E.CooMatrix(n, n, r, cc, v), tau=8, profile=prof)
        dm = E.device_matrix(e, 0)
        xr = E.permute_vector(W.deterministic_vector(n, 9), e.plan)
        want = c_oracle.spmv_ehyb(e, xr)
        xt = torch.from_numpy(xr).to("cuda:0")
        torch.cuda.synchronize()
        ys = []
        for _ in range(4):
            with torch.cuda.stream(busy):
                for _ in range(8):
                    torch.mm(a, b, out=c)
            ys.append(dm.spmv(xt, stream=work))
        torch.cuda.synchronize()
        for y in ys:
            assert y.cpu().numpy().tobytes() == want.tobytes()


@pytest.mark.parametrize("split", [1, 2, 3, 4])
@pytest.mark.parametrize("tau", [4, 8])
def test_work_units_split_partitions(monkeypatch, split, tau):
    # a partition's chunks split over `split` CTAs (each stages the window):
    # the multi-GPU path when a rank owns fewer partitions than SMs. Bitwise
    # on the pool, persistent and shard paths, long rows included
    from paper_2204_06666_b200 import distributed as D
    from paper_2204_06666_b200.device import DeviceMatrix

    monkeypatch.setenv("EHYB_SPLIT", str(split))
    monkeypatch.setenv("EHYB_LONG_ROW", "60")
    n, r, c, v = W.heavy_tail(k=20, n_hubs=3, min_len=100, max_len=900)
    for prof in (E.DeviceProfile(6, 32, 16384), E.DeviceProfile(400, 32, 2048)):
        e = E.build_ehyb(E.CooMatrix(n, n, r, c, v), tau=tau, profile=prof)
        dm = DeviceMatrix(e, 0)
        info = dm.info()
        assert info["split"] >= 1 and info["work_units"] == e.n_parts * info["split"]
        if prof.num_processors == 6:
            assert info["split"] == min(split, (e.params.vec_cache_size + 31) // 32)
        xr = E.permute_vector(W.deterministic_vector(n, split), e.plan)
        want = c_oracle.spmv_ehyb(e, xr)
        xt = torch.from_numpy(xr).to("cuda:0", dm.torch_dtype)
        for _ in range(2):
            assert dm.spmv(xt, exact=True).cpu().numpy().tobytes() == want.tobytes()
        dm.close()
        for world in (2, 3):
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
                assert ys.cpu().numpy().tobytes() == want[lo:hi].tobytes()


@pytest.mark.gpu
@pytest.mark.parametrize("tau", [8, 4])
@pytest.mark.parametrize("knobs", [
    {"EHYB_META_SMEM": "0"}, {"EHYB_META_SMEM": "1"},
    {"EHYB_ORDER_UNITS": "1"}, {"EHYB_ORDER_UNITS": "1", "EHYB_META_SMEM": "1"},
    {"EHYB_ER_WARPS": "12"}, {"EHYB_POOL_FACTOR_LAST": "1.2"},
])
def test_launch_layout_knobs_keep_y_bitwise(monkeypatch, knobs, tau):
    # derived launch layouts (chunk metadata in shared memory, units in cost
    # order with their unit -> partition table, ER-first warp count, the last
    # iteration's pool share) change only where and when rows are computed:
    # y stays bitwise the reference restatement's, one wave and persistent
    n, r, c, v = W.permute_symmetric(*W.stencil27(40, 40, 40), seed=5)
    m = E.CooMatrix(n, n, r, c, v)
    x = W.deterministic_vector(n, 7)
    for k, val in knobs.items():
        monkeypatch.setenv(k, val)
    for prof in (E.DeviceProfile(600, 32, 4096), E.DeviceProfile(64, 32, 4096)):
        e = E.build_ehyb(m, tau=tau, profile=prof)
        xr = E.permute_vector(x, e.plan).astype(e.params.value_dtype)
        want = c_oracle.spmv_ehyb(e, xr)
        dm = E.device_matrix(e, 0)
        xt = torch.from_numpy(xr).to("cuda:0")
        for _ in range(2):
            y = dm.spmv(xt)
            torch.cuda.synchronize()
            assert y.cpu().numpy().tobytes() == want.tobytes()
        dm.close()
