"""Native preprocessing (csrc/prep.cpp via the C ABI) is byte-identical to
the reference: full arrays for the small golden cases, digests for the
512-case corpus and for the BASELINE configs. CPU only (no GPU needed)."""

import numpy as np
import pytest

import paper_2204_06666_b200 as E
from golden_data import config_record, corpus_digests, small_case, small_meta
from golden_util import GRAPH_ARRAYS, PARITY_ARRAYS, collect, digest
from paper_2204_06666_b200 import workloads as W
from pipeline_util import product_pipeline


@pytest.mark.parametrize("name", sorted(small_meta()))
def test_small_case_bit_exact(name):
    meta = small_meta()[name]
    g = small_case(name)
    m, params, graph, parts, cls, plan, e = product_pipeline(
        meta["n"], g["rows"], g["cols"], g["vals"], meta["tau"], meta["profile"],
        assignment=g.get("assignment_in"), n_parts_hint=meta["n_parts_hint"],
        rebalance=meta["rebalance"])
    got = collect(parts, cls, plan, e, graph=graph)
    for key in PARITY_ARRAYS + GRAPH_ARRAYS:
        assert got[key].dtype == g[key].dtype, key
        assert np.array_equal(got[key], g[key]), key
    assert E.traffic_model(e) == meta["traffic_model"]
    assert E.footprint_stats(e).__dict__ == meta["footprint"]
    assert (e.nnz_ell, e.nnz_er) == (meta["nnz_ell"], meta["nnz_er"])
    # conservation: ehyb_to_coo inverts the assembly (format.py:463-498)
    back = E.ehyb_to_coo(e)
    vals = g["vals"] if meta["tau"] == 8 else g["vals"].astype(np.float32).astype(np.float64)
    key = lambda r, c, v: np.lexsort((v, c, r))
    o1 = key(back.rows, back.cols, back.values)
    o2 = key(g["rows"], g["cols"], vals)
    assert np.array_equal(back.rows[o1], g["rows"][o2])
    assert np.array_equal(back.cols[o1], g["cols"][o2])
    assert np.array_equal(back.values[o1], vals[o2])


def test_build_ehyb_rebalance_matches():
    meta = small_meta()["rebalance_tridiag16"]
    g = small_case("rebalance_tridiag16")
    m = E.CooMatrix(meta["n"], meta["n"], g["rows"], g["cols"], g["vals"])
    e = E.build_ehyb(m, tau=8, profile=E.DeviceProfile(*meta["profile"]),
                     partition=E.PartitionMap.from_assignment(g["assignment_in"], n_parts=1))
    assert e.n_parts == 2
    assert np.array_equal(e.val_ell, g["val_ell"])
    assert np.array_equal(e.plan.reorder_table, g["reorder_table"])


def test_corpus_digests():
    recs = corpus_digests()
    for i, (rec, d) in enumerate(zip(recs, W.corpus_specs())):
        assert rec["name"] == d["name"]
        m, params, graph, parts, cls, plan, e = product_pipeline(
            d["n"], d["rows"], d["cols"], d["vals"], d["tau"], d["profile"],
            assignment=d["assignment"], n_parts_hint=d["n_parts_hint"], seed=d["seed"])
        got = collect(parts, cls, plan, e, graph=graph)
        for key in PARITY_ARRAYS + GRAPH_ARRAYS:
            assert digest(got[key]) == rec["digests"][key], (d["name"], key)
        assert E.traffic_model(e) == rec["traffic_model"]


@pytest.mark.parametrize("name", ["cfg1", "cfg2s", "cfg3s", "cfg4s"])
def test_config_digests(name):
    rec = config_record(name)
    if rec is None:
        pytest.skip(f"golden record for {name} not generated")
    n, r, c, v, tau = W.build_config(name)
    m, params, graph, parts, cls, plan, e = product_pipeline(n, r, c, v, tau, tuple(rec["profile"]))
    got = collect(parts, cls, plan, e, graph=graph)
    for key in PARITY_ARRAYS + GRAPH_ARRAYS:
        assert digest(got[key]) == rec["digests"][key], (name, key)
    assert (e.nnz_ell, e.nnz_er) == (rec["nnz_ell"], rec["nnz_er"])
    assert E.traffic_model(e) == rec["traffic_model"]


@pytest.mark.slow
@pytest.mark.parametrize("name", ["cfg2", "cfg3f32", "cfg3f64", "cfg4", "cfg5k4"])
def test_config_digests_full(name):
    test_config_digests.__wrapped__(name) if hasattr(test_config_digests, "__wrapped__") else None
    rec = config_record(name)
    if rec is None:
        pytest.skip(f"golden record for {name} not generated")
    n, r, c, v, tau = W.build_config(name)
    m, params, graph, parts, cls, plan, e = product_pipeline(n, r, c, v, tau, tuple(rec["profile"]))
    got = collect(parts, cls, plan, e, graph=graph)
    for key in PARITY_ARRAYS + GRAPH_ARRAYS:
        assert digest(got[key]) == rec["digests"][key], (name, key)


def test_errors_match_reference_wording():
    with pytest.raises(ValueError, match="infeasible"):
        E.compute_params(100, 8, E.DeviceProfile(1, 32, 128))
    with pytest.raises(ValueError, match="square"):
        E.build_ehyb(E.CooMatrix(2, 3, [0], [1], [1.0]))
    n, r, c, v = W.tridiagonal(8)
    m = E.CooMatrix(n, n, r, c, v)
    with pytest.raises(ValueError, match="dimension mismatch"):
        E.classify_rows(m, E.PartitionMap.from_assignment([0, 0]))
    params = E.compute_params(8, 8, E.DeviceProfile(2, 4, 64))
    overfull = E.PartitionMap.from_assignment([0] * 6 + [1] * 2)
    with pytest.raises(ValueError, match="capacity"):
        E.build_reorder_plan(E.classify_rows(m, overfull), params, overfull)
    with pytest.raises(ValueError, match="infeasible"):
        E.partition_graph(E.build_graph(m), 2, 3)
    with pytest.raises(ValueError, match="parts"):
        E.build_ehyb(m, tau=8, profile=E.DeviceProfile(2, 4, 64),
                     partition=E.random_partition(8, 8, None, seed=0))


@pytest.mark.parametrize("tau,n", [(4, 3000), (8, 3000), (8, 20000)])
def test_duplicate_coordinates_keep_entry_order(tau, n):
    """Duplicate (row, col) entries in scrambled COO order: the native
    radix grouping must reproduce np.lexsort((cols, rows)) — duplicates in
    entry order (format.py:319) — so every parity array equals the oracle's."""
    from oracle import ehyb_oracle as O

    rng = np.random.default_rng(11)
    r = rng.integers(0, n, size=40000)
    c = np.clip(r + rng.integers(-40, 41, size=r.size), 0, n - 1)
    dup = rng.integers(0, r.size, size=5000)  # repeated coordinates, new values
    rows = np.concatenate([r, r[dup]]).astype(np.int64)
    cols = np.concatenate([c, c[dup]]).astype(np.int64)
    vals = rng.uniform(-1, 1, size=rows.size)
    perm = rng.permutation(rows.size)
    rows, cols, vals = rows[perm], cols[perm], vals[perm]
    profile = (4 if n < 10000 else 16, 32, 48 * 1024)
    _, _, _, _, _, _, e = product_pipeline(n, rows, cols, vals, tau, profile)
    s = O.pipeline(n, rows, cols, vals, tau, *profile)
    for key in ("val_ell", "col_ell", "val_er", "col_er", "position_ell", "width_ell",
                "position_er", "width_er", "ell_row_widths", "er_row_widths"):
        got = np.asarray(getattr(e, key))
        assert got.tobytes() == np.asarray(s[key]).tobytes(), key


def test_large_dimension_radix_buckets():
    """n above 2^23 (row buckets of 4096 rows: the in-bucket row pass is wider
    than the 11-bit column passes). build_graph against np.unique over the
    symmetric keys (partition.py:92-98) and the SELL slabs against a
    vectorised restatement of assemble_ehyb's placement (format.py:319-380)."""
    rng = np.random.default_rng(5)
    n = (1 << 23) + 4099
    hubs = rng.integers(0, n, size=4000)
    rows = np.concatenate([hubs, rng.choice(hubs, 60000)]).astype(np.int64)
    cols = np.concatenate([hubs, rng.choice(hubs, 60000)]).astype(np.int64)
    rows = np.concatenate([rows, rows[:5000]])  # duplicate coordinates
    cols = np.concatenate([cols, cols[:5000]])
    vals = rng.uniform(-1, 1, size=rows.size)
    perm = rng.permutation(rows.size)
    rows, cols, vals = rows[perm], cols[perm], vals[perm]
    m, params, g, parts, cls, plan, e = product_pipeline(
        n, rows, cols, vals, 8, (296, 32, 231424))
    off = rows != cols
    keys = np.unique(np.concatenate([rows[off] * n + cols[off], cols[off] * n + rows[off]]))
    assert np.array_equal(g.adj_ptr, np.concatenate([[0], np.cumsum(np.bincount(keys // n, minlength=n))]))
    assert np.array_equal(g.adj, (keys % n).astype(np.int32))

    C, vec = params.warp_size, params.vec_cache_size
    asg, reorder, arrange = parts.assignment, plan.reorder_table, plan.arrange_table
    order = np.lexsort((np.arange(rows.size), cols, rows))
    r, c, v = rows[order], cols[order], vals[order]
    inner = asg[r] == asg[c]

    def ranks(rr):
        return np.arange(rr.size) - np.searchsorted(rr, rr, side="left")

    ri, ci = r[inner], c[inner]
    nr = reorder[ri]
    d = e.position_ell[nr // C] + nr % C + ranks(ri) * C
    want_v = np.zeros_like(e.val_ell)
    want_c = np.zeros_like(e.col_ell)
    want_v[d] = v[inner]
    want_c[d] = reorder[ci] - (nr // vec) * vec
    assert want_v.tobytes() == e.val_ell.tobytes()
    assert want_c.tobytes() == e.col_ell.tobytes()
    ro, co = r[~inner], c[~inner]
    slot = arrange[ro]
    d = e.position_er[slot // C] + slot % C + ranks(ro) * C
    want_v = np.zeros_like(e.val_er)
    want_c = np.zeros_like(e.col_er)
    want_v[d] = v[~inner]
    want_c[d] = reorder[co]
    assert want_v.tobytes() == e.val_er.tobytes()
    assert want_c.tobytes() == e.col_er.tobytes()
