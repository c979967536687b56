"""The C oracle (oracle/ehyb_oracle.c, CPU baseline engine) reproduces the
reference engine's y bit for bit: small golden cases and the reference's y
digests at config scale, for several thread counts."""

import numpy as np
import pytest

import paper_2204_06666_b200 as E
from golden_data import config_record, small_case, small_meta
from golden_util import digest
from oracle import c_oracle
from paper_2204_06666_b200 import workloads as W
from pipeline_util import product_pipeline


@pytest.mark.parametrize("name", sorted(small_meta()))
def test_small(name):
    meta = small_meta()[name]
    g = small_case(name)
    *_, plan, e = product_pipeline(meta["n"], g["rows"], g["cols"], g["vals"], meta["tau"],
                                   meta["profile"], assignment=g.get("assignment_in"),
                                   n_parts_hint=meta["n_parts_hint"], rebalance=meta["rebalance"])
    xr = E.permute_vector(g["x"], plan)
    for threads in (1, 3):
        y = c_oracle.spmv_ehyb(e, xr, threads)
        assert y.tobytes() == g["y_reordered"].tobytes()


@pytest.mark.parametrize("name", ["cfg1", "cfg2s", "cfg3s", "cfg4s"])
def test_config_y_digest(name):
    rec = config_record(name)
    if rec is None:
        pytest.skip("golden record missing")
    n, r, c, v, tau = W.build_config(name)
    *_, plan, e = product_pipeline(n, r, c, v, tau, tuple(rec["profile"]))
    xr = E.permute_vector(W.deterministic_vector(n, 0), plan)
    prep = c_oracle.Prepared(e)
    for threads in (1, 8):
        assert digest(prep.spmv(xr, threads)) == rec["y_reordered"]


# ---- the C restatement of the reference preprocessing (oracle/ehyb_prep_oracle.c)

def _prep_arrays(e):
    """Parity arrays of a c_prep result, under the golden names."""
    cls, plan = e.classification, e.plan
    out = {"assignment": e.assignment, "part_sizes": e.part_sizes,
           "inner_counts": cls.inner_counts, "outer_counts": cls.outer_counts,
           "row_order": cls.row_order, "er_row_order": cls.er_row_order,
           "reorder_table": plan.reorder_table, "inverse_table": plan.inverse_table,
           "arrange_table": plan.arrange_table, "y_idx_er": plan.y_idx_er,
           "adj_ptr": e.adj_ptr, "adj": e.adj}
    for k in ("part_boundary", "position_ell", "width_ell", "ell_row_widths", "col_ell",
              "val_ell", "position_er", "width_er", "er_row_widths", "col_er", "val_er"):
        out[k] = getattr(e, k)
    return out


@pytest.mark.parametrize("name", sorted(small_meta()))
def test_prep_small_cases_match_reference(name):
    """Every parity array equals the reference's own (full arrays committed
    by make_golden.py) on the cases that use the default build path."""
    from oracle import c_prep

    meta = small_meta()[name]
    if meta["external"] or meta["rebalance"]:
        pytest.skip("external / rebalanced partition: not the default build path")
    g = small_case(name)
    e = c_prep.build_ehyb(meta["n"], g["rows"], g["cols"], g["vals"], meta["tau"],
                          tuple(meta["profile"]))
    got = _prep_arrays(e)
    for key, arr in got.items():
        if key in g:
            assert arr.dtype == g[key].dtype, (name, key)
            assert arr.tobytes() == g[key].tobytes(), (name, key)
    xr = np.zeros(e.padded_dimension, g["x"].dtype)
    xr[e.plan.reorder_table[: meta["n"]]] = g["x"]
    assert c_oracle.Prepared(e).spmv(xr, 2).tobytes() == g["y_reordered"].tobytes()


@pytest.mark.parametrize("name", ["cfg1", "cfg2s", "cfg3s", "cfg4s"])
def test_prep_config_digests_match_reference(name):
    from golden_util import GRAPH_ARRAYS, PARITY_ARRAYS
    from oracle import c_prep

    rec = config_record(name)
    if rec is None:
        pytest.skip("golden record missing")
    n, r, c, v, tau = W.build_config(name)
    e = c_prep.build_ehyb(n, r, c, v, tau, tuple(rec["profile"]))
    got = _prep_arrays(e)
    for key in PARITY_ARRAYS + GRAPH_ARRAYS:
        assert digest(got[key]) == rec["digests"][key], (name, key)
