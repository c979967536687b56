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
