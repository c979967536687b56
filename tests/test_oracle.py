"""The oracle (oracle/ehyb_oracle.py) pinned against the real reference's
golden fixtures: full arrays for small cases, digests for the 512-case corpus."""

import numpy as np
import pytest

from golden_data import corpus_digests, small_case, small_meta
from golden_util import GRAPH_ARRAYS, PARITY_ARRAYS, digest
from oracle import ehyb_oracle as O
from paper_2204_06666_b200 import workloads as W


def run_small(name):
    meta = small_meta()[name]
    g = small_case(name)
    procs, warp, shm = meta["profile"]
    s = O.pipeline(meta["n"], g["rows"], g["cols"], g["vals"], meta["tau"], procs, warp, shm,
                   assignment=g.get("assignment_in"), n_parts_hint=meta["n_parts_hint"],
                   rebalance=meta["rebalance"])
    return meta, g, s


@pytest.mark.parametrize("name", sorted(small_meta()))
def test_small_case_bit_exact(name):
    meta, g, s = run_small(name)
    for key in PARITY_ARRAYS + GRAPH_ARRAYS:
        want = g[key]
        got = s[key]
        assert got.dtype == want.dtype, (key, got.dtype, want.dtype)
        assert np.array_equal(got, want), key
    y = O.spmv_ehyb(s, O.permute_vector(g["x"], s["reorder_table"], meta["n"],
                                        s["_meta"]["n_parts"] * s["_meta"]["vec"]))
    assert y.dtype == g["y_reordered"].dtype
    assert y.tobytes() == g["y_reordered"].tobytes()
    yu = O.unpermute_vector(y, s["reorder_table"], meta["n"])
    assert yu.tobytes() == g["y_user"].tobytes()
    ycsr = O.spmv_csr(meta["n"], g["rows"], g["cols"], g["vals"], g["x"])
    assert ycsr.tobytes() == g["y_csr"].tobytes()
    assert O.traffic_model(s) == meta["traffic_model"]


def test_corpus_digests():
    recs = corpus_digests()
    specs = list(W.corpus_specs())
    assert len(recs) == len(specs) == 512
    for i, (rec, d) in enumerate(zip(recs, specs)):
        assert rec["name"] == d["name"]
        procs, warp, shm = d["profile"]
        s = O.pipeline(d["n"], d["rows"], d["cols"], d["vals"], d["tau"], procs, warp, shm,
                       assignment=d["assignment"], n_parts_hint=d["n_parts_hint"],
                       seed=d["seed"])
        for key in PARITY_ARRAYS + GRAPH_ARRAYS:
            assert digest(s[key]) == rec["digests"][key], (d["name"], key)
        x = W.deterministic_vector(d["n"], i)
        xr = O.permute_vector(x, s["reorder_table"], d["n"],
                              s["_meta"]["n_parts"] * s["_meta"]["vec"])
        assert digest(O.spmv_ehyb(s, xr)) == rec["y_reordered"], d["name"]
        assert O.traffic_model(s) == rec["traffic_model"]


def test_compute_params_kats():
    # reference tests/test_format.py:46-57 known answers
    assert O.compute_params(1_270_432, 4, 80, 32, 48 * 1024) == (2, 160, 7968)
    assert O.compute_params(1000, 8, 4, 32, 48 * 1024) == (1, 4, 256)
    assert O.compute_params(85_623, 8, 80, 32, 48 * 1024) == (1, 80, 1088)
    with pytest.raises(ValueError, match="infeasible"):
        O.compute_params(100, 8, 1, 32, 128)


def test_randrange_matches_cpython_recipe():
    # the MT19937 recipe the C oracle and the product restate
    import random
    for seed in (0, 1, 3, 12345):
        r = random.Random(seed)
        got = [r.randrange(m) for m in (2, 3, 7, 100, 1000, 65537, 1 << 20)]
        r2 = random.Random(seed)
        again = [r2.randrange(m) for m in (2, 3, 7, 100, 1000, 65537, 1 << 20)]
        assert got == again
