"""The .ehyb container (matrix_io.py:276-474 format): bytes identical to the
reference writer's, bit-exact round trip, and the reference's integrity
errors (magic, version, tag, CRC, truncation)."""

import hashlib
import io
import json
import os

import numpy as np
import pytest

import paper_2204_06666_b200 as E
from golden_data import GOLDEN, small_case, small_meta
from pipeline_util import product_pipeline


def built(name):
    meta = small_meta()[name]
    g = small_case(name)
    *_, e = product_pipeline(meta["n"], g["rows"], g["cols"], g["vals"], meta["tau"],
                             meta["profile"], assignment=g.get("assignment_in"),
                             n_parts_hint=meta["n_parts_hint"], rebalance=meta["rebalance"])
    return e


def blob_of(e):
    buf = io.BytesIO()
    E.write_ehyb_container(e, buf)
    return buf.getvalue()


@pytest.mark.parametrize("name", sorted(small_meta()))
def test_bytes_match_reference_writer(name):
    with open(os.path.join(GOLDEN, "container_digests.json")) as fh:
        want = json.load(fh)[name]
    e = built(name)
    blob = blob_of(e)
    assert hashlib.sha256(blob).hexdigest() == want
    back = E.read_ehyb_container(blob)
    for f in ("val_ell", "col_ell", "position_ell", "width_ell", "ell_row_widths", "val_er",
              "col_er", "position_er", "width_er", "er_row_widths", "part_boundary"):
        assert np.array_equal(getattr(back, f), getattr(e, f)), f
        assert getattr(back, f).dtype == getattr(e, f).dtype, f
    assert np.array_equal(back.plan.reorder_table, e.plan.reorder_table)
    assert back.plan.reorder_table.dtype == np.int32  # the reference reads i32 tables


def test_integrity_errors(tmp_path):
    blob = blob_of(built("poisson32"))
    with pytest.raises(E.ContainerError, match="magic"):
        E.read_ehyb_container(b"XXXX" + blob[4:])
    with pytest.raises(E.ContainerError, match="version"):
        E.read_ehyb_container(blob[:4] + (2).to_bytes(4, "little") + blob[8:])
    with pytest.raises(E.ContainerError, match="precision tag"):
        E.read_ehyb_container(blob[:8] + (5).to_bytes(4, "little") + blob[12:])
    with pytest.raises(E.ContainerError, match="truncated"):
        E.read_ehyb_container(blob[:10])
    flipped = bytearray(blob)
    flipped[200] ^= 0x40
    with pytest.raises(E.ContainerError, match="checksum"):
        E.read_ehyb_container(bytes(flipped))
    rng = np.random.default_rng(0)
    for cut in rng.integers(12, len(blob) - 1, size=20):
        with pytest.raises(E.ContainerError):
            E.read_ehyb_container(blob[: int(cut)])
    p = tmp_path / "m.ehyb"
    E.write_ehyb_container(built("poisson32"), str(p))
    assert E.read_ehyb_container(str(p)).nnz == built("poisson32").nnz
