"""Shared helpers for golden fixtures: array digests and the parity-array list.

A digest is sha256 over ``dtype.str | shape | raw little-endian bytes``,
truncated to 24 hex chars, so a digest match pins dtype, length and every
byte of the array.
"""

from __future__ import annotations

import hashlib

import numpy as np

# arrays of the parity object (SURVEY.md §8a "Parity object"), in a fixed order
PARITY_ARRAYS = (
    "assignment", "part_sizes",
    "inner_counts", "outer_counts", "row_order", "er_row_order",
    "reorder_table", "inverse_table", "arrange_table", "y_idx_er",
    "part_boundary", "position_ell", "width_ell", "ell_row_widths", "col_ell", "val_ell",
    "position_er", "width_er", "er_row_widths", "col_er", "val_er",
)

GRAPH_ARRAYS = ("adj_ptr", "adj")


def digest(a) -> str:
    a = np.ascontiguousarray(np.asarray(a))
    if a.dtype.byteorder == ">":
        a = a.astype(a.dtype.newbyteorder("<"))
    h = hashlib.sha256()
    h.update(f"{a.dtype.str}|{a.shape}|".encode())
    h.update(a.tobytes())
    return h.hexdigest()[:24]


def collect(parts, cls, plan, e, graph=None) -> dict:
    """Name -> array for every parity array of one pipeline run (works for
    the reference package, the oracle and the product: same field names)."""
    out = {
        "assignment": parts.assignment,
        "part_sizes": parts.part_sizes,
        "inner_counts": cls.inner_counts,
        "outer_counts": cls.outer_counts,
        "row_order": cls.row_order,
        "er_row_order": cls.er_row_order,
        "reorder_table": plan.reorder_table,
        "inverse_table": plan.inverse_table,
        "arrange_table": plan.arrange_table,
        "y_idx_er": plan.y_idx_er,
        "part_boundary": e.part_boundary,
        "position_ell": e.position_ell,
        "width_ell": e.width_ell,
        "ell_row_widths": e.ell_row_widths,
        "col_ell": e.col_ell,
        "val_ell": e.val_ell,
        "position_er": e.position_er,
        "width_er": e.width_er,
        "er_row_widths": e.er_row_widths,
        "col_er": e.col_er,
        "val_er": e.val_er,
    }
    if graph is not None:
        out["adj_ptr"] = graph.adj_ptr
        out["adj"] = graph.adj
    return out


def digests(arrays: dict) -> dict:
    return {k: digest(v) for k, v in arrays.items()}
