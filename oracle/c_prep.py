"""ORACLE — test / CPU-baseline infrastructure only. NOT part of the product.

ctypes wrapper around oracle/ehyb_prep_oracle.c: the reference preprocessing
(build_graph, partition_graph, classify_rows, build_reorder_plan,
assemble_ehyb; partition.py:77-204, format.py:83-409) restated in C. Lets
`bench.py --impl reference` and the tests build the reference's EHYB arrays
without the product library. Returns plain numpy arrays in an object with the
attribute names of the reference's EhybMatrix (what c_oracle.Prepared reads).
"""

from __future__ import annotations

import ctypes as C
from types import SimpleNamespace

import numpy as np

from . import c_oracle

_bound = False


class _Ehyb(C.Structure):
    _fields_ = [(k, C.c_int64) for k in ("n", "padded", "n_parts", "vec", "warp", "tau", "n_er",
                                         "slots_ell", "slots_er")] + [
        (k, C.c_void_p) for k in ("inner_counts", "outer_counts", "row_order", "er_row_order",
                                  "reorder", "inverse", "arrange", "y_idx_er", "ell_row_widths",
                                  "width_ell", "position_ell", "part_boundary", "er_row_widths",
                                  "width_er", "position_er", "val_ell", "col_ell", "val_er",
                                  "col_er")]


def _lib():
    global _bound
    h = c_oracle.lib()
    if not _bound:
        vp, i64 = C.c_void_p, C.c_int64
        h.oracle_build_graph.restype = i64
        h.oracle_build_graph.argtypes = [i64, i64, vp, vp, vp, C.POINTER(C.c_void_p)]
        h.oracle_partition_graph.restype = C.c_int
        h.oracle_partition_graph.argtypes = [i64, vp, vp, i64, i64, i64, vp, vp]
        h.oracle_assemble.restype = C.c_int
        h.oracle_assemble.argtypes = [i64, i64, vp, vp, vp, vp, i64, i64, i64, i64,
                                      C.POINTER(_Ehyb)]
        h.oracle_ehyb_free.argtypes = [C.POINTER(_Ehyb)]
        h.oracle_free.argtypes = [vp]
        _bound = True
    return h


def compute_params(n: int, tau: int, profile) -> SimpleNamespace:
    """format.py:83-107: smallest k whose aligned window fits shm_max."""
    procs, warp, shm = profile
    if warp * tau > shm or warp > 65536:
        raise ValueError("infeasible device profile: a single warp-aligned cache window cannot fit")
    k = 1
    while True:
        n_parts = k * procs
        vec = -(-(-(-n // n_parts)) // warp) * warp
        if vec * tau <= shm and vec <= 65536:
            return SimpleNamespace(k=k, n_parts=n_parts, vec_cache_size=vec, tau=tau,
                                   warp_size=warp)
        k += 1


def build_graph(n: int, rows, cols):
    rows = np.ascontiguousarray(rows, np.int64)
    cols = np.ascontiguousarray(cols, np.int64)
    adj_ptr = np.zeros(n + 1, np.int64)
    p = C.c_void_p()
    cnt = _lib().oracle_build_graph(n, rows.size, rows.ctypes.data, cols.ctypes.data,
                                    adj_ptr.ctypes.data, C.byref(p))
    adj = np.ctypeslib.as_array(C.cast(p, C.POINTER(C.c_int32)), shape=(max(cnt, 1),))[:cnt].copy()
    _lib().oracle_free(p)
    return adj_ptr, adj


def partition_graph(n: int, adj_ptr, adj, n_parts: int, capacity: int, seed: int = 0):
    assignment = np.empty(n, np.int64)
    sizes = np.empty(n_parts, np.int64)
    rc = _lib().oracle_partition_graph(n, adj_ptr.ctypes.data, adj.ctypes.data, n_parts, capacity,
                                       seed, assignment.ctypes.data, sizes.ctypes.data)
    if rc:
        raise ValueError(f"infeasible: {n_parts} parts of capacity {capacity} cannot hold {n} vertices")
    return assignment, sizes


def _take(ptr, ctype, count, dtype):
    if count <= 0:
        return np.zeros(0, dtype)
    return np.ctypeslib.as_array(C.cast(ptr, C.POINTER(ctype)), shape=(count,)).astype(dtype,
                                                                                       copy=True)


def assemble(n: int, rows, cols, vals, assignment, params) -> SimpleNamespace:
    """classify_rows + build_reorder_plan + assemble_ehyb. The result carries
    the reference EhybMatrix attribute names (plan.* for the ReorderPlan)."""
    rows = np.ascontiguousarray(rows, np.int64)
    cols = np.ascontiguousarray(cols, np.int64)
    vals = np.ascontiguousarray(vals, np.float64)
    assignment = np.ascontiguousarray(assignment, np.int64)
    o = _Ehyb()
    rc = _lib().oracle_assemble(n, rows.size, rows.ctypes.data, cols.ctypes.data, vals.ctypes.data,
                                assignment.ctypes.data, params.n_parts, params.vec_cache_size,
                                params.warp_size, params.tau, C.byref(o))
    if rc == 1:
        raise ValueError("a partition exceeds the vector cache capacity")
    if rc:
        raise ValueError("inner entry maps outside its partition cache window" if rc == 2
                         else "slot count exceeds int32 positions")
    try:
        I64, I32 = C.c_int64, C.c_int32
        n_sl, n_ers = o.padded // o.warp, (-(-o.n_er // o.warp) if o.n_er else 0)
        vt = C.c_float if o.tau == 4 else C.c_double
        vd = np.float32 if o.tau == 4 else np.float64
        plan = SimpleNamespace(
            reorder_table=_take(o.reorder, I64, o.padded, np.int64),
            inverse_table=_take(o.inverse, I64, o.padded, np.int64),
            arrange_table=_take(o.arrange, I64, n, np.int64),
            y_idx_er=_take(o.y_idx_er, I64, o.n_er, np.int64),
            n_er_rows=int(o.n_er), dimension=n, padded_dimension=int(o.padded))
        cls = SimpleNamespace(
            inner_counts=_take(o.inner_counts, I64, n, np.int64),
            outer_counts=_take(o.outer_counts, I64, n, np.int64),
            row_order=_take(o.row_order, I64, n, np.int64),
            er_row_order=_take(o.er_row_order, I64, o.n_er, np.int64))
        e = SimpleNamespace(
            params=params, plan=plan, classification=cls, dimension=n,
            padded_dimension=int(o.padded), n_parts=int(o.n_parts),
            val_ell=_take(o.val_ell, vt, o.slots_ell, vd),
            col_ell=_take(o.col_ell, C.c_uint16, o.slots_ell, np.uint16),
            position_ell=_take(o.position_ell, I32, n_sl + 1, np.int32),
            width_ell=_take(o.width_ell, I32, n_sl, np.int32),
            part_boundary=_take(o.part_boundary, I32, o.n_parts + 1, np.int32),
            ell_row_widths=_take(o.ell_row_widths, I32, o.padded, np.int32),
            val_er=_take(o.val_er, vt, o.slots_er, vd),
            col_er=_take(o.col_er, C.c_uint32, o.slots_er, np.uint32),
            position_er=_take(o.position_er, I32, n_ers + 1, np.int32),
            width_er=_take(o.width_er, I32, n_ers, np.int32),
            er_row_widths=_take(o.er_row_widths, I32, o.n_er, np.int32))
        e.nnz_ell = int(e.ell_row_widths.sum(dtype=np.int64))
        e.nnz_er = int(e.er_row_widths.sum(dtype=np.int64))
        e.nnz = e.nnz_ell + e.nnz_er
        return e
    finally:
        _lib().oracle_ehyb_free(C.byref(o))


def build_ehyb(n: int, rows, cols, vals, tau: int, profile, seed: int = 0, timings=None):
    """The reference's default build_ehyb path (format.py:412-442, no external
    partition) on the C restatement."""
    import time

    params = compute_params(n, tau, profile)
    t0 = time.perf_counter()
    adj_ptr, adj = build_graph(n, rows, cols)
    assignment, sizes = partition_graph(n, adj_ptr, adj, params.n_parts, params.vec_cache_size,
                                        seed)
    t1 = time.perf_counter()
    e = assemble(n, rows, cols, vals, assignment, params)
    t2 = time.perf_counter()
    e.assignment, e.part_sizes, e.adj_ptr, e.adj = assignment, sizes, adj_ptr, adj
    if timings is not None:
        timings.update(partition_s=t1 - t0, reorder_assemble_s=t2 - t1)
    return e
