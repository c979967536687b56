"""Preprocessing on the GPU (include/ehyb_b200.h `ehyb_gprep_*`): build_graph
(partition.py:77-98) and classify_rows + build_reorder_plan + assemble_ehyb
(format.py:123-409) as radix-sort / scan / scatter kernels on the B200,
bit-exact with the host path (and so with the reference). The BFS
partitioner in between (partition.py:101-204) is sequential by the
reference's semantics and runs on the host (`partition_graph`).

    e = build_ehyb_gpu(m, tau=8, profile=B200_PROFILE)       # == build_ehyb(m, ...)
"""

from __future__ import annotations

import ctypes as C
import time
import weakref

import numpy as np

from . import _lib as L
from .format import (DEFAULT_PROFILE, DeviceProfile, EhybMatrix, ReorderPlan, RowClassification,
                     compute_params)
from .matrix_io import CooMatrix
from .partition import AdjacencyGraph, PartitionMap, partition_graph, rebalance_partition


class GpuPrep:
    """A COO matrix resident on one GPU, its entries grouped by (row, column,
    entry index) — the order the reference assembles in."""

    def __init__(self, m: CooMatrix, device: int | None = None):
        from .device import default_device

        if not m.is_square:
            raise ValueError("matrix must be square")
        self.device = default_device() if device is None else int(device)
        self.m = m
        rows = L.c_array(m.rows, np.int64)
        cols = L.c_array(m.cols, np.int64)
        vals = L.c_array(m.values, np.float64)
        h = L.vp()
        L.call("ehyb_gprep_create", m.n_rows, rows.size, L.ptr(rows, L.i64p), L.ptr(cols, L.i64p),
               L.ptr(vals, L.f64p), self.device, C.byref(h))
        self._h = h
        self._fin = weakref.finalize(self, L.lib().ehyb_gprep_destroy, h)

    def close(self) -> None:
        self._fin()

    def build_graph(self) -> AdjacencyGraph:
        n = self.m.n_rows
        adj_ptr = np.zeros(n + 1, dtype=np.int64)
        out = L.i32p()
        n_adj = C.c_int64()
        L.call("ehyb_gprep_build_graph", self._h, L.ptr(adj_ptr, L.i64p), C.byref(out),
               C.byref(n_adj))
        return AdjacencyGraph(n_vertices=n, adj_ptr=adj_ptr, adj=L.adopt(out, n_adj.value, np.int32))

    def assemble(self, parts: PartitionMap, params) -> tuple[RowClassification, ReorderPlan,
                                                              EhybMatrix]:
        n = self.m.n_rows
        if parts.n_vertices != n:
            raise ValueError("dimension mismatch between matrix and partition")
        if int(parts.part_sizes.max(initial=0)) > params.vec_cache_size:
            raise ValueError("a partition exceeds the vector cache capacity")
        vec, warp = params.vec_cache_size, params.warp_size
        n_parts = parts.n_parts
        padded = n_parts * vec
        n_sl = padded // warp
        a = L.c_array(parts.assignment, np.int64)
        inner, outer, order = (np.empty(n, np.int64) for _ in range(3))
        reorder, inverse = np.empty(padded, np.int64), np.empty(padded, np.int64)
        arrange = np.empty(n, np.int64)
        position_ell = np.empty(n_sl + 1, np.int32)
        width_ell = np.empty(n_sl, np.int32)
        ell_row_widths = np.empty(padded, np.int32)
        part_boundary = np.empty(n_parts + 1, np.int32)
        er, yidx = L.i64p(), L.i64p()
        pos_er, wid_er, erw = L.i32p(), L.i32p(), L.i32p()
        n_er = C.c_int64()
        v_ell, c_ell, v_er, c_er = L.vp(), L.u16p(), L.vp(), L.u32p()
        s_ell, s_er = C.c_int64(), C.c_int64()
        L.call("ehyb_gprep_assemble", self._h, L.ptr(a, L.i64p), n_parts, vec, warp, params.tau,
               L.ptr(inner, L.i64p), L.ptr(outer, L.i64p), L.ptr(order, L.i64p), C.byref(er),
               C.byref(n_er), L.ptr(reorder, L.i64p), L.ptr(inverse, L.i64p),
               L.ptr(arrange, L.i64p), C.byref(yidx), L.ptr(position_ell, L.i32p),
               L.ptr(width_ell, L.i32p), L.ptr(ell_row_widths, L.i32p),
               L.ptr(part_boundary, L.i32p), C.byref(pos_er), C.byref(wid_er), C.byref(erw),
               C.byref(v_ell), C.byref(c_ell), C.byref(s_ell), C.byref(v_er), C.byref(c_er),
               C.byref(s_er))
        ne = n_er.value
        n_er_sl = -(-ne // warp) if ne else 0
        cls = RowClassification(inner_counts=inner, outer_counts=outer, row_order=order,
                                er_row_order=L.adopt(er, ne, np.int64))
        plan = ReorderPlan(reorder_table=reorder, inverse_table=inverse, arrange_table=arrange,
                           y_idx_er=L.adopt(yidx, ne, np.int64), n_er_rows=ne, dimension=n,
                           padded_dimension=padded)
        dt = params.value_dtype
        e = EhybMatrix(
            params=params, plan=plan, dimension=n, padded_dimension=padded,
            val_ell=L.adopt(v_ell, s_ell.value, dt), col_ell=L.adopt(c_ell, s_ell.value, np.uint16),
            position_ell=position_ell, width_ell=width_ell, part_boundary=part_boundary,
            ell_row_widths=ell_row_widths,
            val_er=L.adopt(v_er, s_er.value, dt), col_er=L.adopt(c_er, s_er.value, np.uint32),
            position_er=L.adopt(pos_er, n_er_sl + 1, np.int32),
            width_er=L.adopt(wid_er, n_er_sl, np.int32),
            er_row_widths=L.adopt(erw, ne, np.int32),
        )
        e.check()
        return cls, plan, e


def build_ehyb_gpu(m: CooMatrix, *, tau: int = 8, profile: DeviceProfile = DEFAULT_PROFILE,
                   partition: PartitionMap | None = None, seed: int = 0, device: int | None = None,
                   timings: dict | None = None) -> EhybMatrix:
    """build_ehyb (format.py:412-442) with build_graph and the classify /
    reorder / assemble steps on the GPU; the same EhybMatrix, byte for byte.
    `timings` (optional dict) receives upload_s, build_graph_s,
    partition_graph_s and reorder_assemble_s."""
    if not m.is_square:
        raise ValueError("matrix must be square")
    params = compute_params(m.n_rows, tau, profile)
    t0 = time.perf_counter()
    gp = GpuPrep(m, device)
    t1 = time.perf_counter()
    try:
        tg = t1
        if partition is None:
            g = gp.build_graph()
            tg = time.perf_counter()
            partition = partition_graph(g, params.n_parts, params.vec_cache_size, seed=seed)
            del g
        else:
            if partition.n_parts > params.n_parts:
                raise ValueError(f"partition declares {partition.n_parts} parts, device "
                                 f"parameters allow {params.n_parts}")
            if partition.n_parts < params.n_parts:
                partition = PartitionMap.from_assignment(partition.assignment,
                                                         n_parts=params.n_parts)
            if int(partition.part_sizes.max(initial=0)) > params.vec_cache_size:
                partition = rebalance_partition(gp.build_graph(), partition,
                                                params.vec_cache_size)
            tg = time.perf_counter()
        t2 = time.perf_counter()
        _, _, e = gp.assemble(partition, params)
        t3 = time.perf_counter()
    finally:
        gp.close()
    if timings is not None:
        timings.update(upload_s=t1 - t0, build_graph_s=tg - t1, partition_graph_s=t2 - tg,
                       reorder_assemble_s=t3 - t2)
    return e
