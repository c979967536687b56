"""EHYB format: parameters (Eq.1-2), row classification and reorder plan
(Alg.1), sliced-ELL + extra-rows assembly (Alg.2) — reference format.py.

Every pipeline step runs natively (csrc/prep.cpp) and produces arrays
byte-identical to the reference's; dataclasses, field names, dtypes and
error wording are the reference's so this module is a drop-in.
"""

from __future__ import annotations

import ctypes as C
from dataclasses import dataclass

import numpy as np

from . import _lib as L
from .matrix_io import CooMatrix
from .partition import PartitionMap, build_graph, partition_graph, rebalance_partition

MAX_LOCAL_INDEX = 1 << 16  # format.py:21

# format.py:23-27: the paper's fp64 footprint figure, surfaced unresolved
QUOTED_DOUBLE_PRECISION_SAVINGS = 0.133


@dataclass(frozen=True)
class DeviceProfile:
    """Device model: processor count, slice height (warp), shared-memory
    window budget per block (format.py:30-44)."""

    num_processors: int
    warp_size: int = 32
    shm_max: int = 48 * 1024

    def __post_init__(self):
        if self.num_processors < 1:
            raise ValueError("num_processors must be >= 1")
        if self.warp_size < 1:
            raise ValueError("warp_size must be >= 1")
        if self.shm_max <= 0:
            raise ValueError("shm_max must be positive")


# V100-class defaults of the reference (format.py:48)
DEFAULT_PROFILE = DeviceProfile(num_processors=80)

#: B200: 148 SMs, 32-lane slices, 227 KB opt-in shared memory per CTA minus
#: 1 KB kept for the kernel's mbarrier and work counters.
B200_SHM_WINDOW = 232448 - 1024
B200_PROFILE = DeviceProfile(num_processors=148, warp_size=32, shm_max=B200_SHM_WINDOW)


def b200_profile(n_gpus: int = 1) -> DeviceProfile:
    """Profile for a job of `n_gpus` B200s (P = 148 per GPU)."""
    return DeviceProfile(num_processors=148 * n_gpus, warp_size=32, shm_max=B200_SHM_WINDOW)


@dataclass(frozen=True)
class EhybParams:
    """Resolved partition parameters (format.py:51-72)."""

    k: int
    n_parts: int
    vec_cache_size: int
    tau: int
    warp_size: int

    def __post_init__(self):
        if self.tau not in (4, 8):
            raise ValueError("tau must be 4 or 8 bytes per value")
        if self.vec_cache_size > MAX_LOCAL_INDEX:
            raise ValueError("vec_cache_size exceeds the 16-bit local index bound")
        if self.vec_cache_size % self.warp_size:
            raise ValueError("vec_cache_size must be a multiple of warp_size")

    @property
    def value_dtype(self):
        return np.float32 if self.tau == 4 else np.float64


def compute_params(dimension: int, tau: int, profile: DeviceProfile = DEFAULT_PROFILE) -> EhybParams:
    """Eq.1-2: smallest k whose warp-aligned window fits shm (format.py:83-107)."""
    if dimension < 1:
        raise ValueError("dimension must be >= 1")
    if tau not in (4, 8):
        raise ValueError("tau must be 4 or 8")
    k, n_parts, vec = C.c_int64(), C.c_int64(), C.c_int64()
    L.call("ehyb_compute_params", int(dimension), int(tau), profile.num_processors,
           profile.warp_size, profile.shm_max, C.byref(k), C.byref(n_parts), C.byref(vec))
    return EhybParams(k=k.value, n_parts=n_parts.value, vec_cache_size=vec.value, tau=tau,
                      warp_size=profile.warp_size)


@dataclass(eq=False)
class RowClassification:
    """Per-row inner/outer counts and the two orders of Alg.1 (format.py:110-120)."""

    inner_counts: np.ndarray
    outer_counts: np.ndarray
    row_order: np.ndarray
    er_row_order: np.ndarray


def classify_rows(m: CooMatrix, parts: PartitionMap) -> RowClassification:
    """format.py:123-137, native."""
    if not m.is_square or parts.n_vertices != m.n_rows:
        raise ValueError("dimension mismatch between matrix and partition")
    n = m.n_rows
    rows = L.c_array(m.rows, np.int64)
    cols = L.c_array(m.cols, np.int64)
    a = L.c_array(parts.assignment, np.int64)
    inner = np.empty(n, np.int64)
    outer = np.empty(n, np.int64)
    order = np.empty(n, np.int64)
    er = L.i64p()
    n_er = C.c_int64()
    L.call("ehyb_classify_rows", n, rows.size, L.ptr(rows, L.i64p), L.ptr(cols, L.i64p),
           L.ptr(a, L.i64p), parts.n_parts, L.ptr(inner, L.i64p), L.ptr(outer, L.i64p),
           L.ptr(order, L.i64p), C.byref(er), C.byref(n_er))
    return RowClassification(inner_counts=inner, outer_counts=outer, row_order=order,
                             er_row_order=L.adopt(er, n_er.value, np.int64))


@dataclass(eq=False)
class ReorderPlan:
    """Symmetric permutation plus ER bookkeeping (format.py:140-158)."""

    reorder_table: np.ndarray
    inverse_table: np.ndarray
    arrange_table: np.ndarray
    y_idx_er: np.ndarray
    n_er_rows: int
    dimension: int
    padded_dimension: int


def build_reorder_plan(cls: RowClassification, params: EhybParams, parts: PartitionMap) -> ReorderPlan:
    """format.py:161-199, native."""
    n = cls.inner_counts.size
    vec = params.vec_cache_size
    n_parts = parts.n_parts
    if int(parts.part_sizes.max(initial=0)) > vec:
        raise ValueError("a partition exceeds the vector cache capacity")
    padded = n_parts * vec
    a = L.c_array(parts.assignment, np.int64)
    sizes = L.c_array(parts.part_sizes, np.int64)
    order = L.c_array(cls.row_order, np.int64)
    er = L.c_array(cls.er_row_order, np.int64)
    n_er = int(er.size)
    reorder = np.empty(padded, np.int64)
    inverse = np.empty(padded, np.int64)
    arrange = np.empty(n, np.int64)
    y_idx = np.empty(n_er, np.int64)
    L.call("ehyb_build_reorder_plan", n, n_parts, vec, L.ptr(a, L.i64p), L.ptr(sizes, L.i64p),
           L.ptr(order, L.i64p), L.ptr(er, L.i64p), n_er, L.ptr(reorder, L.i64p),
           L.ptr(inverse, L.i64p), L.ptr(arrange, L.i64p), L.ptr(y_idx, L.i64p))
    return ReorderPlan(reorder_table=reorder, inverse_table=inverse, arrange_table=arrange,
                       y_idx_er=y_idx, n_er_rows=n_er, dimension=n, padded_dimension=padded)


@dataclass(eq=False)
class EhybMatrix:
    """Assembled hybrid matrix (format.py:202-248): SELL ELL body with u16
    window-local columns, SELL ER body with u32 global columns."""

    params: EhybParams
    plan: ReorderPlan
    dimension: int
    padded_dimension: int
    val_ell: np.ndarray
    col_ell: np.ndarray
    position_ell: np.ndarray
    width_ell: np.ndarray
    part_boundary: np.ndarray
    ell_row_widths: np.ndarray
    val_er: np.ndarray
    col_er: np.ndarray
    position_er: np.ndarray
    width_er: np.ndarray
    er_row_widths: np.ndarray

    @property
    def y_idx_er(self) -> np.ndarray:
        return self.plan.y_idx_er

    @property
    def n_parts(self) -> int:
        return self.params.n_parts

    @property
    def nnz_ell(self) -> int:
        return int(self.ell_row_widths.sum())

    @property
    def nnz_er(self) -> int:
        return int(self.er_row_widths.sum())

    @property
    def nnz(self) -> int:
        return self.nnz_ell + self.nnz_er

    def host_view(self):
        """(ehyb_host_matrix, keep-alive list) for the C ABI."""
        return host_view(self)

    def check(self) -> None:
        """Structural invariants (format.py:250-299), native; raises ValueError."""
        hv, _keep = host_view(self)
        L.call("ehyb_check", C.byref(hv))


def host_view(e: EhybMatrix):
    p = e.params
    keep = []

    def arr(a, dtype, ctype):
        a = L.c_array(a, dtype)
        keep.append(a)
        return L.ptr(a, ctype), a.size

    vdt = np.float32 if p.tau == 4 else np.float64
    hv = L.HostMatrix()
    hv.dimension = e.dimension
    hv.padded_dimension = e.padded_dimension
    hv.plan_padded_dimension = e.plan.padded_dimension
    hv.k = p.k
    hv.n_parts = p.n_parts
    hv.vec_cache_size = p.vec_cache_size
    hv.warp_size = p.warp_size
    hv.tau = p.tau
    hv.n_er_rows = e.plan.n_er_rows
    hv.reorder, hv.n_reorder = arr(e.plan.reorder_table, np.int64, L.i64p)
    hv.inverse, hv.n_inverse = arr(e.plan.inverse_table, np.int64, L.i64p)
    hv.y_idx_er, hv.n_y_idx_er = arr(e.plan.y_idx_er, np.int64, L.i64p)
    hv.part_boundary, hv.n_part_boundary = arr(e.part_boundary, np.int32, L.i32p)
    hv.position_ell, hv.n_position_ell = arr(e.position_ell, np.int32, L.i32p)
    hv.width_ell, hv.n_width_ell = arr(e.width_ell, np.int32, L.i32p)
    hv.ell_row_widths, hv.n_ell_row_widths = arr(e.ell_row_widths, np.int32, L.i32p)
    hv.col_ell, hv.n_col_ell = arr(e.col_ell, np.uint16, L.u16p)
    v, hv.slots_ell = arr(e.val_ell, vdt, L.vp)
    hv.val_ell = C.cast(v, C.c_void_p)
    hv.position_er, hv.n_position_er = arr(e.position_er, np.int32, L.i32p)
    hv.width_er, hv.n_width_er = arr(e.width_er, np.int32, L.i32p)
    hv.er_row_widths, hv.n_er_row_widths = arr(e.er_row_widths, np.int32, L.i32p)
    hv.col_er, hv.n_col_er = arr(e.col_er, np.uint32, L.u32p)
    v, hv.slots_er = arr(e.val_er, vdt, L.vp)
    hv.val_er = C.cast(v, C.c_void_p)
    return hv, keep


def assemble_ehyb(m: CooMatrix, plan: ReorderPlan, params: EhybParams, parts: PartitionMap) -> EhybMatrix:
    """Alg.2 placement (format.py:302-409), native: inner entries into the
    reordered row's ELL slice at a u16 window offset, outer entries into the
    row's ER slot with a u32 global column; entries of a row ranked by
    ascending original column; padding slots 0.0 / column 0."""
    if not m.is_square or parts.n_vertices != m.n_rows:
        raise ValueError("dimension mismatch between matrix and partition")
    n = m.n_rows
    warp = params.warp_size
    vec = params.vec_cache_size
    padded = plan.padded_dimension
    n_parts = padded // vec
    n_er = plan.n_er_rows
    n_sl = padded // warp
    n_er_sl = -(-n_er // warp) if n_er else 0
    rows = L.c_array(m.rows, np.int64)
    cols = L.c_array(m.cols, np.int64)
    vals = L.c_array(m.values, np.float64)
    a = L.c_array(parts.assignment, np.int64)
    reorder = L.c_array(plan.reorder_table, np.int64)
    arrange = L.c_array(plan.arrange_table, np.int64)
    position_ell = np.empty(n_sl + 1, np.int32)
    width_ell = np.empty(n_sl, np.int32)
    ell_row_widths = np.empty(padded, np.int32)
    part_boundary = np.empty(n_parts + 1, np.int32)
    position_er = np.empty(n_er_sl + 1, np.int32)
    width_er = np.empty(n_er_sl, np.int32)
    er_row_widths = np.empty(n_er, np.int32)
    v_ell, c_ell, v_er, c_er = L.vp(), L.u16p(), L.vp(), L.u32p()
    s_ell, s_er = C.c_int64(), C.c_int64()
    L.call("ehyb_assemble", n, rows.size, L.ptr(rows, L.i64p), L.ptr(cols, L.i64p),
           L.ptr(vals, L.f64p), L.ptr(a, L.i64p), L.ptr(reorder, L.i64p), L.ptr(arrange, L.i64p),
           n_er, warp, vec, n_parts, params.tau, L.ptr(position_ell, L.i32p),
           L.ptr(width_ell, L.i32p), L.ptr(ell_row_widths, L.i32p), L.ptr(part_boundary, L.i32p),
           L.ptr(position_er, L.i32p), L.ptr(width_er, L.i32p), L.ptr(er_row_widths, L.i32p),
           C.byref(v_ell), C.byref(c_ell), C.byref(s_ell), C.byref(v_er), C.byref(c_er),
           C.byref(s_er))
    dt = params.value_dtype
    e = EhybMatrix(
        params=params, plan=plan, dimension=n, padded_dimension=padded,
        val_ell=L.adopt(v_ell, s_ell.value, dt), col_ell=L.adopt(c_ell, s_ell.value, np.uint16),
        position_ell=position_ell, width_ell=width_ell, part_boundary=part_boundary,
        ell_row_widths=ell_row_widths,
        val_er=L.adopt(v_er, s_er.value, dt), col_er=L.adopt(c_er, s_er.value, np.uint32),
        position_er=position_er, width_er=width_er, er_row_widths=er_row_widths,
    )
    e.check()
    return e


def build_ehyb(m: CooMatrix, *, tau: int = 8, profile: DeviceProfile = DEFAULT_PROFILE,
               partition: PartitionMap | None = None, seed: int = 0) -> EhybMatrix:
    """Full preprocessing pipeline (format.py:412-442). A supplied partition is
    widened to n_parts when it declares fewer parts and rebalanced when a
    part exceeds the window capacity."""
    if not m.is_square:
        raise ValueError("matrix must be square")
    params = compute_params(m.n_rows, tau, profile)
    if partition is None:
        g = build_graph(m)
        partition = partition_graph(g, params.n_parts, params.vec_cache_size, seed=seed)
    else:
        if partition.n_parts > params.n_parts:
            raise ValueError(
                f"partition declares {partition.n_parts} parts, device parameters allow {params.n_parts}")
        if partition.n_parts < params.n_parts:
            partition = PartitionMap.from_assignment(partition.assignment, n_parts=params.n_parts)
        if int(partition.part_sizes.max(initial=0)) > params.vec_cache_size:
            partition = rebalance_partition(build_graph(m), partition, params.vec_cache_size)
    cls = classify_rows(m, partition)
    plan = build_reorder_plan(cls, params, partition)
    return assemble_ehyb(m, plan, params, partition)


def _is_torch(x) -> bool:
    return type(x).__module__.startswith("torch")


def permute_vector(x, plan: ReorderPlan):
    """x (original order) -> reordered padded vector, zero padding
    (format.py:445-452). numpy in -> numpy out; a CUDA torch tensor is
    permuted on the device (see device.DeviceMatrix.permute)."""
    if _is_torch(x):
        from .device import permute_tensor
        return permute_tensor(x, plan)
    x = np.asarray(x)
    if x.ndim != 1 or x.size != plan.dimension:
        raise ValueError("length mismatch: vector does not match the plan dimension")
    out = np.zeros(plan.padded_dimension, dtype=x.dtype)
    out[plan.reorder_table[: plan.dimension]] = x
    return out


def unpermute_vector(y, plan: ReorderPlan):
    """Inverse of permute_vector, dropping padding (format.py:455-460)."""
    if _is_torch(y):
        from .device import unpermute_tensor
        return unpermute_tensor(y, plan)
    y = np.asarray(y)
    if y.ndim != 1 or y.size != plan.padded_dimension:
        raise ValueError("length mismatch: vector does not match the padded dimension")
    return np.ascontiguousarray(y[plan.reorder_table[: plan.dimension]])


def ehyb_to_coo(e: EhybMatrix) -> CooMatrix:
    """Original-order COO from the assembled arrays, stored precision
    (format.py:463-498); used for conservation checks."""
    warp = e.params.warp_size
    vec = e.params.vec_cache_size
    inv = np.asarray(e.plan.inverse_table, dtype=np.int64)

    def expand(widths, position):
        w = np.asarray(widths, dtype=np.int64)
        owner = np.repeat(np.arange(w.size, dtype=np.int64), w)
        start = np.cumsum(w) - w
        k = np.arange(owner.size, dtype=np.int64) - np.repeat(start, w)
        return owner, np.asarray(position, np.int64)[owner // warp] + owner % warp + k * warp

    nr, idx = expand(e.ell_row_widths, e.position_ell)
    r1 = inv[nr]
    c1 = inv[e.col_ell[idx].astype(np.int64) + (nr // vec) * vec]
    v1 = e.val_ell[idx]
    slot, idx2 = expand(e.er_row_widths, e.position_er)
    r2 = inv[np.asarray(e.plan.y_idx_er, np.int64)[slot]]
    c2 = inv[e.col_er[idx2].astype(np.int64)]
    v2 = e.val_er[idx2]
    return CooMatrix(e.dimension, e.dimension, np.concatenate([r1, r2]),
                     np.concatenate([c1, c2]), np.concatenate([v1, v2]).astype(np.float64))


@dataclass(frozen=True)
class FootprintStats:
    """Device-resident byte counts (format.py:501-513)."""

    ell_bytes: int
    er_bytes: int
    total_bytes: int
    savings_vs_32bit_cols: float


def footprint_stats(e: EhybMatrix) -> FootprintStats:
    """format.py:516-536: value+column+slice metadata per body, plus the ER
    row map; per-slot saving of 16-bit columns 1 - (tau+2)/(tau+4)."""
    tau = e.params.tau
    ell = e.val_ell.nbytes + e.col_ell.nbytes + e.position_ell.nbytes + e.width_ell.nbytes
    er = (e.val_er.nbytes + e.col_er.nbytes + e.position_er.nbytes + e.width_er.nbytes
          + e.plan.y_idx_er.size * 4)
    return FootprintStats(ell_bytes=int(ell), er_bytes=int(er),
                          total_bytes=int(ell + er + e.part_boundary.nbytes),
                          savings_vs_32bit_cols=1.0 - (tau + 2) / (tau + 4))
