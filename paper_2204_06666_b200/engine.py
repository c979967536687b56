"""SpMV execution (reference engine.py): the EHYB product on a B200 and the
CSR reference product (reference summation order) on the GPU.

`spmv_ehyb` / `spmv_ehyb_user` keep the reference signatures and return
types: numpy in -> numpy out (one H2D copy, one fused kernel, one D2H copy),
CUDA torch tensors in -> CUDA tensors out (zero copy, stream-ordered). With
the default strict arithmetic y is bitwise identical to the reference's
simulated engine for every worker count and schedule (engine.py:1-11).
"""

from __future__ import annotations

from dataclasses import dataclass

import numpy as np

from .format import EhybMatrix
from .matrix_io import CsrMatrix

SCHEDULING_MODES = ("static", "stealing")


@dataclass(frozen=True)
class ExecutionConfig:
    """Reference engine.py:27-40. worker_count / scheduling are validated and
    reported but do not change results (as in the reference); on the GPU the
    schedule is one CTA per partition with in-CTA slice stealing. Extensions:
    by default every row whose ELL/ER width is at most the long-row threshold
    (128 entries) is computed with the reference's rounding (bitwise); wider
    rows (heavy-tailed hubs) are summed in fixed 4096-entry segments, a
    deterministic reassociation within 1e-12 (fp64) / 1e-5 (fp32) of the
    serial sum. `exact=True` keeps those rows as one serial chain too (bitwise
    everywhere, latency-bound on hub rows); `fma=True` fuses multiply and add
    everywhere (within the same tolerances)."""

    worker_count: int = 1
    scheduling: str = "static"
    record_stats: bool = True
    fma: bool = False
    exact: bool = False

    def __post_init__(self):
        if self.worker_count < 1:
            raise ValueError("worker_count must be >= 1")
        if self.scheduling not in SCHEDULING_MODES:
            raise ValueError(f"scheduling must be one of {SCHEDULING_MODES}")


@dataclass(eq=False)
class ExecStats:
    """engine.py:43-53."""

    cached_loads: int
    uncached_loads: int
    flops: int
    bytes_touched_model: int
    slices_per_block: np.ndarray
    er_slices_per_worker: np.ndarray


def _metadata_bytes(e: EhybMatrix) -> int:
    return int(e.position_ell.nbytes + e.width_ell.nbytes + e.part_boundary.nbytes
               + e.position_er.nbytes + e.width_er.nbytes + e.plan.y_idx_er.size * 4)


def traffic_model(e: EhybMatrix, tau: int | None = None) -> int:
    """Reporting byte model (engine.py:83-105): slots_ell*(tau+2) +
    slots_er*(tau+4) + metadata + n*tau (x) + nnz_er*tau (ER x) + n*tau (y)."""
    t = e.params.tau if tau is None else tau
    return int(e.val_ell.size * (t + 2) + e.val_er.size * (t + 4) + _metadata_bytes(e)
               + e.dimension * t + e.nnz_er * t + e.dimension * t)


def min_bytes(e: EhybMatrix) -> int:
    """BASELINE minimum-bytes model: nnz_ell*(tau+2) +
    nnz_er*(tau+4) + n*tau (x once) + n*tau (y once)."""
    t = e.params.tau
    return int(e.nnz_ell * (t + 2) + e.nnz_er * (t + 4) + 2 * e.dimension * t)


def exec_stats(e: EhybMatrix, cfg: ExecutionConfig) -> ExecStats:
    """Counters of engine.py:208-215, computed on the host."""
    n_er_slices = int(e.width_er.size)
    w = cfg.worker_count
    claims = np.array([len(range(i, n_er_slices, w)) for i in range(w)], dtype=np.int64)
    return ExecStats(
        cached_loads=e.nnz_ell,
        uncached_loads=e.nnz_er,
        flops=2 * e.nnz,
        bytes_touched_model=traffic_model(e) if cfg.record_stats else 0,
        slices_per_block=np.full(e.n_parts, e.params.vec_cache_size // e.params.warp_size,
                                 dtype=np.int64),
        er_slices_per_worker=claims,
    )


def _is_torch(x) -> bool:
    return type(x).__module__.startswith("torch")


def spmv_ehyb(e: EhybMatrix, x_reordered, cfg: ExecutionConfig = ExecutionConfig()):
    """y_reordered = A_reordered x_reordered on the GPU (engine.py:108-216).

    x_reordered has padded_dimension entries; computation runs at the stored
    precision (x is cast like engine.py:121). Returns (y, ExecStats).
    """
    from .device import device_matrix

    if _is_torch(x_reordered):
        x = x_reordered
        if x.dim() != 1 or x.numel() != e.padded_dimension:
            raise ValueError("length mismatch: x must have padded_dimension entries")
        dm = device_matrix(e, x.device.index)
        if x.dtype != dm.torch_dtype:
            x = x.to(dm.torch_dtype)
        y = dm.spmv(x.contiguous(), fma=cfg.fma, exact=cfg.exact)
        return y, exec_stats(e, cfg)
    x = np.asarray(x_reordered)
    if x.ndim != 1 or x.size != e.padded_dimension:
        raise ValueError("length mismatch: x must have padded_dimension entries")
    y = device_matrix(e).spmv_host(x, user_order=False, fma=cfg.fma, exact=cfg.exact)
    return y, exec_stats(e, cfg)


def spmv_ehyb_user(e: EhybMatrix, x, cfg: ExecutionConfig = ExecutionConfig()):
    """Original-order product (engine.py:219-227): permute, multiply,
    unpermute — all on the device; result dtype is the stored precision."""
    from .device import device_matrix

    if _is_torch(x):
        if x.dim() != 1 or x.numel() != e.dimension:
            raise ValueError("length mismatch: vector does not match the plan dimension")
        dm = device_matrix(e, x.device.index)
        if x.dtype != dm.torch_dtype:
            x = x.to(dm.torch_dtype)
        return dm.spmv_user(x.contiguous(), fma=cfg.fma, exact=cfg.exact)
    x = np.asarray(x)
    if x.ndim != 1 or x.size != e.dimension:
        raise ValueError("length mismatch: vector does not match the plan dimension")
    return device_matrix(e).spmv_host(x, user_order=True, fma=cfg.fma, exact=cfg.exact)


def spmv_csr(m: CsrMatrix, x) -> np.ndarray:
    """CSR y = A x in float64 (engine.py:56-69) on the GPU, bitwise the
    reference oracle: fp64 products v[j]*x[c[j]] summed per non-empty row in
    np.add.reduceat's order (first product, then numpy's pairwise sum of the
    rest), one thread per row (`csr_ref_kernel`); empty rows are 0.0. The
    cuSPARSE comparator is `DeviceCsr.spmv(..., alg=1|2)`."""
    from .device import DeviceCsr, _torch

    x = np.asarray(x)
    if x.ndim != 1 or x.size != m.n_cols:
        raise ValueError("length mismatch: x must have n_cols entries")
    if m.nnz == 0:
        return np.zeros(m.n_rows, dtype=np.float64)
    torch = _torch()
    dc = DeviceCsr(m.n_rows, m.n_cols, m.row_ptr, m.col_idx, m.values, tau=8)
    xt = torch.from_numpy(np.ascontiguousarray(x.astype(np.float64))).to(f"cuda:{dc.device}")
    yt = torch.empty(m.n_rows, dtype=torch.float64, device=xt.device)
    dc.spmv(xt, yt, alg=0)
    return yt.cpu().numpy()
