"""Device residency of an assembled EhybMatrix on a B200.

`DeviceMatrix` owns an `ehyb_dev` handle (include/ehyb_b200.h): the matrix is
uploaded once (plus the derived per-partition ER layout) and every SpMV is a
single fused kernel launch on the caller's stream. torch is used only as the
device-memory / stream plumbing for tensor arguments.
"""

from __future__ import annotations

import ctypes as C
import threading
import weakref

import numpy as np

from . import _lib as L
from .format import EhybMatrix, ReorderPlan, host_view

_cache_lock = threading.Lock()
_by_matrix: "weakref.WeakKeyDictionary[EhybMatrix, dict]" = weakref.WeakKeyDictionary()
_by_plan: "weakref.WeakKeyDictionary[ReorderPlan, DeviceMatrix]" = weakref.WeakKeyDictionary()


def _torch():
    import torch

    return torch


def default_device() -> int:
    torch = _torch()
    if not torch.cuda.is_available():
        raise RuntimeError("EHYB SpMV needs a CUDA device (B200, sm_100a); none is visible. "
                           "There is no CPU fallback.")
    return torch.cuda.current_device()


def _stream_ptr(stream, device: int):
    torch = _torch()
    if stream is None:
        stream = torch.cuda.current_stream(device)
    return C.c_void_p(stream.cuda_stream)


class DeviceMatrix:
    """An EhybMatrix resident on one GPU."""

    def __init__(self, e: EhybMatrix, device: int | None = None):
        self.device = default_device() if device is None else int(device)
        self.e = weakref.proxy(e)
        self.tau = e.params.tau
        self.dimension = e.dimension
        self.padded = e.padded_dimension
        self.dtype = np.float32 if self.tau == 4 else np.float64
        hv, keep = host_view(e)
        h = L.vp()
        L.call("ehyb_dev_create", C.byref(hv), self.device, C.byref(h))
        del keep
        self._h = h
        self._finalizer = weakref.finalize(self, L.lib().ehyb_dev_destroy, h)

    @property
    def handle(self):
        return self._h

    def close(self) -> None:
        self._finalizer()

    def tune(self, *, prefetch_ell: int | None = None, prefetch_er: bool | None = None,
             threads: int | None = None, timing=False, er_warps: int | None = None,
             claim_ahead: int | None = None, phases: int | None = None) -> None:
        """Launch knobs (include/ehyb_b200.h ehyb_dev_tune). `timing`: a CUDA
        int64 tensor of n_ctas*8 zeroed entries to record per-CTA stamps, None to
        stop recording, False (default) to leave it unchanged."""
        if prefetch_ell is not None:
            L.call("ehyb_dev_tune", self._h, L.TUNE_PREFETCH_ELL, int(prefetch_ell))
        if prefetch_er is not None:
            L.call("ehyb_dev_tune", self._h, L.TUNE_PREFETCH_ER, int(bool(prefetch_er)))
        if threads is not None:
            L.call("ehyb_dev_tune", self._h, L.TUNE_THREADS, int(threads))
        if er_warps is not None:
            L.call("ehyb_dev_tune", self._h, L.TUNE_ER_WARPS, int(er_warps))
        if claim_ahead is not None:
            L.call("ehyb_dev_tune", self._h, L.TUNE_CLAIM_AHEAD, int(claim_ahead))
        if phases is not None:  # measurement only: 1 = ELL alone, 2 = ER alone, 0 = both
            L.call("ehyb_dev_tune", self._h, L.TUNE_PHASES, int(phases))
        if timing is not False:
            ptr = 0 if timing is None else int(timing.data_ptr())
            L.call("ehyb_dev_tune", self._h, L.TUNE_TIMING, ptr)

    def info(self) -> dict:
        out = L.DevInfo()
        L.call("ehyb_dev_info_get", self._h, C.byref(out))
        return {f: getattr(out, f) for f, _ in L.DevInfo._fields_}

    @property
    def torch_dtype(self):
        torch = _torch()
        return torch.float32 if self.tau == 4 else torch.float64

    def _check_tensor(self, t, length: int, what: str):
        torch = _torch()
        if not isinstance(t, torch.Tensor) or not t.is_cuda:
            raise TypeError(f"{what} must be a CUDA torch.Tensor")
        if t.dim() != 1 or t.numel() != length:
            raise ValueError(f"length mismatch: {what} must have {length} entries")
        if t.dtype != self.torch_dtype:
            raise TypeError(f"{what} must be {self.torch_dtype}")
        if not t.is_contiguous():
            raise ValueError(f"{what} must be contiguous")
        if t.device.index != self.device:
            raise ValueError(f"{what} lives on cuda:{t.device.index}, matrix on cuda:{self.device}")

    def spmv(self, x, y=None, *, fma: bool = False, exact: bool = False, stream=None):
        """y = A x in reordered space, device tensors, stream-ordered.
        Arithmetic (include/ehyb_b200.h EHYB_MODE_*): default = the reference's
        rounding for every slice row (bitwise), rows wider than the long-row
        threshold summed in fixed segments (1e-12 / 1e-5); exact=True = every
        row bitwise (long rows as one serial chain); fma=True = fused."""
        torch = _torch()
        self._check_tensor(x, self.padded, "x")
        if y is None:
            y = torch.empty(self.padded, dtype=self.torch_dtype, device=x.device)
        else:
            self._check_tensor(y, self.padded, "y")
        L.call("ehyb_dev_spmv", self._h, C.c_void_p(x.data_ptr()), C.c_void_p(y.data_ptr()),
               L.mode(fma, exact), _stream_ptr(stream, self.device))
        return y

    def spmv_user(self, x, y=None, *, fma: bool = False, exact: bool = False, stream=None):
        """Original-order y = A x on device tensors (permute, spmv, unpermute)."""
        torch = _torch()
        self._check_tensor(x, self.dimension, "x")
        if y is None:
            y = torch.empty(self.dimension, dtype=self.torch_dtype, device=x.device)
        else:
            self._check_tensor(y, self.dimension, "y")
        L.call("ehyb_dev_spmv_user", self._h, C.c_void_p(x.data_ptr()), C.c_void_p(y.data_ptr()),
               L.mode(fma, exact), _stream_ptr(stream, self.device))
        return y

    def permute(self, x, out=None, stream=None):
        torch = _torch()
        self._check_tensor(x, self.dimension, "x")
        if out is None:
            out = torch.empty(self.padded, dtype=self.torch_dtype, device=x.device)
        L.call("ehyb_dev_permute", self._h, C.c_void_p(x.data_ptr()), C.c_void_p(out.data_ptr()),
               _stream_ptr(stream, self.device))
        return out

    def unpermute(self, y, out=None, stream=None):
        torch = _torch()
        self._check_tensor(y, self.padded, "y")
        if out is None:
            out = torch.empty(self.dimension, dtype=self.torch_dtype, device=y.device)
        L.call("ehyb_dev_unpermute", self._h, C.c_void_p(y.data_ptr()), C.c_void_p(out.data_ptr()),
               _stream_ptr(stream, self.device))
        return out

    def spmv_host(self, x: np.ndarray, *, user_order: bool, fma: bool = False,
                  exact: bool = False, out: np.ndarray | None = None) -> np.ndarray:
        """Host arrays in, host array out: H2D copy, fused kernel, D2H copy,
        synchronised (the path a numpy caller of the reference API takes)."""
        length = self.dimension if user_order else self.padded
        x = np.ascontiguousarray(x, dtype=self.dtype)
        if x.ndim != 1 or x.size != length:
            raise ValueError("length mismatch: x must have "
                             + ("the matrix dimension" if user_order else "padded_dimension entries"))
        y = np.empty(length, dtype=self.dtype) if out is None else out
        L.call("ehyb_dev_spmv_host", self._h, C.c_void_p(x.ctypes.data), C.c_void_p(y.ctypes.data),
               1 if user_order else 0, L.mode(fma, exact),
               _stream_ptr(None, self.device))
        return y

    def spmv_host_many(self, xs, *, user_order: bool, fma: bool = False, exact: bool = False,
                       out=None):
        """Independent products of several host vectors (ehyb_dev_spmv_host_many):
        each is copied in, multiplied and copied out like `spmv_host`, but the
        copy-in of the next vector and the copy-out of the previous one overlap
        the current product. `xs`: a sequence of 1-D arrays or a 2-D array (one
        vector per row); `out`: matching output arrays (allocated if None).
        Pinned (page-locked) host arrays give the full PCIe rate."""
        length = self.dimension if user_order else self.padded
        xs = [xs[i] for i in range(len(xs))]
        for i, x in enumerate(xs):
            if not (isinstance(x, np.ndarray) and x.dtype == self.dtype and x.ndim == 1
                    and x.flags.c_contiguous):
                x = np.ascontiguousarray(x, dtype=self.dtype)
                xs[i] = x
            if x.ndim != 1 or x.size != length:
                raise ValueError("length mismatch: x must have "
                                 + ("the matrix dimension" if user_order
                                    else "padded_dimension entries"))
        if out is None:
            out = [np.empty(length, dtype=self.dtype) for _ in xs]
        ys = [out[i] for i in range(len(out))]
        if len(ys) != len(xs):
            raise ValueError("length mismatch: one output per input vector")
        for y in ys:
            if not (isinstance(y, np.ndarray) and y.dtype == self.dtype and y.ndim == 1
                    and y.size == length and y.flags.c_contiguous and y.flags.writeable):
                raise ValueError(f"length mismatch: outputs must be writable contiguous "
                                 f"{np.dtype(self.dtype).name} arrays of {length} entries")
        k = len(xs)
        xp = (C.c_void_p * max(k, 1))(*[x.ctypes.data for x in xs])
        yp = (C.c_void_p * max(k, 1))(*[y.ctypes.data for y in ys])
        L.call("ehyb_dev_spmv_host_many", self._h, xp, yp, k, 1 if user_order else 0,
               L.mode(fma, exact), _stream_ptr(None, self.device))
        return out


def device_matrix(e: EhybMatrix, device: int | None = None) -> DeviceMatrix:
    """The cached DeviceMatrix of `e` on `device` (uploaded on first use)."""
    dev = default_device() if device is None else int(device)
    with _cache_lock:
        per = _by_matrix.get(e)
        if per is None:
            per = {}
            _by_matrix[e] = per
        dm = per.get(dev)
        if dm is None:
            dm = DeviceMatrix(e, dev)
            per[dev] = dm
            _by_plan[e.plan] = dm
    return dm


def permute_tensor(x, plan: ReorderPlan):
    dm = _by_plan.get(plan)
    if dm is None:
        raise ValueError("permute_vector on a CUDA tensor needs the EhybMatrix of this plan "
                         "on the device first (device_matrix(e))")
    return dm.permute(x)


def unpermute_tensor(y, plan: ReorderPlan):
    dm = _by_plan.get(plan)
    if dm is None:
        raise ValueError("unpermute_vector on a CUDA tensor needs the EhybMatrix of this plan "
                         "on the device first (device_matrix(e))")
    return dm.unpermute(y)


class DeviceCsr:
    """cuSPARSE CSR comparator (cusparseSpMV) with the same upload-once shape."""

    def __init__(self, n_rows, n_cols, row_ptr, col_idx, values, tau: int = 8,
                 device: int | None = None):
        self.device = default_device() if device is None else int(device)
        self.tau = tau
        self.n_rows, self.n_cols = int(n_rows), int(n_cols)
        rp = L.c_array(row_ptr, np.int64)
        ci = L.c_array(col_idx, np.int64)
        va = L.c_array(values, np.float64)
        h = L.vp()
        L.call("ehyb_csr_create", self.n_rows, self.n_cols, int(va.size), L.ptr(rp, L.i64p),
               L.ptr(ci, L.i64p), L.ptr(va, L.f64p), tau, self.device, C.byref(h))
        self._h = h
        self._finalizer = weakref.finalize(self, L.lib().ehyb_csr_destroy, h)

    def spmv(self, x, y, alg: int = 1, stream=None):
        L.call("ehyb_csr_spmv", self._h, C.c_void_p(x.data_ptr()), C.c_void_p(y.data_ptr()),
               int(alg), _stream_ptr(stream, self.device))
        return y
