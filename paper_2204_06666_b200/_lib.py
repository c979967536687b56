"""ctypes binding of libehyb_b200.so (include/ehyb_b200.h).

The library is required: there is no CPU or Python fallback for any entry
point. Import of this module succeeds without the library (so the package
can be inspected); the first call raises ImportError if it was not built.
"""

from __future__ import annotations

import ctypes as C
import os
import threading
import weakref

import numpy as np

PKG = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.path.join(PKG, "libehyb_b200.so")

EINVAL, ENOMEM, ECUDA = 1, 2, 3
MODE_STRICT, MODE_FMA, MODE_DEFAULT = 0, 1, 2


def mode(fma: bool = False, exact: bool = False) -> int:
    """include/ehyb_b200.h EHYB_MODE_*: fma -> FMA; exact -> STRICT (every row
    bitwise, long rows as one serial chain); else DEFAULT (bitwise except
    rows wider than the long-row threshold, summed in fixed segments)."""
    if fma:
        return MODE_FMA
    return MODE_STRICT if exact else MODE_DEFAULT
TUNE_PREFETCH_ELL, TUNE_PREFETCH_ER, TUNE_THREADS, TUNE_TIMING, TUNE_ER_WARPS = 1, 2, 3, 4, 5
TUNE_CLAIM_AHEAD = 6
TUNE_PHASES = 7

i32p = C.POINTER(C.c_int32)
i64p = C.POINTER(C.c_int64)
u16p = C.POINTER(C.c_uint16)
u32p = C.POINTER(C.c_uint32)
f64p = C.POINTER(C.c_double)
vp = C.c_void_p


class HostMatrix(C.Structure):
    """ehyb_host_matrix (include/ehyb_b200.h)."""

    _fields_ = [
        ("dimension", C.c_int64), ("padded_dimension", C.c_int64),
        ("plan_padded_dimension", C.c_int64), ("k", C.c_int64), ("n_parts", C.c_int64),
        ("vec_cache_size", C.c_int64), ("warp_size", C.c_int64), ("tau", C.c_int64),
        ("n_er_rows", C.c_int64),
        ("reorder", i64p), ("n_reorder", C.c_int64),
        ("inverse", i64p), ("n_inverse", C.c_int64),
        ("y_idx_er", i64p), ("n_y_idx_er", C.c_int64),
        ("part_boundary", i32p), ("n_part_boundary", C.c_int64),
        ("position_ell", i32p), ("n_position_ell", C.c_int64),
        ("width_ell", i32p), ("n_width_ell", C.c_int64),
        ("ell_row_widths", i32p), ("n_ell_row_widths", C.c_int64),
        ("col_ell", u16p), ("n_col_ell", C.c_int64),
        ("val_ell", vp), ("slots_ell", C.c_int64),
        ("position_er", i32p), ("n_position_er", C.c_int64),
        ("width_er", i32p), ("n_width_er", C.c_int64),
        ("er_row_widths", i32p), ("n_er_row_widths", C.c_int64),
        ("col_er", u32p), ("n_col_er", C.c_int64),
        ("val_er", vp), ("slots_er", C.c_int64),
    ]


class DevInfo(C.Structure):
    _fields_ = [
        ("device_bytes", C.c_int64), ("er_slices", C.c_int64), ("er_slots", C.c_int64),
        ("window_bytes", C.c_int64), ("window_in_smem", C.c_int32),
        ("threads_per_cta", C.c_int32), ("ctas", C.c_int32), ("sm_count", C.c_int32),
        ("pool_slices", C.c_int64), ("er_buf_slices", C.c_int32), ("smem_bytes", C.c_int32),
        ("long_rows", C.c_int64), ("ring_bytes", C.c_int64), ("work_units", C.c_int64),
        ("split", C.c_int32), ("reserved", C.c_int32),
    ]


class ShardPlan(C.Structure):
    _fields_ = [("p0", C.c_int64), ("p1", C.c_int64), ("n_halo", C.c_int64),
                ("halo_cols", i64p)]


# name -> (restype, argtypes)
_PROTOS = {
    "ehyb_last_error": (C.c_char_p, []),
    "ehyb_abi_version": (C.c_int, []),
    "ehyb_free": (None, [vp]),
    "ehyb_num_threads": (C.c_int, []),
    "ehyb_compute_params": (C.c_int, [C.c_int64, C.c_int32, C.c_int64, C.c_int64, C.c_int64,
                                      i64p, i64p, i64p]),
    "ehyb_build_graph": (C.c_int, [C.c_int64, C.c_int64, i64p, i64p, i64p,
                                   C.POINTER(i32p), i64p]),
    "ehyb_partition_graph": (C.c_int, [C.c_int64, i64p, i32p, C.c_int64, C.c_int64, C.c_int64,
                                       i64p, i64p]),
    "ehyb_rebalance_partition": (C.c_int, [C.c_int64, i64p, i32p, C.c_int64, C.c_int64, i64p,
                                           i64p, i64p]),
    "ehyb_classify_rows": (C.c_int, [C.c_int64, C.c_int64, i64p, i64p, i64p, C.c_int64, i64p,
                                     i64p, i64p, C.POINTER(i64p), i64p]),
    "ehyb_build_reorder_plan": (C.c_int, [C.c_int64, C.c_int64, C.c_int64, i64p, i64p, i64p, i64p,
                                          C.c_int64, i64p, i64p, i64p, i64p]),
    "ehyb_assemble": (C.c_int, [C.c_int64, C.c_int64, i64p, i64p, f64p, i64p, i64p, i64p,
                                C.c_int64, C.c_int64, C.c_int64, C.c_int64, C.c_int32,
                                i32p, i32p, i32p, i32p, i32p, i32p, i32p,
                                C.POINTER(vp), C.POINTER(u16p), i64p, C.POINTER(vp),
                                C.POINTER(u32p), i64p]),
    "ehyb_gprep_create": (C.c_int, [C.c_int64, C.c_int64, i64p, i64p, f64p, C.c_int,
                                    C.POINTER(vp)]),
    "ehyb_gprep_destroy": (C.c_int, [vp]),
    "ehyb_gprep_build_graph": (C.c_int, [vp, i64p, C.POINTER(i32p), i64p]),
    "ehyb_gprep_assemble": (C.c_int, [vp, i64p, C.c_int64, C.c_int64, C.c_int64, C.c_int32,
                                      i64p, i64p, i64p, C.POINTER(i64p), i64p,
                                      i64p, i64p, i64p, C.POINTER(i64p),
                                      i32p, i32p, i32p, i32p, C.POINTER(i32p), C.POINTER(i32p),
                                      C.POINTER(i32p), C.POINTER(vp), C.POINTER(u16p), i64p,
                                      C.POINTER(vp), C.POINTER(u32p), i64p]),
    "ehyb_check": (C.c_int, [C.POINTER(HostMatrix)]),
    "ehyb_dev_create": (C.c_int, [C.POINTER(HostMatrix), C.c_int, C.POINTER(vp)]),
    "ehyb_dev_create_shard": (C.c_int, [C.POINTER(HostMatrix), C.POINTER(ShardPlan), C.c_int,
                                        C.POINTER(vp)]),
    "ehyb_dev_destroy": (C.c_int, [vp]),
    "ehyb_dev_info_get": (C.c_int, [vp, C.POINTER(DevInfo)]),
    "ehyb_dev_tune": (C.c_int, [vp, C.c_int, C.c_int64]),
    "ehyb_dev_spmv": (C.c_int, [vp, vp, vp, C.c_int, vp]),
    "ehyb_dev_spmv_ell": (C.c_int, [vp, vp, vp, C.c_int, vp]),
    "ehyb_dev_spmv_er": (C.c_int, [vp, vp, vp, C.c_int, vp]),
    "ehyb_dev_permute": (C.c_int, [vp, vp, vp, vp]),
    "ehyb_dev_unpermute": (C.c_int, [vp, vp, vp, vp]),
    "ehyb_dev_spmv_user": (C.c_int, [vp, vp, vp, C.c_int, vp]),
    "ehyb_dev_spmv_host": (C.c_int, [vp, vp, vp, C.c_int, C.c_int, vp]),
    "ehyb_dev_spmv_host_many": (C.c_int, [vp, C.POINTER(C.c_void_p), C.POINTER(C.c_void_p),
                                          C.c_int64, C.c_int, C.c_int, vp]),
    "ehyb_dev_p2p_alloc": (C.c_int, [vp, C.POINTER(C.c_void_p), C.POINTER(C.c_void_p)]),
    "ehyb_ipc_handle": (C.c_int, [vp, vp]),
    "ehyb_ipc_open": (C.c_int, [vp, C.c_int, C.POINTER(C.c_void_p)]),
    "ehyb_ipc_close": (C.c_int, [vp]),
    "ehyb_dev_p2p_setup": (C.c_int, [vp, C.c_int32, C.c_int32, C.POINTER(C.c_void_p),
                                     C.POINTER(C.c_void_p), vp, vp, C.c_int64]),
    "ehyb_dev_spmv_p2p": (C.c_int, [vp, vp, C.c_int, vp]),
    "ehyb_dev_gather": (C.c_int, [vp, vp, C.c_int64, vp, C.c_int32, vp]),
    "ehyb_dev_dot": (C.c_int, [vp, vp, C.c_int64, C.c_int32, vp, vp]),
    "ehyb_dev_cg_xr": (C.c_int, [vp, vp, vp, vp, vp, vp, C.c_int64, C.c_int32, vp, vp]),
    "ehyb_dev_cg_p": (C.c_int, [vp, vp, vp, vp, C.c_int64, C.c_int32, vp]),
    "ehyb_dev_dot2": (C.c_int, [vp, vp, vp, vp, C.c_int64, C.c_int32, vp, vp]),
    "ehyb_dev_cgcg_step": (C.c_int, [vp, vp, vp, vp, vp, vp, C.c_int, C.c_int64, C.c_int32, vp]),
    "ehyb_dev_axpy":(C.c_int, [vp, C.c_double, vp, vp, C.c_int64, C.c_int32, vp]),
    "ehyb_csr_create": (C.c_int, [C.c_int64, C.c_int64, C.c_int64, i64p, i64p, f64p, C.c_int32,
                                  C.c_int, C.POINTER(vp)]),
    "ehyb_csr_spmv": (C.c_int, [vp, vp, vp, C.c_int, vp]),
    "ehyb_csr_destroy": (C.c_int, [vp]),
}

_lock = threading.Lock()
_lib = None


def lib():
    """The loaded library (raises ImportError when it was not built)."""
    global _lib
    if _lib is not None:
        return _lib
    with _lock:
        if _lib is None:
            if not os.path.exists(LIB_PATH):
                raise ImportError(
                    f"EHYB native library missing ({LIB_PATH}); build it with "
                    "`python -c 'import __graft_entry__ as g; g.build()'` "
                    "(nvcc, sm_100a). There is no CPU fallback.")
            handle = C.CDLL(LIB_PATH)
            for name, (res, args) in _PROTOS.items():
                fn = getattr(handle, name)
                fn.restype = res
                fn.argtypes = args
            _lib = handle
    return _lib


def exported_symbols():
    return list(_PROTOS)


def check(rc: int) -> None:
    if rc == 0:
        return
    msg = lib().ehyb_last_error().decode("utf-8", "replace")
    if rc == EINVAL:
        raise ValueError(msg)
    if rc == ENOMEM:
        raise MemoryError(msg)
    raise RuntimeError(msg)


def call(name: str, *args) -> None:
    check(getattr(lib(), name)(*args))


# ---------------------------------------------------------------- arrays
def ptr(a: np.ndarray, ctype):
    return a.ctypes.data_as(ctype)


def c_array(a, dtype) -> np.ndarray:
    return np.ascontiguousarray(np.asarray(a), dtype=dtype)


def adopt(p, count: int, dtype) -> np.ndarray:
    """Wrap a library-allocated buffer as a numpy array that frees it with
    ehyb_free when the last view dies (zero copy)."""
    dtype = np.dtype(dtype)
    addr = C.cast(p, C.c_void_p).value
    if count == 0 or not addr:
        if addr:
            lib().ehyb_free(addr)
        return np.zeros(0, dtype=dtype)
    buf = (C.c_char * (count * dtype.itemsize)).from_address(addr)
    arr = np.frombuffer(buf, dtype=dtype, count=count)
    weakref.finalize(buf, lib().ehyb_free, addr)
    return arr
