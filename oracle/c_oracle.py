"""ORACLE — test / CPU-baseline infrastructure only. NOT part of the product.

ctypes wrapper around oracle/ehyb_oracle.c (the C restatement of the
reference engine.py:108-216) and oracle/ehyb_prep_oracle.c (the C
restatement of the reference preprocessing, partition.py:77-204 and
format.py:123-409), built with gcc into oracle/_build/.
"""

from __future__ import annotations

import ctypes as C
import os
import subprocess

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
SRCS = [os.path.join(HERE, "ehyb_oracle.c"), os.path.join(HERE, "ehyb_prep_oracle.c")]
LIB = os.path.join(HERE, "_build", "libehyb_oracle.so")

_lib = None


def build(force: bool = False) -> str:
    if not force and os.path.exists(LIB) and all(
            os.path.getmtime(LIB) >= os.path.getmtime(s) for s in SRCS):
        return LIB
    os.makedirs(os.path.dirname(LIB), exist_ok=True)
    cmd = ["gcc", "-O3", "-std=c11", "-fopenmp", "-ffp-contract=off", "-fno-fast-math",
           "-shared", "-fPIC", *SRCS, "-o", LIB + ".tmp"]
    subprocess.run(cmd, check=True)
    os.replace(LIB + ".tmp", LIB)
    return LIB


def lib():
    global _lib
    if _lib is None:
        build()
        h = C.CDLL(LIB)
        vp = C.c_void_p
        for name in ("oracle_spmv_ehyb_f64", "oracle_spmv_ehyb_f32"):
            fn = getattr(h, name)
            fn.restype = C.c_int
            fn.argtypes = [C.c_int64, C.c_int64, C.c_int64, vp, vp, vp, vp, C.c_int64, vp, vp,
                           vp, vp, vp, vp, vp, C.c_int, C.c_int64, C.c_int64,
                           C.c_int64, C.c_int64]
        h.oracle_max_threads.restype = C.c_int
        _lib = h
    return _lib


def max_threads() -> int:
    return int(lib().oracle_max_threads())


class Prepared:
    """Contiguous copies of the arrays the C engine reads (prepare once,
    time many)."""

    def __init__(self, e):
        p = e.params
        if p.warp_size > 32:
            raise ValueError("C oracle supports slice heights <= 32")
        self.dt = np.float32 if p.tau == 4 else np.float64
        self.n_parts, self.vec, self.warp = p.n_parts, p.vec_cache_size, p.warp_size
        self.padded = e.padded_dimension
        self.n_er = e.plan.n_er_rows
        c = np.ascontiguousarray
        self.arrs = [
            c(e.val_ell, self.dt), c(e.col_ell, np.uint16), c(e.position_ell, np.int32),
            c(e.width_ell, np.int32), c(e.val_er, self.dt), c(e.col_er, np.uint32),
            c(e.position_er, np.int32), c(e.width_er, np.int32), c(e.plan.y_idx_er, np.int64),
        ]

    @property
    def n_er_slices(self) -> int:
        return -(-self.n_er // self.warp) if self.n_er else 0

    def spmv(self, x_reordered, threads: int | None = None, out=None, parts=None,
             er_slices=None) -> np.ndarray:
        """Full product by default; `parts` / `er_slices` = (lo, hi) ranges
        restrict it to a bounded sample (CPU-baseline timing)."""
        x = np.ascontiguousarray(x_reordered, dtype=self.dt)
        if x.size != self.padded:
            raise ValueError("length mismatch")
        y = np.empty(self.padded, self.dt) if out is None else out
        a = [arr.ctypes.data for arr in self.arrs]
        fn = lib().oracle_spmv_ehyb_f32 if self.dt == np.float32 else lib().oracle_spmv_ehyb_f64
        rc = fn(self.n_parts, self.vec, self.warp, a[0], a[1], a[2], a[3], self.n_er, a[4], a[5],
                a[6], a[7], a[8], x.ctypes.data, y.ctypes.data,
                int(threads or max_threads()), *(parts or (0, self.n_parts)),
                *(er_slices or (0, self.n_er_slices)))
        if rc:
            raise RuntimeError("oracle spmv failed")
        return y


def spmv_ehyb(e, x_reordered, threads: int | None = None) -> np.ndarray:
    return Prepared(e).spmv(x_reordered, threads)
