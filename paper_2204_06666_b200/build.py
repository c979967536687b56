"""Build libehyb_b200.so in-tree with nvcc for sm_100a (no JIT, no torch
extension machinery): host preprocessing (C++17 + OpenMP) and the CUDA
kernels go into one shared library that the ctypes shim loads."""

from __future__ import annotations

import os
import shutil
import subprocess
import sys

PKG = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(PKG)
CSRC = os.path.join(PKG, "csrc")
LIB = os.path.join(PKG, "libehyb_b200.so")

SOURCES = ["prep_common.cpp", "prep.cpp", "device.cu", "prep_gpu.cu"]
HEADERS = ["ehyb_common.h", "kernels.cuh", os.path.join("..", "..", "include", "ehyb_b200.h")]

ARCH = ["-gencode", "arch=compute_100a,code=sm_100a"]


def nvcc() -> str:
    for cand in (shutil.which("nvcc"), "/usr/local/cuda/bin/nvcc"):
        if cand and os.path.exists(cand):
            return cand
    raise RuntimeError("nvcc not found: the EHYB library needs the CUDA 12.9 toolkit")


def _stale(target: str, deps) -> bool:
    if not os.path.exists(target):
        return True
    t = os.path.getmtime(target)
    return any(os.path.getmtime(d) > t for d in deps)


STAMP = LIB + ".flags"  # the dev flags the library was built with ("" = the product build)


def _built_flags() -> str | None:
    try:
        with open(STAMP) as fh:
            return fh.read()
    except OSError:
        return None


def build(force: bool = False, verbose: bool = False) -> str:
    deps = [os.path.join(CSRC, f) for f in SOURCES + HEADERS] + [__file__]
    flags = os.environ.get("EHYB_NVCC_FLAGS", "")
    if flags:
        force = True
    # a library left by a dev experiment (EHYB_NVCC_FLAGS, e.g. a one-variant
    # build) is never taken for the product build
    if _built_flags() != flags:
        force = True
    if not force and not _stale(LIB, deps):
        return LIB
    cmd = [
        nvcc(), *ARCH, "-O3", "-lineinfo", "-std=c++17", "-shared",
        "-Xcompiler", "-fPIC,-fopenmp,-O3,-fvisibility=hidden",
        "-Xptxas", "-v" if verbose else "-O3",
        "-I", os.path.join(ROOT, "include"),
        *os.environ.get("EHYB_NVCC_FLAGS", "").split(),  # dev experiments (-D knobs)
        *[os.path.join(CSRC, f) for f in SOURCES],
        "-o", LIB + ".tmp",
        "-lcusparse", "-lgomp",
    ]
    proc = subprocess.run(cmd, capture_output=True, text=True)
    if proc.returncode != 0:
        sys.stderr.write(proc.stdout + proc.stderr)
        raise RuntimeError("nvcc failed building libehyb_b200.so")
    if verbose:
        sys.stderr.write(proc.stderr)
    os.replace(LIB + ".tmp", LIB)
    with open(STAMP, "w") as fh:
        fh.write(flags)
    return LIB


if __name__ == "__main__":
    print(build(force="--force" in sys.argv, verbose="-v" in sys.argv))
