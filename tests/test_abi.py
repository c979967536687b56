"""The C ABI library loads without a GPU and exports every symbol that
include/ehyb_b200.h declares; the ctypes prototypes cover the same set."""

import ctypes
import os
import re
import subprocess

from paper_2204_06666_b200 import _lib as L

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
HEADER = os.path.join(ROOT, "include", "ehyb_b200.h")


def declared():
    text = open(HEADER).read()
    return sorted(set(re.findall(r"EHYB_API\s+[\w\s\*]+?\b(ehyb_\w+)\s*\(", text)))


def test_header_declares_the_boundary():
    names = declared()
    for must in ("ehyb_build_graph", "ehyb_partition_graph", "ehyb_classify_rows",
                 "ehyb_build_reorder_plan", "ehyb_assemble", "ehyb_check", "ehyb_dev_create",
                 "ehyb_dev_spmv", "ehyb_dev_spmv_user", "ehyb_dev_spmv_host", "ehyb_csr_spmv"):
        assert must in names


def test_library_exports_every_declared_symbol():
    lib = L.lib()
    out = subprocess.run(["nm", "-D", "--defined-only", L.LIB_PATH], capture_output=True,
                         text=True, check=True).stdout
    exported = set(re.findall(r"\bT (ehyb_\w+)", out))
    missing = [n for n in declared() if n not in exported]
    assert not missing, missing
    for n in declared():
        assert isinstance(getattr(lib, n), ctypes._CFuncPtr)
    assert sorted(L.exported_symbols()) == declared()
    assert lib.ehyb_abi_version() == 2
    assert lib.ehyb_num_threads() >= 1


def test_error_reporting_through_the_abi():
    import pytest
    import paper_2204_06666_b200 as E

    with pytest.raises(ValueError, match="infeasible device profile"):
        E.compute_params(10, 8, E.DeviceProfile(1, 32, 64))
    assert "infeasible" in L.lib().ehyb_last_error().decode()
