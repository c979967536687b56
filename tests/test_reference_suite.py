"""The reference's own 182-test suite (pkg/tests) run against the drop-in
through the `ehyb` alias (compat/ehyb: package + engine/format/partition/
matrix_io/cli submodules).

The suite is staged into tests/_reftests/ by
`python scripts/run_reference_tests.py --stage` in the dev container (it is
git-ignored, travels to the GPU box with the snapshot, and is never read from
/root/reference at run time). Without a GPU only the host-side files can pass
(the drop-in has no CPU fallback), so the whole suite is a `gpu` test; the
host-side files also run in the CPU suite.
"""

import os
import subprocess
import sys

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
SCRIPT = os.path.join(ROOT, "scripts", "run_reference_tests.py")
STAGED = os.path.join(ROOT, "tests", "_reftests")

pytestmark = pytest.mark.skipif(not os.path.isfile(os.path.join(STAGED, "helpers.py")),
                                reason="reference suite not staged (scripts/run_reference_tests.py --stage)")


def _run(*files):
    r = subprocess.run([sys.executable, SCRIPT, *files], capture_output=True, text=True,
                       timeout=1800)
    tail = "\n".join((r.stdout + r.stderr).strip().splitlines()[-25:])
    return r.returncode, tail


def test_reference_host_suite():
    """format / partition / matrix_io: preprocessing, I/O and containers."""
    rc, tail = _run("test_format.py", "test_partition.py", "test_matrix_io.py")
    assert rc == 0, tail


@pytest.mark.gpu
def test_reference_full_suite():
    """All six files, including test_engine.py (scheduling, barrier stress,
    stats), test_acceptance.py and test_cli.py (verify / bench on the GPU)."""
    rc, tail = _run()
    assert rc == 0, tail
    assert " passed" in tail and "failed" not in tail, tail
