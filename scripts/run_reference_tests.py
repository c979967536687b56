#!/usr/bin/env python3
"""Run the reference's OWN test files against the B200 drop-in.

Copies /root/reference/pkg/tests (read-only, dev container only) to a
temporary directory OUTSIDE the repo and runs them with compat/ (the `ehyb`
import alias of paper_2204_06666_b200) first on sys.path. Nothing of the
reference is written into the repo.

    python scripts/run_reference_tests.py [test_format.py test_partition.py ...]

Without a GPU the SpMV tests (test_engine.py) cannot run: the drop-in has no
CPU fallback by design.
"""

import os
import shutil
import subprocess
import sys
import tempfile

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
REF_TESTS = "/root/reference/pkg/tests"


def main(argv):
    files = argv or ["test_format.py", "test_partition.py"]
    tmp = tempfile.mkdtemp(prefix="ehyb_reftests_")
    for f in ["conftest.py", "helpers.py", *files]:
        shutil.copy(os.path.join(REF_TESTS, f), tmp)
    env = dict(os.environ)
    env["PYTHONPATH"] = os.pathsep.join([os.path.join(ROOT, "compat"), tmp,
                                         env.get("PYTHONPATH", "")])
    cmd = [sys.executable, "-m", "pytest", "-q", "-p", "no:cacheprovider", *files]
    rc = subprocess.call(cmd, cwd=tmp, env=env)
    shutil.rmtree(tmp, ignore_errors=True)
    return rc


if __name__ == "__main__":
    sys.exit(main(sys.argv[1:]))
