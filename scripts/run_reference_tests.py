#!/usr/bin/env python3
"""Run the reference's OWN test suite against the B200 drop-in.

    python scripts/run_reference_tests.py --stage      # copy the suite (dev container)
    python scripts/run_reference_tests.py [files ...]   # run it (here or on the GPU box)

`--stage` copies /root/reference/pkg/tests (read-only, present only in the
dev container) into tests/_reftests/, which is git-ignored (the suite is not
product source and never enters history) but not gpurun-ignored, so it
travels to the GPU box with the snapshot. Running copies the staged suite to
a temporary directory and runs it with compat/ (the `ehyb` alias of
paper_2204_06666_b200, submodules included) first on sys.path.

Without a GPU the SpMV tests (test_engine.py, most of test_acceptance.py and
the verify/bench CLI tests) fail by design: the drop-in has no CPU fallback.
"""

import os
import shutil
import subprocess
import sys
import tempfile

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
REF_TESTS = "/root/reference/pkg/tests"
STAGED = os.path.join(ROOT, "tests", "_reftests")
ALL_FILES = ["test_acceptance.py", "test_cli.py", "test_engine.py", "test_format.py",
             "test_matrix_io.py", "test_partition.py"]


def stage() -> int:
    if not os.path.isdir(REF_TESTS):
        print(f"{REF_TESTS} not present", file=sys.stderr)
        return 2
    os.makedirs(STAGED, exist_ok=True)
    for f in sorted(os.listdir(REF_TESTS)):
        if f.endswith(".py"):
            shutil.copy(os.path.join(REF_TESTS, f), STAGED)
    print(f"staged {len(os.listdir(STAGED))} files in {STAGED}")
    return 0


def source_dir() -> str | None:
    for d in (STAGED, REF_TESTS):
        if os.path.isfile(os.path.join(d, "helpers.py")):
            return d
    return None


def run(files, extra=(), junit=None) -> int:
    src = source_dir()
    if src is None:
        print("reference test suite not available (run --stage in the dev container)",
              file=sys.stderr)
        return 2
    files = list(files) or ALL_FILES
    tmp = tempfile.mkdtemp(prefix="ehyb_reftests_")
    for f in os.listdir(src):
        if f.endswith(".py"):
            shutil.copy(os.path.join(src, f), tmp)
    env = dict(os.environ)
    env["PYTHONPATH"] = os.pathsep.join([os.path.join(ROOT, "compat"), tmp,
                                         env.get("PYTHONPATH", "")])
    cmd = [sys.executable, "-m", "pytest", "-q", "-p", "no:cacheprovider", "-W", "ignore",
           *extra, *files]
    if junit:
        cmd.append(f"--junitxml={junit}")
    rc = subprocess.call(cmd, cwd=tmp, env=env)
    shutil.rmtree(tmp, ignore_errors=True)
    return rc


def main(argv):
    if argv and argv[0] == "--stage":
        return stage()
    return run(argv)


if __name__ == "__main__":
    sys.exit(main(sys.argv[1:]))
