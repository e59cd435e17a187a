"""The reference's OWN test modules, unmodified, run against this repository's GPU path
(VERDICT r1 "next" #8).

tools/stage_reference_tests.sh copies /root/reference/pkg/tests/{test_cur,test_linalg,
test_quat}.py and their helpers next to the installed reference (baseline/_ref/tests_ref,
git-ignored, travels to the GPU box).  They run in a subprocess whose `qcur` package is the
import shim tests/ref_shim/qcur: every `from qcur.cur import qmcur` resolves to
paper_2402_19147_b200 (the C ABI underneath), nothing of the reference's implementation is
importable there.  Skipped when the staged copy is absent.
"""
import os
import subprocess
import sys

import pytest

pytestmark = pytest.mark.gpu

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
STAGED = os.path.join(ROOT, "baseline", "_ref", "tests_ref")
SHIM = os.path.join(ROOT, "tests", "ref_shim")


def run_reference_module(name: str):
    path = os.path.join(STAGED, name)
    if not os.path.exists(path):
        pytest.skip(f"reference tests not staged ({path}); run tools/stage_reference_tests.sh")
    env = dict(os.environ)
    env["PYTHONPATH"] = os.pathsep.join([SHIM, ROOT])
    env["PYTHONDONTWRITEBYTECODE"] = "1"
    out = subprocess.run([sys.executable, "-m", "pytest", path, "-q", "-p", "no:cacheprovider", "-rf",
                          "--rootdir", STAGED, "-o", "addopts="],
                         cwd=STAGED, env=env, capture_output=True, text=True, timeout=1800)
    tail = "\n".join(out.stdout.strip().splitlines()[-40:])
    print(tail)
    # the shim must have served the imports: the reference implementation is not on the path
    assert "baseline/_ref/qcur" not in out.stdout + out.stderr
    return out.returncode, tail


def test_reference_test_cur_on_gpu():
    rc, tail = run_reference_module("test_cur.py")
    assert rc == 0, tail


def test_reference_test_linalg_on_gpu():
    rc, tail = run_reference_module("test_linalg.py")
    assert rc == 0, tail


def test_reference_test_quat_on_gpu():
    rc, tail = run_reference_module("test_quat.py")
    assert rc == 0, tail
