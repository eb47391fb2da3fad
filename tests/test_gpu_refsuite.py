"""Drop-in proof from the reference's side: the reference's OWN test files
(test_solvers.py, test_acceptance.py, test_analysis.py, test_cli.py) run with
its solver seam ``_solve_h`` / ``_solve_aug`` (solvers.py:280, :366) replaced
by the INTEGRATION.md ctypes binding over ``fftc_solve_host``
(tests/ref_seam.py).  Everything must pass except the four acceptance
checks that fail by design in the reference's own record
(pkg/test_output.txt:397-401: criteria 2, 3, 4 and 7, the insulating point
sigma1 = 0).

Needs the unmodified reference installed under baseline/_ref and its test
files under baseline/_ref_tests (git-ignored copies made in the dev
container: pip install --target baseline/_ref, cp -r pkg/tests); skipped
where they are absent."""

from __future__ import annotations

import os
import re
import subprocess
import sys

import pytest

pytestmark = pytest.mark.gpu

REPO = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
REF = os.path.join(REPO, "baseline", "_ref")
REF_TESTS = os.path.join(REPO, "baseline", "_ref_tests")
FILES = ["test_solvers.py", "test_acceptance.py", "test_analysis.py", "test_cli.py"]
BY_DESIGN = {"test_acceptance.py::test_criterion_2_benchmark_sigma0", "test_acceptance.py::test_criterion_3_rate_prediction",
             "test_acceptance.py::test_criterion_4_acceleration_ordering",
             "test_acceptance.py::test_criterion_7_misestimation"}


def test_reference_suite_through_the_b200_seam(tmp_path):
    if not (os.path.isdir(os.path.join(REF, "fftcond")) and all(
            os.path.exists(os.path.join(REF_TESTS, f)) for f in FILES)):
        pytest.skip("reference install (baseline/_ref) or its tests (baseline/_ref_tests) absent")
    env = dict(os.environ)
    env["PYTHONPATH"] = os.pathsep.join([REF, os.path.join(REPO, "tests"), env.get("PYTHONPATH", "")])
    env["PYTHONDONTWRITEBYTECODE"] = "1"
    cmd = [sys.executable, "-m", "pytest", "-p", "no:cacheprovider", "-p", "ref_seam_plugin", "-q", "-rf",
           "--tb=no", "--rootdir", str(tmp_path), "-o", "addopts="] + [os.path.join(REF_TESTS, f) for f in FILES]
    p = subprocess.run(cmd, capture_output=True, text=True, env=env, cwd=str(tmp_path), timeout=1500)
    out = p.stdout + p.stderr
    failed = {m.split("/")[-1] for m in re.findall(r"FAILED (\S+)", out)}
    summary = [ln for ln in out.splitlines() if re.search(r"\d+ (passed|failed)", ln)]
    assert failed == BY_DESIGN, f"failures {sorted(failed)}\n{out[-3000:]}"
    m = re.search(r"(\d+) passed", summary[-1] if summary else "")
    assert m and int(m.group(1)) >= 100, summary
