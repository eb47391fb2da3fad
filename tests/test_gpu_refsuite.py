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
BY_DESIGN = {"test_criterion_2_benchmark_sigma0", "test_criterion_3_rate_prediction",
             "test_criterion_4_acceleration_ordering", "test_criterion_7_misestimation"}
# One more reference test compares two evaluations of the same residual to
# 1e-9 RELATIVE at a residual of ~5e-12 (test_solvers.py:407-410: the host's
# real-space ||Gamma_1 J|| of the returned flux against the last history
# record).  The device records the residual by Parseval in Fourier space
# (deviations), so the two differ by FFT roundoff
# (~1e-16 absolute, ~1e-5 of 5e-12) with either sign.  It may pass or fail;
# test_returned_flux_residual_matches_history below checks the same pair of
# numbers to the parity protocol's residual tolerance instead.
ROUNDOFF = {"test_converged_solution_residual_small"}


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
    # (node ids are relative to a rootdir the files are not under: compare test names)
    failed = {m.split("::")[-1] for m in re.findall(r"FAILED (\S+)", out)}
    summary = [ln for ln in out.splitlines() if re.search(r"\d+ (passed|failed)", ln)]
    assert failed - ROUNDOFF == BY_DESIGN, f"failures {sorted(failed)}\n{out[-3000:]}"
    m = re.search(r"(\d+) passed", summary[-1] if summary else "")
    assert m and int(m.group(1)) >= 100, summary


def test_returned_flux_residual_matches_history():
    """The pair of numbers reference test_solvers.py:407-410 compares -- the
    reference's own equilibrium_residual of the returned J (host, real space)
    and the last recorded residual (device, Parseval) -- agree to the parity
    protocol's residual tolerance (tests/parity.py: 1e-4 relative plus the
    1e-14 roundoff floor)."""
    if not os.path.isdir(os.path.join(REF, "fftcond")):
        pytest.skip("reference install (baseline/_ref) absent")
    code = (
        "import fftcond, ref_seam\n"
        "from fftcond.solvers import equilibrium_residual, solve_basic, SolverConfig, SchemeKind\n"
        "from fftcond.geometry import build_square_array\n"
        "ref_seam.install(fftcond)\n"
        "r = solve_basic(build_square_array(32, 0.5), SolverConfig(scheme=SchemeKind.BASIC, sigma1=2.0, tol=1e-11))\n"
        "print('RES', repr(equilibrium_residual(r.J_field)), repr(r.history.residuals()[-1]))\n")
    env = dict(os.environ)
    env["PYTHONPATH"] = os.pathsep.join([REF, os.path.join(REPO, "tests"), env.get("PYTHONPATH", "")])
    p = subprocess.run([sys.executable, "-c", code], capture_output=True, text=True, env=env, timeout=600)
    m = re.search(r"RES (\S+) (\S+)", p.stdout)
    assert m, p.stdout + p.stderr
    host, dev = float(m.group(1)), float(m.group(2))
    assert abs(host - dev) <= 1e-4 * dev + 1e-14, (host, dev)
