"""CPU: the C-ABI library loads and exports every symbol include/*.h
declares; the ctypes structs match the header layout.  No compute calls."""

from __future__ import annotations

import ctypes as C
import os
import re

REPO = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
HEADER = os.path.join(REPO, "include", "fftcond_b200.h")


def _declared_functions():
    text = open(HEADER).read()
    text = re.sub(r"/\*.*?\*/", "", text, flags=re.S)
    return sorted(set(re.findall(r"\b(fftc_[a-z0-9_]+)\s*\(", text)))


def test_library_exports_every_declared_symbol():
    from paper_2001_08289_b200 import native

    L = native.lib()
    names = _declared_functions()
    assert "fftc_solve" in names and "fftc_gamma1" in names
    for name in names:
        assert hasattr(L, name), name
    assert set(names) == set(native.EXPORTS)


def test_version_and_lengths():
    from paper_2001_08289_b200 import native

    L = native.lib()
    assert L.fftc_version() >= 100
    for n in (2, 4, 64, 256, 1024, 2048, 4096):
        assert L.fftc_supported_length(n) == 1 and L.fftc_fused_length(n) == 1
    for n in (6, 12, 100, 8192, 3000):  # even: the general path (cuFFT)
        assert L.fftc_supported_length(n) == 1 and L.fftc_fused_length(n) == 0
    for n in (0, 1, 3, 7, 101):
        assert L.fftc_supported_length(n) == 0 and L.fftc_fused_length(n) == 0
    assert L.fftc_last_error() is not None


def test_struct_layout_matches_header():
    from paper_2001_08289_b200 import native

    # sizes implied by the header: all fields naturally aligned
    assert C.sizeof(native.Problem) == 4 + 4 + 3 * 8 + 8
    assert C.sizeof(native.Params) == 4 + 4 + 2 * 8 * 6 + 3 * 2 * 8 + 8 + 8 + 8
    assert C.sizeof(native.Result) == 4 + 4 + 8 + 16 + 48 + 48 + 8 + 8
    assert C.sizeof(native.KStat) == 32 + 8 + 8


def test_bad_arguments_are_errors_not_crashes():
    from paper_2001_08289_b200 import native

    L = native.lib()
    p = native.Problem()
    p.d = 4  # invalid dimension: rejected before any CUDA call
    par = native.Params()
    res = native.Result()
    rc = L.fftc_solve(C.byref(p), C.byref(par), None, 0, None, None, None, C.byref(res), None)
    assert rc != 0
    assert b"d must be 2 or 3" in L.fftc_last_error()
    p.d = 2
    p.n[0], p.n[1], p.n[2] = 7, 8, 1  # odd axis: the reference's PhaseMap rejects it too
    rc = L.fftc_solve(C.byref(p), C.byref(par), None, 0, None, None, None, C.byref(res), None)
    assert rc == 3


def test_reference_seam_binding_structs_and_host_errors():
    """tests/ref_seam.py (the INTEGRATION.md binding): its ctypes structs match
    the library's, and the reference's own validation still raises before any
    device call once the seam is installed (solvers.py:221-240)."""
    import pytest

    import ref_seam
    from paper_2001_08289_b200 import native

    for a, b in ((ref_seam._Problem, native.Problem), (ref_seam._Params, native.Params),
                 (ref_seam._Result, native.Result)):
        assert C.sizeof(a) == C.sizeof(b) and [f[0] for f in a._fields_] == [f[0] for f in b._fields_]
    assert hasattr(ref_seam.lib(), "fftc_solve_host")
    try:
        from paper_2001_08289_b200 import selftest

        selftest.reference_module()
        import fftcond
    except Exception:
        pytest.skip("reference package not installed (baseline/_ref)")
    fc = fftcond
    orig = fc.solvers._solve_h, fc.solvers._solve_aug
    try:
        ref_seam.install(fc)
        assert fc.solvers._solve_h is not orig[0]
        cfg = fc.SolverConfig(scheme=fc.SchemeKind.EYRE_MILTON, sigma1=-2.0)
        with pytest.raises(fc.BranchCutError):
            fc.solve(fc.build_square_array(8, 0.5), cfg)
    finally:
        fc.solvers._solve_h, fc.solvers._solve_aug = orig
