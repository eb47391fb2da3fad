"""GPU: the public operator surface (paper_2001_08289_b200.spectral, the
reference's spectral_ops.py:96-278 and solvers.py:147-204 names) against the
live reference's outputs (tests/golden/ops.*), 3-D against the oracle, and the
reference selftest (selftest.py:89-205) run on the B200 operators.

Tolerance: the reductions are fixed-order device trees, not math.fsum, and
the pointwise kernels may contract to FMA, so values agree to ~1e-15
relative; the bar is 1e-12 (the reference selftest's own threshold)."""

from __future__ import annotations

import json
import os

import numpy as np
import pytest

from golden_io import GOLDEN
from oracle import fftcond_oracle as O

pytestmark = pytest.mark.gpu

META = json.load(open(os.path.join(GOLDEN, "ops.json")))
ARR = np.load(os.path.join(GOLDEN, "ops.npz"))
TOL = 1e-12


def _c(v):
    return complex(*v)


def _rel(a, b):
    a, b = np.asarray(a), np.asarray(b)
    return float(np.max(np.abs(a - b))) / max(float(np.max(np.abs(b))), 1e-300)


def _fields(case):
    import paper_2001_08289_b200 as fb

    p = case["name"] + "/"
    pm = fb.PhaseMap(ARR[p + "chi"])
    vf, vg = fb.VectorField(ARR[p + "f"]), fb.VectorField(ARR[p + "g"])
    F = fb.AugmentedField(*(fb.VectorField(ARR[p + f"F{k}"]) for k in range(3)))
    H = fb.AugmentedField(*(fb.VectorField(ARR[p + f"H{k}"]) for k in range(3)))
    return p, pm, vf, vg, F, H


@pytest.mark.parametrize("case", META["cases"], ids=[c["name"] for c in META["cases"]])
def test_operators_match_reference(case):
    import paper_2001_08289_b200 as fb
    from paper_2001_08289_b200 import spectral as S

    p, pm, vf, vg, F, H = _fields(case)
    params = fb.solve_p(fb.SpectralInterval(*case["interval"]))
    t, shift, s1 = _c(case["t"]), _c(case["shift"]), _c(case["sigma1"])
    e0 = [_c(z) for z in case["e0"]]
    assert abs(S.inner(vf, vg) - _c(case["inner"])) <= TOL * abs(_c(case["inner"]))
    assert abs(S.norm(vf) - case["norm"]) <= TOL * case["norm"]
    assert _rel(S.gamma0(vf), [_c(z) for z in case["gamma0"]]) <= TOL
    assert abs(S.inner_aug(F, H, pm) - _c(case["inner_aug"])) <= TOL * abs(_c(case["inner_aug"]))
    assert abs(S.norm_aug(F, pm) - case["norm_aug"]) <= TOL * case["norm_aug"]
    assert _rel(S.gamma1(vf).data, ARR[p + "gamma1_f"]) <= TOL
    for tag, out in (("gamma1_aug", S.gamma1_aug(F, pm)), ("chi_aug", S.apply_chi_aug(F, params, pm)),
                     ("local_A", S.apply_local_A(F, t, params, pm)),
                     ("inv_shifted", S.invert_shifted_A(F, t, shift, params, pm))):
        for slot in "QST":
            want = ARR[p + f"{tag}_{slot}"]
            got = getattr(out, slot).data
            if not np.any(want):
                assert not np.any(got), (tag, slot)
            else:
                assert _rel(got, want) <= TOL, (tag, slot)
                assert not np.any(got[:, ~ARR[p + "chi"]]) or slot == "Q", (tag, slot)
    E, J = S.recover_physical_fields(F, t, params, pm)
    assert np.array_equal(E.data, ARR[p + "recover_E"])
    assert _rel(J.data, ARR[p + "recover_J"]) <= TOL
    ss = _c(case["sigma_star"])
    assert abs(S.extract_sigma_star(vf, pm, s1, e0) - ss) <= TOL * abs(ss)
    ssa = _c(case["sigma_star_aug"])
    assert abs(S.extract_sigma_star_aug(F, t, params, pm, e0) - ssa) <= TOL * abs(ssa)
    assert abs(S.equilibrium_residual(vf) - case["eq_residual"]) <= TOL * case["eq_residual"]
    assert abs(S.equilibrium_residual_aug(F, pm) - case["eq_residual_aug"]) <= TOL * case["eq_residual_aug"]


def test_support_and_contract_errors():
    import paper_2001_08289_b200 as fb
    from paper_2001_08289_b200 import spectral as S

    pm = fb.build_square_array(16, 0.5)
    rng = np.random.default_rng(3)
    bad = np.zeros((2, 16, 16), complex)
    bad[0, 0, 0] = 1e-200  # tiny but nonzero, on a phase-2 pixel
    F = fb.AugmentedField(fb.VectorField(rng.standard_normal((2, 16, 16)) + 0j), fb.VectorField(bad),
                          fb.VectorField.zeros(16, 16))
    with pytest.raises(fb.SupportError):
        S.gamma1_aug(F, pm)
    with pytest.raises(fb.ContractError):
        S.equilibrium_residual(fb.VectorField.zeros(16, 16))
    with pytest.raises(fb.ContractError):
        S.extract_sigma_star(fb.VectorField.zeros(16, 16), pm, 2.0, (0.0, 0.0))


def test_3d_operators_match_oracle():
    import paper_2001_08289_b200 as fb
    from paper_2001_08289_b200 import spectral as S

    rng = np.random.default_rng(7)
    shape = (8, 16, 32)
    chi = rng.random(shape) < 0.3
    pm = fb.PhaseMap(chi)

    def rnd():
        return rng.standard_normal((3,) + shape) + 1j * rng.standard_normal((3,) + shape)

    Fa = (rnd(), np.where(chi, rnd(), 0.0), np.where(chi, rnd(), 0.0))
    F = fb.AugmentedField(*(fb.VectorField(x) for x in Fa))
    params = fb.solve_p(fb.SpectralInterval(0.25, 4.0))
    p = (params.p1, params.p2, params.p3)
    t = fb.map_t(50.0, fb.SpectralInterval(0.25, 4.0))
    e0 = (1 / 3 ** 0.5,) * 3
    for got, want in ((S.apply_local_A(F, t, params, pm), O.apply_local_A(Fa, t, p, chi)),
                      (S.invert_shifted_A(F, t, 1.9, params, pm), O.invert_shifted_A(Fa, t, 1.9, p, chi)),
                      (S.gamma1_aug(F, pm), O.gamma1_aug(Fa, chi))):
        for k, slot in enumerate("QST"):
            if np.any(want[k]):
                assert _rel(getattr(got, slot).data, want[k]) <= TOL
            else:
                assert not np.any(getattr(got, slot).data)
    assert abs(S.norm_aug(F, pm) - O.norm_aug(Fa, chi)) <= TOL * O.norm_aug(Fa, chi)
    w = O.extract_sigma_star_aug(Fa, t, p, chi, e0)
    assert abs(S.extract_sigma_star_aug(F, t, params, pm, e0) - w) <= TOL * abs(w)
    w = O.equilibrium_residual_aug(Fa, chi)
    assert abs(S.equilibrium_residual_aug(F, pm) - w) <= TOL * w
    w = O.extract_sigma_star(Fa[0], chi, 50.0, e0)
    assert abs(S.extract_sigma_star(F.Q, pm, 50.0, e0) - w) <= TOL * abs(w)


def test_selftest_on_gpu_operators():
    """The reference's own selftest.py:89-205, its operator names bound to the
    B200 operators: every check passes, same names, thresholds and order as
    the reference's report (needs the reference installed, baseline/_ref)."""
    from paper_2001_08289_b200 import selftest
    from paper_2001_08289_b200.exceptions import BackendError

    try:
        selftest.reference_module()
    except BackendError:
        pytest.skip("reference package not installed (baseline/_ref)")

    res = selftest.run_selftest()
    assert [(r.name, r.threshold) for r in res] == [(r["name"], r["threshold"]) for r in META["selftest"]]
    assert all(r.passed for r in res), selftest.format_report(res)
    ref = {r["name"]: r["measured"] for r in META["selftest"]}
    for r in res[:4]:  # host scalar algebra: identical to the reference
        assert r.measured == ref[r.name]
    assert selftest.format_report(res).endswith("13/13 checks passed\n")


def test_large_reduction_is_deterministic():
    """Repeated reductions of a 2048^2 field are bit identical."""
    import torch

    import paper_2001_08289_b200 as fb
    from paper_2001_08289_b200 import spectral as S

    g = torch.Generator(device="cuda").manual_seed(5)
    t = torch.randn((2, 2048, 2048), dtype=torch.complex128, device="cuda", generator=g)
    f = fb.VectorField.from_device(t)
    vals = [(S.norm(f), tuple(S.gamma0(f)), S.inner(f, f)) for _ in range(3)]
    assert vals[0] == vals[1] == vals[2]
    assert abs(vals[0][0] ** 2 - vals[0][2].real) <= 1e-12 * vals[0][0] ** 2
