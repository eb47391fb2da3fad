"""CPU: the oracle's restatement of the public operator surface reproduces
the live reference's outputs (tests/golden/ops.*, made by
oracle/gen_golden_ops.py), and the host-side checks of the GPU operator API
raise the reference's exceptions before any device work."""

from __future__ import annotations

import json
import os

import numpy as np
import pytest

from golden_io import GOLDEN
from oracle import fftcond_oracle as O

META = json.load(open(os.path.join(GOLDEN, "ops.json")))
ARR = np.load(os.path.join(GOLDEN, "ops.npz"))


def _c(v):
    return complex(*v)


def _case_inputs(case):
    p = case["name"] + "/"
    chi = ARR[p + "chi"]
    F = tuple(ARR[p + f"F{k}"] for k in range(3))
    H = tuple(ARR[p + f"H{k}"] for k in range(3))
    return p, chi, ARR[p + "f"], ARR[p + "g"], F, H


def _close(a, b, tol=1e-14):
    a, b = np.asarray(a), np.asarray(b)
    scale = max(1.0, float(np.max(np.abs(b))) if b.size else 1.0)
    assert float(np.max(np.abs(a - b))) <= tol * scale


@pytest.mark.parametrize("case", META["cases"], ids=[c["name"] for c in META["cases"]])
def test_oracle_ops_match_reference(case):
    p, chi, f, g, F, H = _case_inputs(case)
    a, b = case["interval"]
    params = O.solve_p(a, b)
    t, shift, s1 = _c(case["t"]), _c(case["shift"]), _c(case["sigma1"])
    e0 = [_c(z) for z in case["e0"]]
    assert O.map_t(s1, a, b) == t
    assert O.inner(f, g) == _c(case["inner"])
    assert O.norm(f) == case["norm"]
    assert np.array_equal(O.gamma0(f), np.array([_c(z) for z in case["gamma0"]]))
    assert O.inner_aug(F, H, chi) == _c(case["inner_aug"])
    assert O.norm_aug(F, chi) == case["norm_aug"]
    _close(O.gamma1(f), ARR[p + "gamma1_f"], 0.0)
    for tag, out in (("gamma1_aug", O.gamma1_aug(F, chi)), ("chi_aug", O.apply_chi_aug(F, params, chi)),
                     ("local_A", O.apply_local_A(F, t, params, chi)),
                     ("inv_shifted", O.invert_shifted_A(F, t, shift, params, chi))):
        for k, slot in enumerate("QST"):
            assert np.array_equal(out[k], ARR[p + f"{tag}_{slot}"]), (tag, slot)
    assert O.extract_sigma_star(f, chi, s1, e0) == _c(case["sigma_star"])
    assert O.extract_sigma_star_aug(F, t, params, chi, e0) == _c(case["sigma_star_aug"])
    assert O.equilibrium_residual(f) == case["eq_residual"]
    assert O.equilibrium_residual_aug(F, chi) == case["eq_residual_aug"]


def test_host_checks_raise_before_device_work():
    import paper_2001_08289_b200 as fb
    from paper_2001_08289_b200 import spectral

    pm = fb.build_square_array(8, 0.5)
    F = fb.AugmentedField.from_mean((1.0, 0.0), 8, 8)
    params = fb.solve_p(fb.SpectralInterval(0.25, 4.0))
    with pytest.raises(fb.DegenerateParamError):
        spectral.invert_shifted_A(F, 2.0, -1.0, params, pm)
    with pytest.raises(fb.DegenerateParamError):
        spectral.invert_shifted_A(F, 2.0 + 1.0j, -2.0 - 1.0j, params, pm)


def test_scalar_selftest_lines_match_reference():
    """The host half of the selftest (scalar algebra) is bit-identical to the
    reference's (same draws, same formulas)."""
    import paper_2001_08289_b200.scalars as sc
    from paper_2001_08289_b200 import selftest
    from paper_2001_08289_b200.exceptions import BackendError

    try:
        S = selftest.reference_module()  # the reference's own draws (selftest.py:55-72)
    except BackendError:
        pytest.skip("reference package not installed (baseline/_ref)")
    rng = np.random.default_rng(S.SEED)
    worst = [0.0] * 4
    for _ in range(200):
        ivr = S._random_interval(rng)
        s = S._random_sigma1(rng, ivr)
        iv = sc.SpectralInterval(ivr.alpha, ivr.beta)  # this package's scalar algebra from here on
        t = sc.map_t(s, iv)
        worst[0] = max(worst[0], S._rel(sc.inverse_map_t(t, iv) - s, s))
        pr = sc.solve_p(iv)
        a_rec = -1.0 - pr.p1 ** 2 / (pr.p2 ** 2 - 1.0)
        b_rec = -1.0 - pr.p1 ** 2 / pr.p2 ** 2
        worst[1] = max(worst[1], S._rel(a_rec - iv.alpha, iv.alpha), S._rel(b_rec - iv.beta, iv.beta))
        worst[2] = max(worst[2], S._rel(sc.verify_sigma1(t, pr) - s, s))
        e2p, j3p = sc.aux_constants(t, pr)
        row2 = (t - 1.0) * (pr.p1 * pr.p2 + pr.p2 ** 2 * e2p) + e2p
        row3 = (t - 1.0) * (pr.p1 * pr.p3 + pr.p2 * pr.p3 * e2p) - j3p
        worst[3] = max(worst[3], S._rel(row2, e2p), S._rel(row3, j3p))
    ref = {r["name"]: r["measured"] for r in META["selftest"]}
    names = ["t_map_round_trip", "interval_recovery_from_p", "sigma1_reconstruction", "field_equation_rows"]
    assert [ref[n] for n in names] == worst
