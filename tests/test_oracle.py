"""CPU: pin the oracle restatement against the golden fixtures produced by
the live reference (oracle/gen_golden.py), bit for bit at d = 2, and check
the d = 3 generalisation's known answers.  No GPU needed."""

from __future__ import annotations

import math

import numpy as np
import pytest

from golden_io import load_group
from oracle import fftcond_oracle as O

ALPHA, BETA = 0.25, 4.0


def _chi(geom):
    from test_gpu_parity import _chi as build

    return build(geom)


def _run(case):
    e0 = None if case.get("e0") is None else [complex(*v) for v in case["e0"]]
    ov = None if case.get("sigma0_override") is None else complex(*case["sigma0_override"])
    return O.solve(_chi(case["geom"]), case["scheme"], complex(*case["sigma1"]), e0=e0, tol=case["tol"],
                   max_iters=case["max_iters"], alpha=ALPHA, beta=BETA, sigma0_override=ov)


def _small(g, limit=2e5):
    """Cases cheap enough for the CPU suite (voxels x iterations)."""
    n = int(np.prod(_chi(g["case"]["geom"]).shape))
    return n * max(g["iterations"], 1) <= limit


def _params(group, pred=lambda g: True):
    return [pytest.param(v, id=k) for k, v in load_group(group).items() if pred(v)]


@pytest.mark.parametrize("g", _params("edge", _small) + _params("c1")
                         + _params("general", lambda g: g["source"].startswith("reference") and _small(g)))
def test_oracle_bit_identical_to_reference(g):
    """d = 2: the restatement reproduces the live reference bit for bit."""
    if g["source"].startswith("oracle"):
        pytest.skip("3-D fixture")
    r = _run(g["case"])
    assert r.status == g["status"]
    assert r.iterations == g["iterations"]
    assert r.degenerate_flux == g["degenerate_flux"]
    h = g["history"]
    for (k, s, res), row in zip(r.history, h):
        assert k == int(row[0])
        assert s.real == row[1] and s.imag == row[2], (k, s, row)
        assert res == row[3]
    assert complex(r.sigma_star) == complex(*g["sigma_star"])


@pytest.mark.parametrize("g", _params("c2small", lambda g: g["case"]["geom"]["n"] == 64 and g["iterations"] < 400))
def test_oracle_c2_reduced(g):
    r = _run(g["case"])
    assert r.iterations == g["iterations"]
    assert complex(r.sigma_star) == complex(*g["sigma_star"])


@pytest.mark.parametrize("g", _params("c5small", lambda g: int(g["case"]["name"][-3:]) % 32 == 0
                                      and g["iterations"] < 300))
def test_oracle_c5_sample(g):
    r = _run(g["case"])
    assert r.status == g["status"] and r.iterations == g["iterations"]
    assert complex(r.sigma_star) == complex(*g["sigma_star"])


def test_embedding_3d_reproduces_2d_reference():
    """A z-invariant 3-D cell (n_z = 2, e0 in the xy plane) is the 2-D problem."""
    g2 = {k: v for k, v in load_group("c2small").items()}
    chi2 = O.centred_box(16, 8)
    chi3 = np.repeat(chi2[None], 2, axis=0)
    for scheme in ("basic", "em", "basic_sub", "em_sub"):
        r2 = O.solve(chi2, scheme, 10.0, tol=1e-10, max_iters=5000, alpha=ALPHA, beta=BETA)
        r3 = O.solve(chi3, scheme, 10.0, tol=1e-10, max_iters=5000, alpha=ALPHA, beta=BETA)
        assert r2.iterations == r3.iterations
        assert abs(r3.sigma_star - r2.sigma_star) <= 1e-13 * abs(r2.sigma_star)
    assert g2 is not None


def test_3d_golden_records_match_oracle():
    """3-D fixtures (from the oracle) stay reproducible."""
    for name, g in load_group("3d").items():
        if name not in ("3d_cube16_basic", "3d_embed_em", "3d_random16_em_sub"):
            continue
        r = _run(g["case"])
        assert r.iterations == g["iterations"]
        assert complex(r.sigma_star) == complex(*g["sigma_star"])


class TestKnownAnswers3D:
    """Reference known answers (tests/test_solvers.py) restated at d = 3."""

    def test_uniform_phase2_one_iteration(self):
        for scheme in ("basic", "em", "basic_sub", "em_sub"):
            r = O.solve(np.zeros((4, 4, 4), bool), scheme, 3.0, alpha=ALPHA, beta=BETA)
            assert r.status == "Converged" and r.iterations == 1
            assert abs(r.sigma_star - 1.0) <= 1e-13

    def test_laminates(self):
        # layers normal to x (series): harmonic mean; normal to z (parallel to x): arithmetic
        chi = np.zeros((8, 8, 8), bool)
        chi[:, :, ::2] = True
        r = O.solve(chi, "basic", 3.0, tol=1e-12)
        assert r.sigma_star == pytest.approx(1.5, rel=1e-10)
        chi = np.zeros((8, 8, 8), bool)
        chi[::2] = True
        r = O.solve(chi, "basic", 3.0, tol=1e-12)
        assert r.sigma_star == pytest.approx(2.0, rel=1e-10)

    def test_geometric_series_all_phase1(self):
        # test_solvers.py:177-192 in 3-D: sigma*_k = s1 + (first - s1) g^k
        s1 = 2.0
        r = O.solve(np.ones((4, 4, 4), bool), "basic_sub", s1, tol=1e-13, max_iters=200, alpha=ALPHA,
                    beta=BETA, e0=(1.0, 0.0, 0.0))
        p1, p2, _ = O.solve_p(ALPHA, BETA)
        t = O.map_t(s1, ALPHA, BETA)
        g = (t - 1.0) * (1.0 - 2.0 * p2 ** 2) / (t + 1.0)
        first = 1.0 + (t - 1.0) * p1 ** 2
        for k, (_, s, _) in enumerate(r.history):
            expected = s1 + (first - s1) * g ** k
            assert abs(s - expected) <= 1e-12 * max(1.0, abs(expected))

    def test_gamma1_properties_3d(self):
        rng = np.random.default_rng(0)
        f = rng.standard_normal((3, 8, 8, 8)) + 1j * rng.standard_normal((3, 8, 8, 8))
        g = O.gamma1(f)
        assert np.abs(O.gamma1(g) - g).max() <= 1e-12 * np.abs(g).max()
        assert np.abs(g.mean(axis=(1, 2, 3))).max() <= 1e-13
        c = np.ones((3, 8, 8, 8), complex)
        assert np.abs(O.gamma1(c)).max() <= 1e-14


@pytest.mark.parametrize("shape,scheme,s1,e0", [
    ((32, 32), "basic", 50.0, None),
    ((32, 32), "em_sub", -30.0 + 5.0j, None),
    ((16, 16, 16), "basic", 50.0, (3 ** -0.5,) * 3),
    ((16, 16, 16), "em_sub", 100.0, (1.0, 0.0, 0.0)),
    ((8, 12, 16), "em_sub", 20.0 + 3.0j, (0.6, 0.2j, -0.3)),
])
def test_lean_oracle_bitwise(shape, scheme, s1, e0):
    """oracle/lean_oracle.py (the bounded-memory form used for the 512^3 and
    1024^3 fixtures) reproduces fftcond_oracle bit for bit: every history
    record, sigma*, the returned fields and (em_sub) the augmented slots."""
    from oracle import lean_oracle as LO

    rng = np.random.default_rng(7)
    chi = O.centred_box(shape[0], shape[0] // 2, len(shape)) if len(set(shape)) == 1 else rng.random(shape) < 0.3
    a = O.solve(chi, scheme, s1, e0=e0, tol=1e-10, max_iters=150, alpha=ALPHA, beta=BETA)
    b = LO.solve(chi, scheme, s1, e0=e0, tol=1e-10, max_iters=150, alpha=ALPHA, beta=BETA)
    assert (a.status, a.iterations) == (b.status, b.iterations)
    for (ka, sa, ra), (kb, sb, rb) in zip(a.history, b.history):
        assert (ka, sa, ra) == (kb, sb, rb)
    assert np.array_equal(a.E, b.E) and np.array_equal(a.J, b.J)
    if scheme == "em_sub":
        assert all(np.array_equal(x, y) for x, y in zip(a.aug, b.aug))


def test_c4_medium_frozen_digest(tmp_path):
    """The config-4 recipe is deterministic: a small instance rebuilt twice is
    identical, and the frozen 1024^3 digest is what c4_phase_map checks."""
    from paper_2001_08289_b200 import cell

    a = cell.build_random_medium(32, 3, seed=cell.C4_SEED, smoothing=cell.C4_SMOOTHING, fraction=cell.C4_FRACTION)
    b = cell.c4_phase_map(32, directory=str(tmp_path))
    assert a == b and abs(float(a.volume_fraction) - 0.30) < 1e-3
    assert set(cell.C4_CHI_SHA256) == {1024} and len(cell.C4_CHI_SHA256[1024]) == 64
