"""GPU: the slab-decomposed 3-D path (fftc_slab_* kernels + the slab driver)
at world size 1 against the 3-D golden fixtures, and against the monolithic
fftc_solve on a larger random medium."""

from __future__ import annotations

import numpy as np
import pytest

from golden_io import load_group
from parity import REL

pytestmark = pytest.mark.gpu
ALPHA, BETA = 0.25, 4.0


def _cfg(case):
    import paper_2001_08289_b200 as fb

    sk = fb.SchemeKind(case["scheme"])
    kw = dict(scheme=sk, sigma1=complex(*case["sigma1"]), tol=case["tol"], max_iters=case["max_iters"])
    if sk.substituted:
        kw["interval"] = fb.SpectralInterval(ALPHA, BETA)
    if case.get("e0") is not None:
        kw["e0"] = tuple(complex(*v) for v in case["e0"])
    return fb.SolverConfig(**kw)


@pytest.mark.parametrize("name", ["3d_cube16_basic", "3d_cube16_em", "3d_cube16_basic_sub", "3d_cube16_em_sub",
                                  "3d_random16_em_sub", "3d_embed_basic", "3d_cube32_em_sub"])
def test_slab_world1_matches_golden(name):
    from paper_2001_08289_b200.slab import solve_slab
    from test_gpu_parity import _chi

    g = load_group("3d")[name]
    r = solve_slab(_chi(g["case"]["geom"]), _cfg(g["case"]))
    assert r["status"].value == g["status"] and r["iterations"] == g["iterations"]
    gs = complex(*g["sigma_star"])
    assert abs(r["sigma_star"] - gs) <= REL * abs(gs)
    h = g["history"]
    dev = np.array([s for s, _ in r["history"]])
    assert np.max(np.abs(dev - (h[:, 1] + 1j * h[:, 2])) / np.abs(h[:, 1] + 1j * h[:, 2])) <= REL


def test_slab_world1_matches_monolithic_64():
    import paper_2001_08289_b200 as fb
    from paper_2001_08289_b200.slab import solve_slab

    pm = fb.build_random_medium(64, 3, seed=20260809, smoothing=4.0, fraction=0.3)
    for scheme in ("basic", "em_sub"):
        sk = fb.SchemeKind(scheme)
        cfg = fb.SolverConfig(scheme=sk, sigma1=50.0, tol=1e-8, max_iters=2000, e0=(1 / 3 ** 0.5,) * 3,
                              interval=fb.SpectralInterval(ALPHA, BETA) if sk.substituted else None)
        a = fb.solve(pm, cfg)
        b = solve_slab(pm.chi, cfg)
        assert a.iterations == b["iterations"]
        assert abs(a.sigma_star - b["sigma_star"]) <= 1e-12 * abs(a.sigma_star)
