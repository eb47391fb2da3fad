"""GPU parity at the BASELINE 3-D configurations (C3: 512^3 cube, em_sub,
sigma1 = 100; C4: 1024^3 seeded random medium, basic and em_sub, sigma1 = 50)
against the oracle restatement of the reference loops (solvers.py:280-331,
:366-443; the reference itself is 2-D only):

* full solves of the same recipes at 128^3 and 256^3 (c3red, c4red), through
  the TMA-tiled column passes on the z-blocked work layout, with per-component
  sum |F|^2 of the returned fields as a size-independent field check;
* the first iterations AT the stated sizes (c3first: 512^3; c4first:
  1024^3 on the frozen medium), every history record within the protocol;
* the memory-lean em_sub schedule (compact S/T, one work field -- what runs
  C4's accelerated arm on one GPU) bit for bit against the normal schedule,
  and against the 512^3 fixture.
Protocol: tests/parity.py."""

from __future__ import annotations

import math
import os

import numpy as np
import pytest

from golden_io import load_group
from parity import check
from test_gpu_parity import _chi, run_case

pytestmark = pytest.mark.gpu


def _cases(group):
    return [pytest.param(v, id=k) for k, v in load_group(group).items()]


def _sumsq_check(r, g, rel=1e-9):
    """sum |F_c|^2 of E, J (and S, T) against the oracle's, per component."""
    want = g.get("field_sumsq") or {}
    got = {"E": r.E_field, "J": r.J_field}
    if r.aug_field is not None:
        got.update(S=r.aug_field.S, T=r.aug_field.T)
    for key, ref in want.items():
        data = got[key].data
        scale = max(max(ref), 1e-300)
        for c, v in enumerate(ref):
            s = float(np.sum(np.abs(data[c]) ** 2))
            assert abs(s - v) <= rel * scale, f"{g['case']['name']} {key}[{c}]: {s!r} vs {v!r}"


@pytest.mark.parametrize("g", _cases("c3red") + _cases("c4red"))
def test_3d_config_recipes_full_solve(g):
    r = run_case(g["case"])
    check(r, g)
    if g["status"] == "Converged":
        _sumsq_check(r, g)


@pytest.mark.parametrize("g", _cases("c3first") + _cases("c4first"))
def test_3d_configs_first_iterations_at_size(g):
    import paper_2001_08289_b200 as fb

    case = g["case"]
    chi = _chi(case["geom"])
    sch = fb.SchemeKind(case["scheme"])
    cfg = fb.SolverConfig(scheme=sch, sigma1=complex(*case["sigma1"]), tol=case["tol"], max_iters=case["max_iters"],
                          e0=tuple(complex(*v) for v in case["e0"]),
                          interval=fb.SpectralInterval(0.25, 4.0) if sch.substituted else None)
    r = fb.solve(fb.PhaseMap(chi), cfg, fields=False)
    check(r, g)
    if sch is fb.SchemeKind.EYRE_MILTON_SUB:  # the memory-lean schedule on the same fixture
        os.environ["FFTC_LEAN"] = "1"
        try:
            rl = fb.solve(fb.PhaseMap(chi), cfg, fields=False)
        finally:
            os.environ.pop("FFTC_LEAN", None)
        check(rl, g)
        assert [(h.sigma_star, h.residual) for h in rl.history] == [(h.sigma_star, h.residual) for h in r.history]


def _lean_pair(chi, sigma1, e0, max_iters, fields):
    import paper_2001_08289_b200 as fb
    from paper_2001_08289_b200 import native

    cfg = fb.SolverConfig(scheme=fb.SchemeKind.EYRE_MILTON_SUB, sigma1=sigma1, tol=1e-10, max_iters=max_iters, e0=e0,
                          interval=fb.SpectralInterval(0.25, 4.0))
    out = []
    for lean in ("0", "1"):
        os.environ["FFTC_LEAN"] = lean
        try:
            r = fb.solve(fb.PhaseMap(chi), cfg, fields=fields)
            out.append((r, native.last_layout()))
        finally:
            os.environ.pop("FFTC_LEAN", None)
    (a, la), (b, lb) = out
    assert not (la & 256) and (lb & 256), (la, lb)
    return a, b


@pytest.mark.parametrize("shape,frac,sigma1", [((256, 256, 512), 0.3, 50.0), ((256, 512, 512), 0.25, 20.0 + 3.0j)])
def test_lean_em_sub_bit_identical(shape, frac, sigma1):
    """Compact S/T slots and the split flux / residual-field transforms change
    where values live and the launch order, not the arithmetic: histories,
    sigma*, <E>, <J> and the returned fields equal the normal schedule's bit
    for bit."""
    rng = np.random.default_rng(3)
    chi = rng.random(shape) < frac
    a, b = _lean_pair(chi, sigma1, (0.6, 0.0, 0.8), 60, True)
    assert (a.status, a.iterations) == (b.status, b.iterations)
    assert [(h.sigma_star, h.residual) for h in a.history] == [(h.sigma_star, h.residual) for h in b.history]
    assert np.array_equal(a.mean_E, b.mean_E) and np.array_equal(a.mean_J, b.mean_J)
    for fa, fb_ in ((a.E_field, b.E_field), (a.J_field, b.J_field), (a.aug_field.S, b.aug_field.S),
                    (a.aug_field.T, b.aug_field.T)):
        assert np.array_equal(fa.data, fb_.data)


def test_lean_em_sub_c3_converged():
    """C3's cube at 512 x 256 x 256 (lean schedule) runs to convergence with
    the same records as the normal one."""
    n = (256, 256, 512)
    chi = np.zeros(n, dtype=bool)
    chi[48:208, 48:208, 96:416] = True
    a, b = _lean_pair(chi, 100.0, (1.0, 0.0, 0.0), 2000, False)
    assert a.status.value == "Converged" and b.iterations == a.iterations
    assert b.sigma_star == a.sigma_star and math.isfinite(abs(b.sigma_star))
