"""GPU: the batched sweep path (fftc_solve_batch via sweep.solve_sweep)
against golden fixtures of BASELINE config 5 (64^2 for every 16th point;
1024^2 points where the live-reference goldens exist)."""

from __future__ import annotations

import numpy as np
import pytest

from golden_io import load_group
from parity import REL

pytestmark = pytest.mark.gpu
ALPHA, BETA = 0.25, 4.0


def _check(recs, goldens):
    for r, g in zip(recs, goldens):
        name = g["case"]["name"]
        assert r["status"].value == g["status"], name
        assert r["iterations"] == g["iterations"], name
        gs = complex(*g["sigma_star"])
        assert abs(r["sigma_star"] - gs) <= REL * abs(gs), (name, r["sigma_star"], gs)
        h = g["history"]
        if len(h):
            dev = r["history"]
            srel = np.abs((dev[:, 0] + 1j * dev[:, 1]) - (h[:, 1] + 1j * h[:, 2])) / np.abs(h[:, 1] + 1j * h[:, 2])
            assert srel.max() <= REL, name


def _run(goldens, n):
    import paper_2001_08289_b200 as fb
    from paper_2001_08289_b200.sweep import solve_sweep

    cfgs = [fb.SolverConfig(scheme=fb.SchemeKind.EYRE_MILTON_SUB, sigma1=complex(*g["case"]["sigma1"]),
                            tol=g["case"]["tol"], max_iters=g["case"]["max_iters"],
                            interval=fb.SpectralInterval(ALPHA, BETA)) for g in goldens]
    return solve_sweep(fb.build_square_array(n, 0.5), cfgs)


def test_sweep_64_sample():
    g = load_group("c5small")
    sample = [v for k, v in g.items() if int(k[-3:]) % 16 == 1]
    _check(_run(sample, 64), sample)


def test_sweep_1024_goldens():
    g = load_group("c5full")
    if not g:
        pytest.skip("no 1024^2 config-5 goldens")
    vals = list(g.values())
    _check(_run(vals, 1024), vals)


def test_misestimation_reports_batched_match_sequential():
    """analysis.py:166-201 batched: every run equals the same em_sub solve
    made on its own (one fftc_solve_batch for all pairs)."""
    import paper_2001_08289_b200 as fb

    pm = fb.build_square_array(64, 0.5)
    cfg = fb.SolverConfig(scheme=fb.SchemeKind.EYRE_MILTON_SUB, sigma1=1.0, tol=1e-8, max_iters=400,
                          interval=fb.SpectralInterval(0.25, 4.0))
    true_iv, bench_iv = fb.SpectralInterval(0.25, 4.0), fb.SpectralInterval(0.1, 10.0)
    cases = [(2.0, true_iv, bench_iv), (10.0 + 1.0j, true_iv, bench_iv), (0.5, bench_iv, true_iv)]
    reps = fb.misestimation_reports(pm, cases, cfg, rate_window=3)
    assert len(reps) == 3
    for (s1, tiv, aiv), rep in zip(cases, reps):
        for iv, run in ((tiv, rep.true_run), (aiv, rep.assumed_run)):
            one = fb.solve(pm, fb.SolverConfig(scheme=fb.SchemeKind.EYRE_MILTON_SUB, sigma1=s1, tol=1e-8,
                                               max_iters=400, interval=iv))
            assert (run.status, run.iterations, run.sigma_star) == (one.status, one.iterations, one.sigma_star)
            assert run.interval is iv and run.wall_time > 0
        assert rep.rate_penalty is None or abs(rep.rate_penalty) < 1
    single = fb.misestimation_report(pm, 2.0, true_iv, bench_iv, cfg, rate_window=3)
    assert single.true_run.sigma_star == reps[0].true_run.sigma_star
