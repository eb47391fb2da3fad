"""GPU parity: the CUDA iteration (through the public API and the C ABI)
against golden fixtures frozen from the live reference (2-D) and the
oracle restatement (3-D).  Protocol in tests/parity.py."""

from __future__ import annotations

import os

import numpy as np
import pytest

from golden_io import GOLDEN, load_group
from parity import check, field_check

pytestmark = pytest.mark.gpu

ALPHA, BETA = 0.25, 4.0


def _chi(geom):
    # same builders as oracle/gen_golden.py (duplicated: the GPU box has no
    # /root/reference and tests must not depend on the generator's imports)
    kind = geom["kind"]
    if kind == "square":
        n, m = geom["n"], geom["side"]
        chi = np.zeros((n, n), dtype=bool)
        lo = (n - m) // 2
        chi[lo:lo + m, lo:lo + m] = True
        return chi
    if kind == "uniform":
        return np.full((geom["ny"], geom["nx"]), bool(geom["phase1"]))
    if kind == "laminate_x":
        chi = np.zeros((geom["n"], geom["n"]), dtype=bool)
        chi[:, ::2] = True
        return chi
    if kind == "laminate_y":
        chi = np.zeros((geom["n"], geom["n"]), dtype=bool)
        chi[::2, :] = True
        return chi
    if kind == "rect":
        ny, nx, my, mx = geom["ny"], geom["nx"], geom["my"], geom["mx"]
        chi = np.zeros((ny, nx), dtype=bool)
        chi[(ny - my) // 2:(ny - my) // 2 + my, (nx - mx) // 2:(nx - mx) // 2 + mx] = True
        return chi
    if kind == "random":
        rng = np.random.default_rng(geom["seed"])
        return rng.random((geom["ny"], geom["nx"])) < geom["frac"]
    if kind == "cube":
        n, m = geom["n"], geom["side"]
        chi = np.zeros((n, n, n), dtype=bool)
        lo = (n - m) // 2
        chi[lo:lo + m, lo:lo + m, lo:lo + m] = True
        return chi
    if kind == "embed2d":
        return np.repeat(_chi(geom["base"])[None], geom["nz"], axis=0)
    if kind == "random3d":
        rng = np.random.default_rng(geom["seed"])
        return rng.random((geom["n"],) * 3) < geom["frac"]
    if kind == "c4medium":  # BASELINE config 4 recipe (frozen SHA-256 at 1024^3)
        from paper_2001_08289_b200 import cell

        return np.asarray(cell.c4_phase_map(geom["n"]).chi)
    raise ValueError(kind)


def run_case(case):
    import paper_2001_08289_b200 as fb

    chi = _chi(case["geom"])
    sch = fb.SchemeKind(case["scheme"])
    kw = dict(scheme=sch, sigma1=complex(*case["sigma1"]), tol=case["tol"], max_iters=case["max_iters"])
    if sch.substituted:
        kw["interval"] = fb.SpectralInterval(ALPHA, BETA)
    if case.get("e0") is not None:
        kw["e0"] = tuple(complex(*v) for v in case["e0"])
    if case.get("sigma0_override") is not None:
        kw["sigma0_override"] = complex(*case["sigma0_override"])
    return fb.solve(fb.PhaseMap(chi), fb.SolverConfig(**kw))


def _cases(group, pred=None):
    g = load_group(group)
    return [pytest.param(v, id=k) for k, v in g.items() if pred is None or pred(v)]


@pytest.mark.parametrize("g", _cases("edge"))
def test_edge_cases(g):
    r = run_case(g["case"])
    check(r, g)
    if g.get("fields_file") and g["status"] == "Converged":
        field_check(r, os.path.join(GOLDEN, g["fields_file"]))


@pytest.mark.parametrize("g", _cases("c1"))
def test_config1(g):
    r = run_case(g["case"])
    rep = check(r, g)
    assert r.iterations == 62


@pytest.mark.parametrize("g", _cases("c2small"))
def test_config2_reduced(g):
    check(run_case(g["case"]), g)


@pytest.mark.parametrize("g", _cases("c2full"))
def test_config2_full_size(g):
    """BASELINE configs[1] at 2048^2 against the live reference's outputs."""
    check(run_case(g["case"]), g)


@pytest.mark.parametrize("g", _cases("c5full"))
def test_config5_full_size(g):
    """BASELINE configs[4] points at 1024^2 against the live reference (complex sigma1)."""
    check(run_case(g["case"]), g)


@pytest.mark.parametrize("g", _cases("3d"))
def test_3d(g):
    r = run_case(g["case"])
    check(r, g)
    if g.get("fields_file") and g["status"] == "Converged":
        field_check(r, os.path.join(GOLDEN, g["fields_file"]))


@pytest.mark.parametrize("g", _cases("c5small", lambda v: int(v["case"]["name"][-3:]) % 8 == 0))
def test_config5_sample(g):
    check(run_case(g["case"]), g)


def test_bit_identical_histories():
    # reference tests/test_solvers.py:518-527: two runs, identical records
    import paper_2001_08289_b200 as fb

    pm = fb.build_square_array(32, 0.5)
    cfg = fb.SolverConfig(scheme=fb.SchemeKind.EYRE_MILTON_SUB, sigma1=2.0,
                          interval=fb.SpectralInterval(ALPHA, BETA), tol=1e-10)
    r1, r2 = fb.solve(pm, cfg), fb.solve(pm, cfg)
    assert len(r1.history) == len(r2.history)
    for a, b in zip(r1.history, r2.history):
        assert a.sigma_star == b.sigma_star and a.residual == b.residual


def test_repeat_determinism_long_em_sub():
    """Repeats of a 1000-iteration em_sub solve at 1024^2 are bit identical.
    Guards the column sweep's shared TMA ring: a half running ahead on
    parseval-only lines once read a slot still in flight, corrupting one
    residual record in a few hundred repeats (cols_tma.cuh, cbars)."""
    g = load_group("c5full")["c5_1024_p004"]
    runs = [run_case(g["case"]) for _ in range(6)]
    h0 = [(h.sigma_star, h.residual) for h in runs[0].history]
    assert len(h0) == 1000
    for r in runs[1:]:
        assert [(h.sigma_star, h.residual) for h in r.history] == h0


@pytest.mark.parametrize("shape, scheme", [((256, 256, 8), "em_sub"), ((256, 256, 8), "basic"),
                                           ((512, 256, 4), "em"), ((1024, 256, 2), "basic_sub")])
def test_3d_tma_column_passes_vs_oracle(shape, scheme):
    """Grids whose y and z lines (256..1024) run the TMA tile kernels
    (cols3_lg.cuh), against the oracle restatement (pinned to the reference
    by the 2-D goldens and the 2-D embedding check)."""
    import paper_2001_08289_b200 as fb
    from oracle import fftcond_oracle as O

    rng = np.random.default_rng(3)
    chi = rng.random(shape) < 0.3
    sk = fb.SchemeKind(scheme)
    e0 = (0.6, 0.0, 0.8)
    cfg = fb.SolverConfig(scheme=sk, sigma1=10.0 + 2j, tol=1e-8, max_iters=200, e0=e0,
                          interval=fb.SpectralInterval(ALPHA, BETA) if sk.substituted else None)
    r = fb.solve(fb.PhaseMap(chi), cfg)
    ref = O.solve(chi, scheme, 10.0 + 2j, e0=e0, tol=1e-8, max_iters=200, alpha=ALPHA, beta=BETA)
    assert r.iterations == len(ref.history) and r.status.value == ref.status
    for h, (_, s, res) in zip(r.history, ref.history):
        assert abs(h.sigma_star - s) <= 1e-10 * abs(s)
        assert abs(h.residual - res) <= 1e-6 * res


@pytest.mark.parametrize("shape, scheme", [((256, 256, 8), "em_sub"), ((512, 256, 8), "basic"),
                                           ((256, 512, 8), "em"), ((256, 256, 16), "basic_sub")])
def test_3d_zblocked_work_layout_bit_identical(shape, scheme, monkeypatch):
    """The z-blocked work-field layout (Args::zbs, 32 z-planes per block) only
    moves data: histories are bit identical to the reference layout
    (FFTC_ZBLOCK=0), for several block shifts."""
    import paper_2001_08289_b200 as fb

    rng = np.random.default_rng(5)
    pm = fb.PhaseMap(rng.random(shape) < 0.3)
    sk = fb.SchemeKind(scheme)
    cfg = fb.SolverConfig(scheme=sk, sigma1=10.0 + 2j, tol=1e-9, max_iters=120, e0=(0.6, 0.0, 0.8),
                          interval=fb.SpectralInterval(ALPHA, BETA) if sk.substituted else None)
    from paper_2001_08289_b200 import native

    runs = {}
    for zb in ("0", "5", "3", "8"):
        monkeypatch.setenv("FFTC_ZBLOCK", zb)
        r = fb.solve(pm, cfg)
        assert native.last_layout() == int(zb)  # the blocked path really ran
        runs[zb] = [(h.sigma_star, h.residual) for h in r.history]
    for zb in ("5", "3", "8"):
        assert runs[zb] == runs["0"], zb


@pytest.mark.parametrize("g", _cases("general"))
def test_general_grids(g):
    """Even axis lengths outside the fused transforms (6, 24, 30, 40, 48, 50,
    96, 12^3, 24^3): the general path (general.cuh around cuFFT) against the
    live reference (2-D) and the oracle (3-D)."""
    from paper_2001_08289_b200 import native

    assert not all(native.lib().fftc_fused_length(n) for n in _chi(g["case"]["geom"]).shape)
    check(run_case(g["case"]), g)


@pytest.mark.parametrize("g", _cases("c2small", lambda v: v["case"]["geom"]["n"] == 64) + _cases("c1")
                         + _cases("3d", lambda v: "16" in v["case"]["name"]))
def test_general_path_on_fused_grids(g, monkeypatch):
    """FFTC_GENERAL=1 runs power-of-two grids on the general path: same
    goldens, same iteration counts as the fused sweeps."""
    monkeypatch.setenv("FFTC_GENERAL", "1")
    check(run_case(g["case"]), g)


@pytest.mark.parametrize("g", _cases("big"))
def test_largest_lengths(g):
    """Axes at the fused maximum (4096: 4096 x 64, 64 x 4096, 4096^2 for three
    iterations) and beyond it (8192: the general path), against the live
    reference."""
    check(run_case(g["case"]), g)
