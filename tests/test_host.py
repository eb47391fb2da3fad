"""CPU: host-side mirror of the reference API (config validation, reference
medium, scalar algebra, geometry) -- the parts that stay on the host.
Mirrors reference tests/test_transform.py, test_geometry.py and the config
sections of test_solvers.py."""

from __future__ import annotations

import cmath
from fractions import Fraction

import numpy as np
import pytest

import paper_2001_08289_b200 as fb
from paper_2001_08289_b200.solver import _reference_aug, _reference_h

BENCH = fb.SpectralInterval(0.25, 4.0)


def cfg_for(scheme, sigma1, **kw):
    kw.setdefault("interval", BENCH if scheme.substituted else None)
    return fb.SolverConfig(scheme=scheme, sigma1=sigma1, **kw)


class TestConfig:
    def test_sub_scheme_requires_interval(self):
        with pytest.raises(fb.IntervalError):
            fb.SolverConfig(scheme=fb.SchemeKind.EYRE_MILTON_SUB, sigma1=2.0)

    def test_bad_tolerance(self):
        with pytest.raises(ValueError):
            fb.SolverConfig(scheme=fb.SchemeKind.BASIC, sigma1=2.0, tol=0.0)

    def test_bad_max_iters(self):
        with pytest.raises(ValueError):
            fb.SolverConfig(scheme=fb.SchemeKind.BASIC, sigma1=2.0, max_iters=0)

    def test_zero_applied_field(self):
        with pytest.raises(fb.ContractError):
            fb.SolverConfig(scheme=fb.SchemeKind.BASIC, sigma1=2.0, e0=(0.0, 0.0))

    def test_e0_padding_and_dimension(self):
        c = fb.SolverConfig(scheme=fb.SchemeKind.BASIC, sigma1=2.0, e0=(1.0, 0.5))
        assert list(c.e0_vector(3)) == [1.0, 0.5, 0.0]
        c3 = fb.SolverConfig(scheme=fb.SchemeKind.BASIC, sigma1=2.0, e0=(1.0, 0.5, 0.25))
        with pytest.raises(fb.ContractError):
            c3.e0_vector(2)

    def test_scheme_mismatch(self):
        pm = fb.build_square_array(8, 0.5)
        with pytest.raises(fb.ContractError):
            fb.solve_basic(pm, cfg_for(fb.SchemeKind.EYRE_MILTON, 2.0))


class TestReferenceMedium:
    """solvers.py:221-240 and :334-352: values and errors."""

    def test_values(self):
        assert _reference_h(cfg_for(fb.SchemeKind.BASIC, 10.0), False) == 5.5
        assert _reference_h(cfg_for(fb.SchemeKind.EYRE_MILTON, 9.0), True) == 3.0
        t = fb.map_t(10.0, BENCH)
        assert _reference_aug(cfg_for(fb.SchemeKind.BASIC_SUB, 10.0), t, False) == (t + 1) / 2
        assert _reference_aug(cfg_for(fb.SchemeKind.EYRE_MILTON_SUB, 10.0), t, True) == cmath.sqrt(t)

    def test_branch_cut(self):
        with pytest.raises(fb.BranchCutError):
            _reference_h(cfg_for(fb.SchemeKind.EYRE_MILTON, -0.5), True)
        with pytest.raises(fb.BranchCutError):
            _reference_h(cfg_for(fb.SchemeKind.EYRE_MILTON, 0.0), True)
        t = fb.map_t(-1.0, BENCH)  # inside [-4, -1/4]
        with pytest.raises(fb.BranchCutError):
            _reference_aug(cfg_for(fb.SchemeKind.EYRE_MILTON_SUB, -1.0), t, True)

    def test_degenerate(self):
        with pytest.raises(fb.DegenerateParamError):
            _reference_h(cfg_for(fb.SchemeKind.BASIC, -1.0), False)

    def test_override(self):
        assert _reference_h(cfg_for(fb.SchemeKind.EYRE_MILTON, -0.5, sigma0_override=1.0), True) == 1.0


class TestScalars:
    """Known answers of reference tests/test_transform.py:162-199."""

    def test_p_values(self):
        p = fb.solve_p(BENCH)
        assert p.p1 ** 2 == pytest.approx(5 / 3, rel=1e-14)
        assert p.p2 ** 2 == pytest.approx(-1 / 3, rel=1e-14)
        assert p.p3 ** 2 == pytest.approx(-1 / 3, rel=1e-14)
        assert p.p1.imag == 0 and p.p1.real > 0 and p.p2.imag > 0 and p.p3.imag > 0

    def test_map_t(self):
        assert fb.map_t(1.0, BENCH) == pytest.approx(1.0)
        assert fb.map_t(-0.25, BENCH) == pytest.approx(0.0, abs=1e-15)
        assert fb.map_t(10.0, BENCH) == pytest.approx(2.928571428571429, rel=1e-14)
        with pytest.raises(fb.PoleError):
            fb.map_t(-4.0, BENCH)

    def test_interval_validation(self):
        for a, b in ((0.0, 1.0), (2.0, 1.0), (1.0, float("inf"))):
            with pytest.raises(fb.IntervalError):
                fb.SpectralInterval(a, b)

    def test_matches_oracle(self):
        from oracle import fftcond_oracle as O

        p = fb.solve_p(BENCH)
        assert (p.p1, p.p2, p.p3) == O.solve_p(0.25, 4.0)
        for s in (0.1, 10.0, 1000.0, 19.207 + 4.118j):
            assert fb.map_t(s, BENCH) == O.map_t(s, 0.25, 4.0)

    def test_map_z(self):
        z = fb.map_z(fb.SchemeKind.BASIC, 10.0)
        assert z == pytest.approx(9 / 11)
        assert abs(fb.map_z(fb.SchemeKind.EYRE_MILTON, 9.0)) == pytest.approx(0.5)


class TestGeometry:
    def test_square_array(self):
        pm = fb.build_square_array(256, 0.5)
        assert pm.volume_fraction == Fraction(1, 4)
        assert pm.chi[64:192, 64:192].all() and pm.chi.sum() == 128 * 128
        with pytest.raises(ValueError):
            fb.build_square_array(8, 0.375)
        with pytest.raises(ValueError):
            fb.build_square_array(5, 0.4)

    def test_phase_map_validation(self):
        with pytest.raises(ValueError):
            fb.PhaseMap(np.zeros((3, 4), bool))
        with pytest.raises(ValueError):
            fb.PhaseMap(np.zeros((4,), bool))
        pm = fb.PhaseMap(np.zeros((4, 6, 8), bool))
        assert pm.dim == 3 and (pm.nx, pm.ny, pm.nz) == (8, 6, 4)
        assert not pm.chi.flags.writeable

    def test_cube_and_random(self):
        pm = fb.build_cube_array(16, 10)
        assert pm.chi.sum() == 1000
        rm = fb.build_random_medium(16, 3, seed=20260809, smoothing=2.0, fraction=0.3)
        assert abs(float(rm.volume_fraction) - 0.3) < 0.01
        assert rm == fb.build_random_medium(16, 3, seed=20260809, smoothing=2.0, fraction=0.3)


class TestHistory:
    def test_contracts(self):
        h = fb.ConvergenceHistory()
        h.append(1, 1.0 + 0j, 0.5)
        with pytest.raises(fb.ContractError):
            h.append(1, 1.0 + 0j, 0.4)
        with pytest.raises(fb.ContractError):
            h.append(2, 1.0 + 0j, float("nan"))

    def test_estimate_rate(self):
        h = fb.ConvergenceHistory()
        for k, r in enumerate([2.0 ** -k for k in range(12)], start=1):
            h.append(k, 1.0 + 0j, r)
        assert fb.estimate_rate(h, 10) == pytest.approx(0.5, rel=1e-12)
        with pytest.raises(fb.ContractError):
            fb.estimate_rate(h, 20)


def test_no_cpu_fallback_without_gpu(monkeypatch):
    """The product path fails loudly when CUDA is unavailable."""
    import torch

    if torch.cuda.is_available():
        pytest.skip("GPU present")
    with pytest.raises(fb.BackendError):
        fb.solve(fb.build_square_array(8, 0.5), cfg_for(fb.SchemeKind.BASIC, 2.0))


def test_bench_gpus_flag_relaunches_under_torchrun(monkeypatch):
    """bench.py --gpus N without a torchrun environment relaunches itself as N
    ranks (torch.distributed.run, 127.0.0.1); a WORLD_SIZE that disagrees with
    --gpus is an error, not a silent single-GPU run."""
    import subprocess
    import types

    import bench

    seen = {}

    def fake_run(cmd, *a, **k):
        seen["cmd"] = cmd
        return types.SimpleNamespace(returncode=0)

    monkeypatch.delenv("WORLD_SIZE", raising=False)
    monkeypatch.setattr(subprocess, "run", fake_run)
    monkeypatch.setattr(bench.sys, "argv", ["bench.py", "--gpus", "4", "--steps", "2"])
    assert bench._relaunch(types.SimpleNamespace(gpus=4)) == 0
    cmd = seen["cmd"]
    assert cmd[1:4] == ["-m", "torch.distributed.run", "--nnodes=1"] and "--nproc-per-node=4" in cmd
    assert "127.0.0.1" in cmd and cmd[-4:] == ["--gpus", "4", "--steps", "2"]
    assert bench._relaunch(types.SimpleNamespace(gpus=1)) is None
    monkeypatch.setenv("WORLD_SIZE", "2")
    assert bench._relaunch(types.SimpleNamespace(gpus=2)) is None
    assert bench._relaunch(types.SimpleNamespace(gpus=4)) == 2


def test_bench_byte_models():
    """Per-launch algorithmic bytes add up to the
    schedule totals quoted there."""
    import bench

    f = 0.25
    V = 48.0
    k = bench._bytes_per_voxel("em_sub", 3, f)
    assert abs(sum(k.values()) - (14 * V + 7 * f * V + 2)) < 1e-9
    assert abs(bench._survey_bytes("em_sub", 3, f) - (15 * V + 6 * f * V + 2)) < 1e-9
    lean = bench._bytes_lean(f)
    tot = sum(v * bench.LEAN_LAUNCHES.get(n, 1) for n, v in lean.items())
    assert abs(tot - (15 * V + 9 * f * V + 6)) < 1e-9
    k2 = bench._bytes_per_voxel("basic", 2, f)
    assert abs(sum(k2.values()) - (7 * 32 + 2)) < 1e-9
