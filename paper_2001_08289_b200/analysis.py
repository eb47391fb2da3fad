"""Batched mis-estimation study.

The reference's ``misestimation_report`` (fftcond/analysis.py:166-201) runs
the accelerated substituted scheme twice -- under the true singularity
interval and under an assumed one -- one solve after the other.  Here both
runs, and any number of such pairs, are independent points of ONE
``fftc_solve_batch`` call (include/fftcond_b200.h), which runs them
concurrently on the device.  The records and their fields mirror the
reference's ``MisestimationRun`` / ``MisestimationReport``; ``wall_time`` is
each solve's device time (batched runs overlap, so there is no per-run wall
clock).
"""

from __future__ import annotations

from dataclasses import dataclass
from typing import Sequence

from .cell import PhaseMap
from .scalars import SchemeKind, SpectralInterval
from .solver import SolveResult, SolverConfig, TerminationStatus, estimate_rate


@dataclass
class MisestimationRun:
    interval: SpectralInterval
    status: TerminationStatus
    iterations: int
    estimated_rate: float | None
    sigma_star: complex
    wall_time: float

    @classmethod
    def from_result(cls, interval, result: SolveResult, window, wall_time):
        """analysis.py:134-149: the rate over the last `window` steps when the
        history is long enough and strictly positive there."""
        rate = None
        if len(result.history) >= window + 1 and all(r > 0 for r in result.history.residuals()[-(window + 1):]):
            rate = estimate_rate(result.history, window)
        return cls(interval=interval, status=result.status, iterations=result.iterations, estimated_rate=rate,
                   sigma_star=result.sigma_star, wall_time=wall_time)


@dataclass
class MisestimationReport:
    """Side-by-side accelerated runs under two singularity estimates (analysis.py:152-163)."""

    sigma1: complex
    true_run: MisestimationRun
    assumed_run: MisestimationRun

    @property
    def rate_penalty(self) -> float | None:
        if self.true_run.estimated_rate is None or self.assumed_run.estimated_rate is None:
            return None
        return self.assumed_run.estimated_rate - self.true_run.estimated_rate


def _em_sub_cfg(sigma1, interval, cfg: SolverConfig) -> SolverConfig:
    return SolverConfig(scheme=SchemeKind.EYRE_MILTON_SUB, sigma1=sigma1, interval=interval, e0=cfg.e0, tol=cfg.tol,
                        max_iters=cfg.max_iters, sigma0_override=cfg.sigma0_override)


def misestimation_reports(pmap: PhaseMap, cases: Sequence[tuple], cfg: SolverConfig,
                          rate_window: int = 10) -> list[MisestimationReport]:
    """One report per (sigma1, true_interval, assumed_interval) case; all
    2 * len(cases) em_sub solves run as one device batch."""
    from .sweep import _solve_local_gpu

    cfgs = []
    for sigma1, true_iv, assumed_iv in cases:
        cfgs += [_em_sub_cfg(sigma1, true_iv, cfg), _em_sub_cfg(sigma1, assumed_iv, cfg)]
    res = _solve_local_gpu(pmap, cfgs)
    out = []
    for i, (sigma1, true_iv, assumed_iv) in enumerate(cases):
        rt, ra = res[2 * i], res[2 * i + 1]
        out.append(MisestimationReport(
            sigma1=complex(sigma1),
            true_run=MisestimationRun.from_result(true_iv, rt, rate_window, (rt.device_ms or 0.0) / 1e3),
            assumed_run=MisestimationRun.from_result(assumed_iv, ra, rate_window, (ra.device_ms or 0.0) / 1e3)))
    return out


def misestimation_report(pmap: PhaseMap, sigma1: complex, true_interval: SpectralInterval,
                         assumed_interval: SpectralInterval, cfg: SolverConfig,
                         rate_window: int = 10) -> MisestimationReport:
    """analysis.py:166-201 with its two runs batched on the device."""
    return misestimation_reports(pmap, [(sigma1, true_interval, assumed_interval)], cfg, rate_window)[0]
