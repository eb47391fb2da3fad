"""Host-side scalar algebra that parameterises the device iteration.

Restates the reference's scheme enum, interval, t-map and p-solve
(``fftcond/transform.py:23-168``).  These run once per solve on the host;
only their outputs (t, p1..p3, sigma0) cross the C ABI.
"""

from __future__ import annotations

import cmath
import math
from dataclasses import dataclass
from enum import Enum

from .exceptions import BranchCutError, DegenerateParamError, IntervalError, PoleError

_REL_TOL = 1e-12


class SchemeKind(Enum):
    """basic Moulinec-Suquet, Eyre-Milton, and their substituted variants."""

    BASIC = "basic"
    EYRE_MILTON = "em"
    BASIC_SUB = "basic_sub"
    EYRE_MILTON_SUB = "em_sub"

    @property
    def substituted(self) -> bool:
        return self in (SchemeKind.BASIC_SUB, SchemeKind.EYRE_MILTON_SUB)

    @property
    def accelerated(self) -> bool:
        return self in (SchemeKind.EYRE_MILTON, SchemeKind.EYRE_MILTON_SUB)

    @property
    def abi_code(self) -> int:
        return {"basic": 0, "em": 1, "basic_sub": 2, "em_sub": 3}[self.value]


@dataclass(frozen=True)
class SpectralInterval:
    """Assumed singular set [-beta, -alpha] of sigma*(sigma1)."""

    alpha: float
    beta: float

    def __post_init__(self):
        a, b = self.alpha, self.beta
        if not (math.isfinite(a) and math.isfinite(b) and 0.0 < a < b):
            raise IntervalError(f"need 0 < alpha < beta < inf, got alpha={a}, beta={b}")


@dataclass(frozen=True)
class SubstitutionParams:
    """(p1, p2, p3) with p1^2 + p2^2 + p3^2 = 1 realising an interval."""

    interval: SpectralInterval
    p1: complex
    p2: complex
    p3: complex

    def __post_init__(self):
        q1, q2, q3 = self.p1 ** 2, self.p2 ** 2, self.p3 ** 2
        scale = max(1.0, abs(q1) + abs(q2) + abs(q3))
        if abs(q1 + q2 + q3 - 1.0) > _REL_TOL * scale:
            raise ValueError(f"p1^2+p2^2+p3^2 = {q1 + q2 + q3} is not 1")
        alpha_back = -1.0 - q1 / (q2 - 1.0)
        beta_back = -1.0 - q1 / q2
        a, b = self.interval.alpha, self.interval.beta
        if (abs(alpha_back - a) > _REL_TOL * max(1.0, abs(a))
                or abs(beta_back - b) > _REL_TOL * max(1.0, abs(b))):
            raise ValueError(f"params recover ({alpha_back}, {beta_back}), expected ({a}, {b})")


def map_t(sigma1: complex, interval: SpectralInterval) -> complex:
    """t = (sigma1 + alpha)(1 + beta) / ((sigma1 + beta)(1 + alpha))."""
    s = complex(sigma1)
    a, b = interval.alpha, interval.beta
    den = (s + b) * (1.0 + a)
    if den == 0:
        raise PoleError(f"map_t has a pole at sigma1 = {-b}")
    return (s + a) * (1.0 + b) / den


def map_z(scheme: SchemeKind, sigma1: complex, interval: SpectralInterval | None = None) -> complex:
    """Disk coordinate z = (x - 1)/(x + 1), x = sigma1, sqrt(sigma1), t or sqrt(t)."""
    x = complex(sigma1)
    if scheme.substituted:
        if interval is None:
            raise IntervalError(f"scheme {scheme.value} requires an interval")
        x = map_t(x, interval)
    if scheme.accelerated:
        if x.imag == 0.0 and x.real <= 0.0:
            raise BranchCutError(
                f"{'t' if scheme.substituted else 'sigma1'} = {x} lies on the closed negative real axis")
        x = cmath.sqrt(x)
    if x == -1.0:
        raise PoleError(f"map_z pole: argument {x} gives a zero denominator")
    return (x - 1.0) / (x + 1.0)


def solve_p(interval: SpectralInterval) -> SubstitutionParams:
    """p1 = sqrt((1+a)(1+b)/(b-a)) > 0, p2 = i sqrt((1+a)/(b-a)), p3 from p.p = 1, Im p3 > 0."""
    a, b = interval.alpha, interval.beta
    width = b - a
    sq1 = (1.0 + a) * (1.0 + b) / width
    sq2 = -(1.0 + a) / width
    sq3 = 1.0 - sq1 - sq2
    p3 = cmath.sqrt(complex(sq3))
    if p3.imag < 0:
        p3 = -p3
    return SubstitutionParams(interval=interval, p1=complex(math.sqrt(sq1)),
                              p2=1j * math.sqrt(-sq2), p3=p3)


def inverse_map_t(t: complex, interval: SpectralInterval) -> complex:
    """Inverse of map_t (transform.py:113-122); pole at t = (1+beta)/(1+alpha)."""
    tt = complex(t)
    a, b = interval.alpha, interval.beta
    den = tt * (1.0 + a) - (1.0 + b)
    if den == 0:
        raise PoleError(f"inverse_map_t has a pole at t = {(1.0 + b) / (1.0 + a)}")
    return (a * (1.0 + b) - b * tt * (1.0 + a)) / den


def _coupling_denominator(t: complex, params: SubstitutionParams) -> complex:
    """(t-1) p2^2 + 1 (transform.py:171-177)."""
    den = (t - 1.0) * params.p2 ** 2 + 1.0
    if den == 0:
        raise DegenerateParamError(f"(t-1)*p2^2 + 1 vanishes at t = {t}; coupling is degenerate")
    return den


def aux_constants(t: complex, params: SubstitutionParams) -> tuple[complex, complex]:
    """(E2p, J3p): slot couplings of the gradient- and flux-type fields (transform.py:180-190)."""
    tt = complex(t)
    den = _coupling_denominator(tt, params)
    return (1.0 - tt) * params.p1 * params.p2 / den, params.p1 * params.p3 * (tt - 1.0) / den


def verify_sigma1(t: complex, params: SubstitutionParams) -> complex:
    """sigma1 reproduced by the 3-vector model at t (transform.py:193-201)."""
    tt = complex(t)
    return 1.0 + params.p1 ** 2 * (tt - 1.0) / _coupling_denominator(tt, params)
