"""Solver entry points: the reference API in front of the CUDA iteration.

Public surface and semantics follow ``fftcond/solvers.py``:

* ``SolverConfig`` validation            -- solvers.py:93-125
* ``SolveResult`` / history containers   -- solvers.py:54-90, :128-144
* reference-medium choice and its errors -- solvers.py:221-240, :334-352
* ``solve_basic`` ... ``solve`` dispatch -- solvers.py:446-491

What changed is below the seam: ``_solve_h`` / ``_solve_aug``
(solvers.py:280-331, :366-443) no longer loop in numpy; they hand the
problem to ``fftc_solve`` in ``libfftcond_b200.so`` (include/fftcond_b200.h),
which runs the fused FFT sweeps and the stopping monitor on the GPU and
returns the history, status and field averages.  Fields stay on the device
until read.  There is no CPU fallback.
"""

from __future__ import annotations

import cmath
import ctypes as C
import math
import threading
import weakref
from dataclasses import dataclass
from enum import Enum

import numpy as np

from . import fields as _fields
from . import native
from .cell import PhaseMap
from .exceptions import BackendError, BranchCutError, ContractError, DegenerateParamError, IntervalError
from .fields import AugmentedField, VectorField
from .scalars import SchemeKind, SpectralInterval, map_t, solve_p

DIVERGENCE_FACTOR = 1e6
_TINY = 1e-300


class TerminationStatus(Enum):
    CONVERGED = "Converged"
    MAX_ITERS = "MaxIters"
    DIVERGED = "Diverged"


_STATUS = {native.FFTC_CONVERGED: TerminationStatus.CONVERGED,
           native.FFTC_MAX_ITERS: TerminationStatus.MAX_ITERS,
           native.FFTC_DIVERGED: TerminationStatus.DIVERGED}


@dataclass(frozen=True)
class HistoryRecord:
    iteration: int
    sigma_star: complex
    residual: float


class ConvergenceHistory:
    """(iteration, sigma*, residual) per recorded iteration."""

    def __init__(self):
        self.records: list[HistoryRecord] = []

    def append(self, iteration: int, sigma_star: complex, residual: float):
        if not math.isfinite(residual):
            raise ContractError(f"residual must be finite, got {residual}")
        if self.records and iteration <= self.records[-1].iteration:
            raise ContractError("iteration indices must increase strictly")
        self.records.append(HistoryRecord(iteration, sigma_star, residual))

    @classmethod
    def from_array(cls, arr: np.ndarray) -> "ConvergenceHistory":
        h = cls()
        h.records = [HistoryRecord(k + 1, complex(float(r[0]), float(r[1])), float(r[2]))
                     for k, r in enumerate(arr)]
        return h

    def __len__(self) -> int:
        return len(self.records)

    def __iter__(self):
        return iter(self.records)

    def residuals(self) -> list[float]:
        return [r.residual for r in self.records]

    def sigma_stars(self) -> list[complex]:
        return [r.sigma_star for r in self.records]


@dataclass
class SolverConfig:
    """Run parameters (same fields and checks as the reference).

    ``e0`` may have 2 or 3 components; on a 3-D cell a 2-vector is padded
    with a zero z component.
    """

    scheme: SchemeKind
    sigma1: complex
    interval: SpectralInterval | None = None
    e0: tuple = (1.0, 0.0)
    tol: float = 1e-8
    max_iters: int = 1000
    sigma0_override: complex | None = None

    def __post_init__(self):
        if self.tol <= 0:
            raise ValueError(f"tol must be positive, got {self.tol}")
        if self.max_iters < 1:
            raise ValueError(f"max_iters must be >= 1, got {self.max_iters}")
        if self.scheme.substituted and self.interval is None:
            raise IntervalError(f"scheme {self.scheme.value} needs a spectral interval")
        if len(self.e0) not in (2, 3):
            raise ContractError(f"applied field e0 needs 2 or 3 components, got {len(self.e0)}")
        if all(abs(complex(v)) == 0 for v in self.e0):
            raise ContractError("applied field e0 must be nonzero")

    def e0_vector(self, dim: int | None = None) -> np.ndarray:
        v = [complex(x) for x in self.e0]
        if dim is not None:
            if len(v) > dim:
                if any(abs(x) != 0 for x in v[dim:]):
                    raise ContractError(f"e0 has {len(v)} components on a {dim}-D cell")
                v = v[:dim]
            v = v + [0j] * (dim - len(v))
        return np.array(v, dtype=np.complex128)


@dataclass
class SolveResult:
    sigma_star: complex
    E_field: VectorField
    J_field: VectorField
    history: ConvergenceHistory
    status: TerminationStatus
    degenerate_flux: bool = False
    aug_field: AugmentedField | None = None
    mean_E: np.ndarray | None = None       # <E> computed on the device
    mean_J: np.ndarray | None = None       # <J> computed on the device
    device_ms: float | None = None         # device time of the solve
    kernel_launches: int = 0

    @property
    def iterations(self) -> int:
        return len(self.history)

    @property
    def converged(self) -> bool:
        return self.status is TerminationStatus.CONVERGED


# ---------------------------------------------------------------------------
# reference-medium choice (solvers.py:221-240, :334-352)
# ---------------------------------------------------------------------------

def _reference_h(cfg: SolverConfig, accelerated: bool) -> complex:
    s1 = complex(cfg.sigma1)
    if cfg.sigma0_override is not None:
        s0 = complex(cfg.sigma0_override)
    elif accelerated:
        if s1.imag == 0.0 and s1.real <= 0.0:
            raise BranchCutError(
                f"sigma1 = {s1} lies on the closed negative real axis; the square-root reference is undefined")
        s0 = cmath.sqrt(s1)
    else:
        s0 = (s1 + 1.0) / 2.0
    if s0 == 0:
        raise DegenerateParamError("reference conductivity sigma0 vanishes")
    if accelerated and (s1 + s0 == 0 or 1.0 + s0 == 0):
        raise DegenerateParamError(f"sigma + sigma0 vanishes in one phase (sigma0 = {s0})")
    return s0


def _reference_aug(cfg: SolverConfig, t: complex, accelerated: bool) -> complex:
    if cfg.sigma0_override is not None:
        s0 = complex(cfg.sigma0_override)
    elif accelerated:
        if t.imag == 0.0 and t.real <= 0.0:
            raise BranchCutError(
                f"t = {t} lies on the closed negative real axis; sigma1 sits inside the assumed singular interval")
        s0 = cmath.sqrt(t)
    else:
        if t == -1.0:
            raise DegenerateParamError("t = -1 makes the reference (t+1)/2 vanish")
        s0 = (t + 1.0) / 2.0
    if s0 == 0:
        raise DegenerateParamError("reference sigma0 vanishes")
    if accelerated and (1.0 + s0 == 0 or t + s0 == 0):
        raise DegenerateParamError(f"A + sigma0 I is singular for sigma0 = {s0}")
    return s0


# ---------------------------------------------------------------------------
# the seam: device solve
# ---------------------------------------------------------------------------

def _torch():
    import torch

    if not torch.cuda.is_available():
        raise BackendError("no CUDA device: the B200 backend has no CPU fallback")
    return torch


# Device copies of phase maps, per map (by identity: PhaseMap hashes its
# whole indicator) and per device, dropped when the map is collected.
_CHI_CACHE: dict = {}  # id(pmap) -> (weakref to pmap, {device index: tensor})
_CHI_LOCK = threading.Lock()


def _device_chi(pmap: PhaseMap, torch):
    dev = torch.cuda.current_device()
    key = id(pmap)
    with _CHI_LOCK:
        ent = _CHI_CACHE.get(key)
        if ent is not None and ent[0]() is pmap and dev in ent[1]:
            return ent[1][dev]
    t = torch.from_numpy(pmap.chi.astype(np.uint8)).to(device="cuda")
    with _CHI_LOCK:
        ent = _CHI_CACHE.get(key)
        if ent is None or ent[0]() is not pmap:
            ent = (weakref.ref(pmap, lambda _r, k=key: _CHI_CACHE.pop(k, None)), {})
            _CHI_CACHE[key] = ent
        ent[1][dev] = t
    return t


def release_device_copies(pmap: PhaseMap) -> None:
    """Drop the cached device copies of a phase map (1 GiB at 1024^3)."""
    with _CHI_LOCK:
        _CHI_CACHE.pop(id(pmap), None)


def _check_grid(pmap: PhaseMap):
    L = native.lib()
    for n in pmap.grid:
        if not L.fftc_supported_length(int(n)):
            raise ContractError(f"grid axis of length {n} is not supported (even lengths >= 2)")


def _problem(pmap: PhaseMap, chi) -> native.Problem:
    prob = native.Problem()
    prob.d = pmap.dim
    prob.n[0], prob.n[1], prob.n[2] = pmap.nx, pmap.ny, pmap.nz
    prob.chi = chi.data_ptr()
    return prob


def _params(cfg: SolverConfig, d: int) -> native.Params:
    """Host-side scalar setup of one solve (reference expressions), packed for the ABI.

    Raises exactly what the reference raises before its loop starts:
    _reference_h / _reference_aug (solvers.py:221-240, :334-352), map_t and
    solve_p (transform.py:99-168).
    """
    scheme = cfg.scheme
    t, p = 1.0 + 0j, (0j, 0j, 0j)
    if scheme.substituted:
        t = map_t(complex(cfg.sigma1), cfg.interval)
        sp = solve_p(cfg.interval)
        p = (sp.p1, sp.p2, sp.p3)
        s0 = _reference_aug(cfg, t, scheme.accelerated)
    else:
        s0 = _reference_h(cfg, scheme.accelerated)
    e0 = cfg.e0_vector(d)
    par = native.Params()
    par.scheme = scheme.abi_code
    par.sigma1[:] = native.cpair(cfg.sigma1)
    par.sigma0[:] = native.cpair(s0)
    par.t[:] = native.cpair(t)
    par.p1[:] = native.cpair(p[0])
    par.p2[:] = native.cpair(p[1])
    par.p3[:] = native.cpair(p[2])
    for c in range(3):
        par.e0[c][:] = native.cpair(e0[c] if c < d else 0)
    par.tol = float(cfg.tol)
    par.max_iters = int(cfg.max_iters)
    par.gamma1_scale = float(_fields._gamma1_scale)
    return par


def _result_from(res: native.Result, hist: np.ndarray, d: int, E=None, J=None, aug=None) -> SolveResult:
    n = int(res.iterations)
    aug_field = None
    E_field = VectorField.from_device(E) if E is not None else None
    if aug is not None:
        Q = VectorField.from_device(aug[0])
        aug_field = AugmentedField(Q, VectorField.from_device(aug[1]), VectorField.from_device(aug[2]))
        if E_field is None:
            E_field = Q  # one field behind both names, like the reference
    return SolveResult(
        sigma_star=complex(res.sigma_star[0], res.sigma_star[1]),
        E_field=E_field,
        J_field=VectorField.from_device(J) if J is not None else None,
        history=ConvergenceHistory.from_array(hist[:n]),
        status=_STATUS[int(res.status)],
        degenerate_flux=bool(res.degenerate_flux),
        aug_field=aug_field,
        mean_E=np.array([complex(res.mean_E[c][0], res.mean_E[c][1]) for c in range(d)]),
        mean_J=np.array([complex(res.mean_J[c][0], res.mean_J[c][1]) for c in range(d)]),
        device_ms=float(res.device_ms),
        kernel_launches=int(res.kernel_launches),
    )


def _run_device(pmap: PhaseMap, cfg: SolverConfig, want_fields: bool = True) -> SolveResult:
    par = _params(cfg, pmap.dim)  # host validation first: raises before any device work
    torch = _torch()
    L = native.lib()
    _check_grid(pmap)
    d = pmap.dim
    chi = _device_chi(pmap, torch)
    grid = pmap.grid
    prob = _problem(pmap, chi)
    hist = np.empty((int(cfg.max_iters), 3), dtype=np.float64)
    E = J = aug = None
    if want_fields:
        J = torch.empty((d,) + grid, dtype=torch.complex128, device="cuda")
        if cfg.scheme.substituted:
            # E and aug.Q are one array, as in the reference (solvers.py:435-443
            # wraps the same fq in both): the library writes Q once
            aug = torch.empty((3, d) + grid, dtype=torch.complex128, device="cuda")
        else:
            E = torch.empty((d,) + grid, dtype=torch.complex128, device="cuda")
    res = native.Result()
    stream = torch.cuda.current_stream().cuda_stream
    rc = L.fftc_solve(C.byref(prob), C.byref(par), hist.ctypes.data, hist.shape[0],
                      None if E is None else E.data_ptr(), None if J is None else J.data_ptr(),
                      None if aug is None else aug.data_ptr(), C.byref(res), stream)
    if rc != 0:
        raise BackendError(f"fftc_solve failed ({rc}): {native.last_error()}")
    return _result_from(res, hist, d, E, J, aug)


def _solve_h(pmap: PhaseMap, cfg: SolverConfig, accelerated: bool, want_fields: bool = True) -> SolveResult:
    """H-space loop (basic / em) on the device; replaces solvers.py:280-331."""
    expected = SchemeKind.EYRE_MILTON if accelerated else SchemeKind.BASIC
    if cfg.scheme is not expected:
        cfg = SolverConfig(scheme=expected, sigma1=cfg.sigma1, e0=cfg.e0, tol=cfg.tol,
                           max_iters=cfg.max_iters, sigma0_override=cfg.sigma0_override)
    return _run_device(pmap, cfg, want_fields)


def _solve_aug(pmap: PhaseMap, cfg: SolverConfig, accelerated: bool, want_fields: bool = True) -> SolveResult:
    """Augmented loop (basic_sub / em_sub) on the device; replaces solvers.py:366-443."""
    expected = SchemeKind.EYRE_MILTON_SUB if accelerated else SchemeKind.BASIC_SUB
    if cfg.scheme is not expected:
        cfg = SolverConfig(scheme=expected, sigma1=cfg.sigma1, interval=cfg.interval, e0=cfg.e0,
                           tol=cfg.tol, max_iters=cfg.max_iters, sigma0_override=cfg.sigma0_override)
    return _run_device(pmap, cfg, want_fields)


def _check_scheme(cfg: SolverConfig, expected: SchemeKind):
    if cfg.scheme is not expected:
        raise ContractError(f"config carries scheme {cfg.scheme.value!r}, expected {expected.value!r}")


def solve_basic(pmap: PhaseMap, cfg: SolverConfig, *, fields: bool = True) -> SolveResult:
    """Moulinec-Suquet basic scheme, sigma0 = (sigma1 + 1)/2."""
    _check_scheme(cfg, SchemeKind.BASIC)
    return _solve_h(pmap, cfg, accelerated=False, want_fields=fields)


def solve_em(pmap: PhaseMap, cfg: SolverConfig, *, fields: bool = True) -> SolveResult:
    """Eyre-Milton scheme, sigma0 = sqrt(sigma1)."""
    _check_scheme(cfg, SchemeKind.EYRE_MILTON)
    return _solve_h(pmap, cfg, accelerated=True, want_fields=fields)


def solve_basic_sub(pmap: PhaseMap, cfg: SolverConfig, *, fields: bool = True) -> SolveResult:
    """Basic scheme in the substituted (Q, S, T) space, t = map_t(sigma1)."""
    _check_scheme(cfg, SchemeKind.BASIC_SUB)
    return _solve_aug(pmap, cfg, accelerated=False, want_fields=fields)


def solve_em_sub(pmap: PhaseMap, cfg: SolverConfig, *, fields: bool = True) -> SolveResult:
    """Eyre-Milton scheme in the substituted space, sigma0 = sqrt(t)."""
    _check_scheme(cfg, SchemeKind.EYRE_MILTON_SUB)
    return _solve_aug(pmap, cfg, accelerated=True, want_fields=fields)


_DISPATCH = {
    SchemeKind.BASIC: solve_basic,
    SchemeKind.EYRE_MILTON: solve_em,
    SchemeKind.BASIC_SUB: solve_basic_sub,
    SchemeKind.EYRE_MILTON_SUB: solve_em_sub,
}


def solve(pmap: PhaseMap, cfg: SolverConfig, *, fields: bool = True) -> SolveResult:
    """Run the scheme named by ``cfg.scheme``.

    ``fields=False`` (extension) skips the E / J / augmented output fields --
    sigma*, the history and the field means are still returned.  At 1024^3
    two device fields are 96 GB on top of the ~96 GB iteration workspace."""
    return _DISPATCH[cfg.scheme](pmap, cfg, fields=fields)


def estimate_rate(history: ConvergenceHistory, window: int) -> float:
    """Geometric-mean residual ratio over the last ``window`` steps (solvers.py:207-218)."""
    if window < 1:
        raise ContractError(f"window must be >= 1, got {window}")
    if len(history) < window + 1:
        raise ContractError(f"need {window + 1} records for a window of {window}, got {len(history)}")
    tail = history.residuals()[-(window + 1):]
    if any(r <= 0 for r in tail):
        raise ContractError("rate estimate needs strictly positive residuals")
    return (tail[-1] / tail[0]) ** (1.0 / window)
