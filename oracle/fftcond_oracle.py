"""CPU oracle for the FFT field iteration -- TEST INFRASTRUCTURE ONLY.

This module is the checker, never the product.  Only ``tests/``,
``__graft_entry__.smoke()`` and ``bench.py``'s ``cpu_baseline`` /
``--impl reference`` legs may import it.  The product path
(``paper_2001_08289_b200``) never imports it and has no CPU fallback.

What it is: a d-generic (d = 2 or 3) numpy restatement of the reference
fixed-point loops of ``fftcond`` (arXiv 2001.08289 companion package).
Every numerical step keeps the reference's numpy operation order so that
at d = 2 it reproduces the reference bit for bit (pinned by
``tests/test_oracle.py`` against golden fixtures produced by the live
reference, see ``oracle/gen_golden.py``).  At d = 3 there is no
reference (the reference is strictly 2-D, ``geometry.py:33-34``); the
restatement generalises the same formulas with a third wave-vector
component and is pinned by the 2-D embedding check (a z-invariant cell
with nz = 2 reproduces the 2-D reference) and by the 3-D known answers
in ``tests/test_oracle.py``.

Reference citations (``/root/reference/pkg/src/fftcond``):

* reductions         -- spectral_ops.py:33-55  (_compensated_total,
                        _compensated_ctotal, _mean_vec)
* wave vectors       -- spectral_ops.py:109-117 (_wavevectors)
* Gamma_1 projection -- spectral_ops.py:120-128 (_gamma1_arr)
* stopping monitor   -- solvers.py:243-277 (_Monitor), constants :50-51
* H-space loop       -- solvers.py:280-331 (_solve_h), sigma0 :221-240
* augmented loop     -- solvers.py:366-443 (_solve_aug), sigma0 :334-352,
                        local operator A :355-363
* scalar setup       -- transform.py:99-110 (map_t), :152-168 (solve_p)
"""

from __future__ import annotations

import cmath
import math
from dataclasses import dataclass, field
from functools import lru_cache

import numpy as np

DIVERGENCE_FACTOR = 1e6  # solvers.py:50
TINY = 1e-300  # solvers.py:51

SCHEMES = ("basic", "em", "basic_sub", "em_sub")


# --------------------------------------------------------------------------
# scalar setup (transform.py:99-110, :152-168; solvers.py:221-240, :334-352)
# --------------------------------------------------------------------------

def map_t(sigma1: complex, alpha: float, beta: float) -> complex:
    """t = (s + a)(1 + b) / ((s + b)(1 + a))  -- transform.py:99-110."""
    s = complex(sigma1)
    return (s + alpha) * (1.0 + beta) / ((s + beta) * (1.0 + alpha))


def solve_p(alpha: float, beta: float):
    """(p1, p2, p3) with p1 real > 0, Im p2 > 0, Im p3 > 0 -- transform.py:152-168."""
    p1_sq = (1.0 + alpha) * (1.0 + beta) / (beta - alpha)
    p2_sq = -(1.0 + alpha) / (beta - alpha)
    p3_sq = 1.0 - p1_sq - p2_sq
    p1 = complex(math.sqrt(p1_sq))
    p2 = 1j * math.sqrt(-p2_sq)
    p3 = cmath.sqrt(complex(p3_sq))
    if p3.imag < 0:
        p3 = -p3
    return p1, p2, p3


def reference_sigma0(scheme: str, sigma1: complex, t: complex | None,
                     override: complex | None = None) -> complex:
    """Reference-medium choice; raises ValueError where the reference raises."""
    if override is not None:
        s0 = complex(override)
    elif scheme == "basic":
        s0 = (complex(sigma1) + 1.0) / 2.0
    elif scheme == "em":
        s = complex(sigma1)
        if s.imag == 0.0 and s.real <= 0.0:
            raise ValueError("branch cut")
        s0 = cmath.sqrt(s)
    elif scheme == "basic_sub":
        if t == -1.0:
            raise ValueError("degenerate")
        s0 = (t + 1.0) / 2.0
    else:
        if t.imag == 0.0 and t.real <= 0.0:
            raise ValueError("branch cut")
        s0 = cmath.sqrt(t)
    return s0


# --------------------------------------------------------------------------
# reductions (spectral_ops.py:33-55), d-generic: rows run along x
# --------------------------------------------------------------------------

def total_real(values: np.ndarray) -> float:
    """Row sums (numpy pairwise) combined by an exactly rounded fsum."""
    rows = np.sum(values.reshape(-1, values.shape[-1]), axis=-1)
    if not np.all(np.isfinite(rows)):
        return float(np.sum(rows))
    return math.fsum(rows.tolist())


def total_complex(values: np.ndarray) -> complex:
    if np.iscomplexobj(values):
        return complex(total_real(values.real), total_real(values.imag))
    return complex(total_real(values), 0.0)


def component_means(data: np.ndarray) -> np.ndarray:
    """Per-component compensated mean of a (d, *grid) array."""
    npts = int(np.prod(data.shape[1:]))
    return np.array([total_complex(data[c]) / npts for c in range(data.shape[0])])


# --------------------------------------------------------------------------
# Gamma_1 (spectral_ops.py:109-128), d-generic
# --------------------------------------------------------------------------

@lru_cache(maxsize=8)
def wave_vectors(grid: tuple):
    """Integer wave vectors, component c = 0 (x) runs along the LAST axis.

    Returns ([k_x, k_y(, k_z)] broadcastable to ``grid``, 1/|k|^2 with the
    zero mode set to 0).  Nyquist modes keep the fftfreq value -n/2.
    """
    d = len(grid)
    ks = []
    for c in range(d):
        axis = d - 1 - c
        n = grid[axis]
        shape = [1] * d
        shape[axis] = n
        ks.append(np.fft.fftfreq(n, d=1.0 / n).reshape(shape))
    k2 = ks[0] * ks[0]
    for c in range(1, d):
        k2 = k2 + ks[c] * ks[c]
    k2 = np.broadcast_to(k2, grid).copy()
    inv = np.zeros_like(k2)
    nz = k2 != 0
    inv[nz] = 1.0 / k2[nz]
    return ks, inv


def gamma1(data: np.ndarray, scale: float = 1.0) -> np.ndarray:
    """Curl-free zero-mean projection k (k . F) / |k|^2 of a (d, *grid) field."""
    d = data.shape[0]
    grid = tuple(data.shape[1:])
    ks, inv = wave_vectors(grid)
    axes = tuple(range(-d, 0))
    fh = np.fft.fftn(data, axes=axes)
    dot = ks[0] * fh[0]
    for c in range(1, d):
        dot = dot + ks[c] * fh[c]
    dot = dot * (inv * scale)
    out = np.empty_like(fh)
    for c in range(d):
        out[c] = ks[c] * dot
    return np.fft.ifftn(out, axes=axes)


# --------------------------------------------------------------------------
# monitor (solvers.py:243-277)
# --------------------------------------------------------------------------

@dataclass
class OracleResult:
    status: str = "MaxIters"
    degenerate_flux: bool = False
    history: list = field(default_factory=list)  # (k, sigma*, residual)
    sigma_star: complex = 0j
    E: np.ndarray | None = None
    J: np.ndarray | None = None
    aug: tuple | None = None

    @property
    def iterations(self) -> int:
        return len(self.history)


class _Stop:
    def __init__(self, tol: float):
        self.tol = tol
        self.res0 = None
        self.prev = None

    def __call__(self, out: OracleResult, k: int, sstar: complex, res: float) -> bool:
        if not (math.isfinite(res) and cmath.isfinite(sstar)):
            out.status = "Diverged"
            return True
        out.history.append((k, sstar, res))
        if self.res0 is None:
            self.res0 = res
        settled = self.prev is None or abs(sstar - self.prev) <= self.tol * abs(sstar)
        if res <= self.tol and settled:
            out.status = "Converged"
            return True
        if self.res0 > 0 and res > DIVERGENCE_FACTOR * self.res0:
            out.status = "Diverged"
            return True
        self.prev = sstar
        return False


# --------------------------------------------------------------------------
# the solve loops
# --------------------------------------------------------------------------

def _applied(e0, grid):
    e0v = np.array([complex(v) for v in e0], dtype=np.complex128)
    e0f = np.empty((len(e0v),) + tuple(grid), dtype=np.complex128)
    for c in range(len(e0v)):
        e0f[c] = e0v[c]
    return e0v, np.vdot(e0v, e0v).real, e0f


def solve(chi: np.ndarray, scheme: str, sigma1: complex, *, e0=None, tol: float = 1e-8,
          max_iters: int = 1000, alpha: float | None = None, beta: float | None = None,
          sigma0_override: complex | None = None, gamma1_scale: float = 1.0,
          max_records: int | None = None) -> OracleResult:
    """Run one scheme on indicator ``chi`` (shape grid, d = chi.ndim).

    Mirrors ``fftcond.solve`` (solvers.py:489-491) for d = 2 and extends
    it to d = 3.  ``e0`` defaults to the unit x vector.
    """
    chi = np.asarray(chi, dtype=bool)
    d = chi.ndim
    if e0 is None:
        e0 = (1.0,) + (0.0,) * (d - 1)
    if scheme in ("basic", "em"):
        return _loop_h(chi, scheme == "em", complex(sigma1), e0, tol, max_iters,
                       sigma0_override, gamma1_scale)
    return _loop_aug(chi, scheme == "em_sub", complex(sigma1), e0, tol, max_iters,
                     alpha, beta, sigma0_override, gamma1_scale)


def _loop_h(chi, accelerated, sigma1, e0, tol, max_iters, override, scale):
    """solvers.py:280-331 restated."""
    s0 = reference_sigma0("em" if accelerated else "basic", sigma1, None, override)
    grid = chi.shape
    npts = chi.size
    sig = np.where(chi, sigma1, 1.0 + 0j)
    e0v, e0sq, e0f = _applied(e0, grid)
    out = OracleResult()
    stop = _Stop(tol)
    if accelerated:
        w = (sig + s0) * e0f
    else:
        e_raw = e0f.copy()
    e = j = g = None
    sstar = 0j
    with np.errstate(over="ignore", invalid="ignore"):
        for k in range(1, max_iters + 1):
            if k > 1:
                if accelerated:
                    rw = (sig - s0) * e_raw
                    w = 2.0 * s0 * e0f - 2.0 * gamma1(rw, scale) + rw
                else:
                    e_raw = e - g / s0
            if accelerated:
                e_raw = w / (sig + s0)
            delta = e0v - component_means(e_raw)
            e = e_raw + delta.reshape((-1,) + (1,) * len(grid))
            j = sig * e
            jm = component_means(j)
            den = float(np.linalg.norm(jm))
            sstar = complex(np.vdot(e0v, jm)) / e0sq
            if den < TINY and math.isfinite(den):
                out.degenerate_flux = True
                out.status = "Diverged"
                break
            g = gamma1(j, scale)
            res = math.sqrt(total_real(np.abs(g) ** 2) / npts) / den
            if stop(out, k, sstar, res):
                break
    out.sigma_star = out.history[-1][1] if out.history else sstar
    out.E, out.J = e, j
    return out


def apply_A(q, s, tt, t, p, chi):
    """A = (t - 1) chi'' + I on (Q, S, T) -- solvers.py:355-363."""
    p1, p2, p3 = p
    u = np.where(chi, p1 * q + p2 * s + p3 * tt, 0.0)
    tm1 = t - 1.0
    return (tm1 * p1 * u + q,
            np.where(chi, tm1 * p2 * u + s, 0.0),
            np.where(chi, tm1 * p3 * u + tt, 0.0))


def _loop_aug(chi, accelerated, sigma1, e0, tol, max_iters, alpha, beta, override, scale):
    """solvers.py:366-443 restated."""
    t = map_t(sigma1, alpha, beta)
    p = solve_p(alpha, beta)
    p1, p2, p3 = p
    s0 = reference_sigma0("em_sub" if accelerated else "basic_sub", sigma1, t, override)
    grid = chi.shape
    npts = chi.size
    e0v, e0sq, e0f = _applied(e0, grid)
    zeros = np.zeros_like(e0f)
    chif = chi.astype(np.float64)
    out = OracleResult()
    stop = _Stop(tol)
    fq_raw, fs_raw, ft_raw = e0f.copy(), zeros.copy(), zeros.copy()
    if accelerated:
        aq, as_, at = apply_A(fq_raw, fs_raw, ft_raw, t, p, chi)
        wq, ws, wt = aq + s0 * fq_raw, as_ + s0 * fs_raw, at + s0 * ft_raw
        inv_scale = 1.0 / (1.0 + s0)
        inv_c = (t - 1.0) / (t + s0)
    fq = fs = ft = jq = js = g = None
    jq_raw = js_raw = jt_raw = None
    tau = (t - 1.0) * p1 * chif
    sstar = 0j
    bshape = (-1,) + (1,) * len(grid)
    with np.errstate(over="ignore", invalid="ignore"):
        for k in range(1, max_iters + 1):
            if k > 1:
                if accelerated:
                    rq = jq_raw - s0 * fq_raw
                    rs = js_raw - s0 * fs_raw
                    rt = jt_raw - s0 * ft_raw
                    wq = 2.0 * s0 * e0f - 2.0 * gamma1(rq, scale) + rq
                    ws = -rs
                    wt = rt
                else:
                    fq_raw = fq - g / s0
                    fs_raw = np.where(chi, fs - js / s0, 0.0)
            if accelerated:
                u = np.where(chi, p1 * wq + p2 * ws + p3 * wt, 0.0)
                fq_raw = inv_scale * (wq - inv_c * p1 * u)
                fs_raw = np.where(chi, inv_scale * (ws - inv_c * p2 * u), 0.0)
                ft_raw = np.where(chi, inv_scale * (wt - inv_c * p3 * u), 0.0)
            jq_raw, js_raw, jt_raw = apply_A(fq_raw, fs_raw, ft_raw, t, p, chi)
            delta = e0v - component_means(fq_raw)
            dfield = delta.reshape(bshape)
            fq, fs, ft = fq_raw + dfield, fs_raw, ft_raw
            jq = jq_raw + p1 * tau * dfield + dfield
            js = js_raw + p2 * tau * dfield
            jm = component_means(jq)
            den = float(np.linalg.norm(jm))
            sstar = complex(np.vdot(e0v, jm)) / e0sq
            if den < TINY and math.isfinite(den):
                out.degenerate_flux = True
                out.status = "Diverged"
                break
            g = gamma1(jq, scale)
            tot = total_real(np.abs(g) ** 2)
            tot += total_real(np.abs(js) ** 2 * chi)
            res = math.sqrt(tot / npts) / den
            if stop(out, k, sstar, res):
                break
    out.sigma_star = out.history[-1][1] if out.history else sstar
    out.E, out.J = fq, jq
    out.aug = (fq, fs, ft)
    return out


# --------------------------------------------------------------------------
# geometry helpers used to build the BASELINE inputs (geometry.py:85-106)
# --------------------------------------------------------------------------

def centred_box(n: int, side: int, d: int = 2) -> np.ndarray:
    """Centred axis-aligned box of ``side`` voxels on an n^d grid."""
    chi = np.zeros((n,) * d, dtype=bool)
    lo = (n - side) // 2
    chi[tuple(slice(lo, lo + side) for _ in range(d))] = True
    return chi


# --------------------------------------------------------------------------
# public operator surface (spectral_ops.py:96-278, solvers.py:147-204),
# d-generic restatements on (d, *grid) arrays; aug fields are (Q, S, T)
# tuples.  Same numpy operation order as the reference.
# --------------------------------------------------------------------------

def inner(f, g) -> complex:
    """spectral_ops.py:96-99: mean of conj(f).g over all components."""
    return total_complex(np.conj(f) * g) / int(np.prod(f.shape[1:]))


def norm(f) -> float:
    """spectral_ops.py:102-106."""
    return math.sqrt(total_real(np.abs(f) ** 2) / int(np.prod(f.shape[1:])))


def gamma0(f) -> np.ndarray:
    """spectral_ops.py:136-138 (VectorField.mean)."""
    return component_means(f)


def inner_aug(F, G, chi) -> complex:
    """spectral_ops.py:182-190."""
    total = total_complex(np.conj(F[0]) * G[0])
    total += total_complex((np.conj(F[1]) * G[1] + np.conj(F[2]) * G[2]) * chi)
    return total / chi.size


def norm_aug(F, chi) -> float:
    """spectral_ops.py:193-200."""
    total = total_real(np.abs(F[0]) ** 2)
    total += total_real((np.abs(F[1]) ** 2 + np.abs(F[2]) ** 2) * chi)
    return math.sqrt(total / chi.size)


def off_support(F, chi) -> bool:
    """spectral_ops.py:176-179: S or T nonzero on a phase-2 voxel."""
    outside = ~chi
    return bool(np.any(F[1][:, outside]) or np.any(F[2][:, outside]))


def gamma1_aug(F, chi, scale: float = 1.0):
    """spectral_ops.py:208-212: (Gamma_1 Q, S, 0); raises on off-support data."""
    if off_support(F, chi):
        raise ValueError("S/T slots carry data on phase-2 pixels")
    return gamma1(F[0], scale), F[1].copy(), np.zeros_like(F[1])


def _chi_aug(F, p, chi):
    """spectral_ops.py:215-224."""
    u = p[0] * F[0] + p[1] * F[1] + p[2] * F[2]
    u = np.where(chi, u, 0.0)
    return p[0] * u, p[1] * u, p[2] * u


def apply_chi_aug(F, p, chi):
    """spectral_ops.py:227-237."""
    return _chi_aug(F, p, chi)


def apply_local_A(F, t, p, chi):
    """spectral_ops.py:240-250 (same algebra as apply_A, reference op order)."""
    qo, so, to = _chi_aug(F, p, chi)
    tm1 = complex(t) - 1.0
    return (tm1 * qo + F[0], np.where(chi, tm1 * so + F[1], 0.0), np.where(chi, tm1 * to + F[2], 0.0))


def invert_shifted_A(F, t, sigma0, p, chi):
    """spectral_ops.py:253-278 (the singular-shift checks are the caller's)."""
    tt, s0 = complex(t), complex(sigma0)
    qo, so, to = _chi_aug(F, p, chi)
    c = (tt - 1.0) / (tt + s0)
    scale = 1.0 / (1.0 + s0)
    return (scale * (F[0] - c * qo), np.where(chi, scale * (F[1] - c * so), 0.0),
            np.where(chi, scale * (F[2] - c * to), 0.0))


def extract_sigma_star(e, chi, sigma1, e0) -> complex:
    """solvers.py:147-155."""
    e0v = np.array([complex(x) for x in e0])
    sigma = np.where(chi, complex(sigma1), 1.0 + 0j)
    jmean = component_means(sigma * e)
    return complex(np.vdot(e0v, jmean)) / np.vdot(e0v, e0v).real


def extract_sigma_star_aug(F, t, p, chi, e0) -> complex:
    """solvers.py:158-171."""
    e0v = np.array([complex(x) for x in e0])
    flux = apply_local_A(F, t, p, chi)
    return complex(np.vdot(e0v, component_means(flux[0]))) / np.vdot(e0v, e0v).real


def equilibrium_residual(j, scale: float = 1.0) -> float:
    """solvers.py:187-192."""
    den = float(np.linalg.norm(component_means(j)))
    return norm(gamma1(j, scale)) / den


def equilibrium_residual_aug(J, chi, scale: float = 1.0) -> float:
    """solvers.py:195-204."""
    den = float(np.linalg.norm(component_means(J[0])))
    g = gamma1(J[0], scale)
    total = total_real(np.abs(g) ** 2) + total_real(np.abs(J[1]) ** 2 * chi)
    return math.sqrt(total / chi.size) / den
