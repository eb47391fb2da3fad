"""Public operator surface on the GPU: the reference's ``spectral_ops``
functions and the field-level helpers of ``solvers``, with the same names,
arguments, return types and exceptions, computed by this package's CUDA
kernels (``fftc_gamma1``, ``fftc_aug_apply``, ``fftc_apply_sigma``,
``fftc_reduce`` in include/fftcond_b200.h).

Reference functions mirrored (fftcond/spectral_ops.py, fftcond/solvers.py):

    inner, norm                     spectral_ops.py:96-106
    gamma1, gamma0                  spectral_ops.py:131-138 (Gamma_1 of :120-128)
    inner_aug, norm_aug             spectral_ops.py:182-200
    gamma0_aug, gamma1_aug          spectral_ops.py:203-212
    apply_chi_aug                   spectral_ops.py:227-237
    apply_local_A                   spectral_ops.py:240-250
    invert_shifted_A                spectral_ops.py:253-278
    extract_sigma_star(_aug)        solvers.py:147-171
    recover_physical_fields         solvers.py:174-184
    equilibrium_residual(_aug)      solvers.py:187-204

Fields may be host (numpy) or device resident; operators return fields that
stay on the device (read ``.data`` to copy to the host).  Reductions are
fixed-order device trees: deterministic, and equal to the reference's
compensated sums to rounding.  d = 2 as in the reference, and d = 3.
There is no CPU fallback: without the CUDA library these raise.
"""

from __future__ import annotations

import ctypes as C
import math

import numpy as np

from . import fields as _fields
from . import native
from .cell import PhaseMap
from .exceptions import BackendError, ContractError, DegenerateParamError, SupportError
from .fields import AugmentedField, VectorField
from .scalars import SubstitutionParams

_TINY = 1e-300  # solvers.py:51


# -- plumbing -------------------------------------------------------------------
def _torch():
    import torch

    if not torch.cuda.is_available():
        raise BackendError("the operator API runs on the GPU; no CUDA device is visible")
    return torch


def _stream(torch):
    return torch.cuda.current_stream().cuda_stream


def _dev(f: VectorField):
    """Device tensor of a field (uploads host data; does not alias it)."""
    torch = _torch()
    t = f.device_tensor
    if t is None:
        t = torch.from_numpy(np.ascontiguousarray(f.data, dtype=np.complex128)).to("cuda")
    elif t.dtype != torch.complex128 or not t.is_contiguous() or t.device.type != "cuda":
        t = t.to(device="cuda", dtype=torch.complex128).contiguous()
    return t


def _problem(grid, pmap: PhaseMap | None = None) -> native.Problem:
    grid = tuple(int(n) for n in grid)
    if len(grid) not in (2, 3):
        raise ContractError(f"fields must be 2-D or 3-D, got grid {grid}")
    p = native.Problem()
    p.d = len(grid)
    p.n[0] = grid[-1]
    p.n[1] = grid[-2]
    p.n[2] = grid[0] if len(grid) == 3 else 1
    if pmap is not None:
        if tuple(pmap.grid) != grid:
            raise ContractError(f"phase map grid {pmap.grid} does not match field grid {grid}")
        from .solver import _device_chi

        p.chi = _device_chi(pmap, _torch()).data_ptr()
    return p


def _check(rc, what):
    if rc:
        raise BackendError(f"{what} failed ({rc}): {native.last_error()}")


def _reduce(op, grid, a, b=None, *, pmap=None, mask=False):
    torch = _torch()
    prob = _problem(grid, pmap)
    d = len(grid)
    out = np.zeros(2 * d if op == native.FFTC_RED_SUM else 2)
    rc = native.lib().fftc_reduce(C.byref(prob), op, native.FFTC_MASK_CHI if mask else native.FFTC_MASK_NONE,
                                  a.data_ptr(), None if b is None else b.data_ptr(), out.ctypes.data,
                                  _stream(torch))
    _check(rc, "fftc_reduce")
    return out


def _npix(grid) -> int:
    return int(np.prod(grid))


def _sum_vec(t, grid) -> np.ndarray:
    s = _reduce(native.FFTC_RED_SUM, grid, t)
    return np.array([complex(s[2 * c], s[2 * c + 1]) for c in range(len(grid))])


def _dot(a, b, grid, pmap=None, mask=False) -> complex:
    s = _reduce(native.FFTC_RED_DOT, grid, a, b, pmap=pmap, mask=mask)
    return complex(s[0], s[1])


def _norm2(a, grid, pmap=None, mask=False) -> float:
    return float(_reduce(native.FFTC_RED_NORM2, grid, a, pmap=pmap, mask=mask)[0])


def _grid(f: VectorField) -> tuple:
    return tuple(f.grid_shape)


# -- spectral_ops.py ------------------------------------------------------------
def inner(f: VectorField, g: VectorField) -> complex:
    """Mean over pixels of conj(f) . g (spectral_ops.py:96-99)."""
    grid = _grid(f)
    return _dot(_dev(f), _dev(g), grid) / _npix(grid)


def norm(f: VectorField) -> float:
    """Norm induced by :func:`inner` (spectral_ops.py:102-106)."""
    grid = _grid(f)
    return math.sqrt(_norm2(_dev(f), grid) / _npix(grid))


def gamma1(f: VectorField) -> VectorField:
    """Projection onto zero-mean curl-free fields (spectral_ops.py:131-133)."""
    from .operators import gamma1 as _g1

    return VectorField.from_device(_g1(_dev(f), scale=_fields._gamma1_scale))


def gamma0(f: VectorField) -> np.ndarray:
    """Projection onto constants: the pixel mean (spectral_ops.py:136-138)."""
    grid = _grid(f)
    return _sum_vec(_dev(f), grid) / _npix(grid)


def _check_support(f: AugmentedField, pmap: PhaseMap):
    """spectral_ops.py:176-179, counted on the device."""
    grid = _grid(f.Q)
    n = _reduce(native.FFTC_RED_OFF_SUPPORT, grid, _dev(f.S), _dev(f.T), pmap=pmap)[0]
    if n > 0:
        raise SupportError("S/T slots carry data on phase-2 pixels")


def inner_aug(f: AugmentedField, g: AugmentedField, pmap: PhaseMap) -> complex:
    """Mean of conj(Q).Q' + [conj(S).S' + conj(T).T'] chi (spectral_ops.py:182-190)."""
    grid = _grid(f.Q)
    total = _dot(_dev(f.Q), _dev(g.Q), grid)
    total += _dot(_dev(f.S), _dev(g.S), grid, pmap, True) + _dot(_dev(f.T), _dev(g.T), grid, pmap, True)
    return total / _npix(grid)


def norm_aug(f: AugmentedField, pmap: PhaseMap) -> float:
    """spectral_ops.py:193-200."""
    grid = _grid(f.Q)
    total = _norm2(_dev(f.Q), grid)
    total += _norm2(_dev(f.S), grid, pmap, True) + _norm2(_dev(f.T), grid, pmap, True)
    return math.sqrt(total / _npix(grid))


def gamma0_aug(f: AugmentedField) -> np.ndarray:
    """Mean of the Q slot (spectral_ops.py:203-205)."""
    return gamma0(f.Q)


def _zeros_like(t):
    return _torch().zeros_like(t)


def gamma1_aug(f: AugmentedField, pmap: PhaseMap) -> AugmentedField:
    """(gamma1 Q, S, 0) (spectral_ops.py:208-212)."""
    _check_support(f, pmap)
    s = _dev(f.S).clone()
    return AugmentedField(gamma1(f.Q), VectorField.from_device(s), VectorField.from_device(_zeros_like(s)))


def _coef(params: SubstitutionParams, t: complex = 1.0, sigma0: complex = 0.0) -> np.ndarray:
    vals = [params.p1, params.p2, params.p3, complex(t), complex(sigma0)]
    return np.array([x for z in vals for x in (complex(z).real, complex(z).imag)], dtype=np.float64)


def _aug_apply(op, f: AugmentedField, pmap: PhaseMap, coef: np.ndarray) -> AugmentedField:
    torch = _torch()
    grid = _grid(f.Q)
    prob = _problem(grid, pmap)
    q, s, t = _dev(f.Q), _dev(f.S), _dev(f.T)
    qo, so, to = torch.empty_like(q), torch.empty_like(q), torch.empty_like(q)
    rc = native.lib().fftc_aug_apply(C.byref(prob), op, coef.ctypes.data, q.data_ptr(), s.data_ptr(), t.data_ptr(),
                                     qo.data_ptr(), so.data_ptr(), to.data_ptr(), _stream(torch))
    _check(rc, "fftc_aug_apply")
    return AugmentedField(VectorField.from_device(qo), VectorField.from_device(so), VectorField.from_device(to))


def apply_chi_aug(f: AugmentedField, params: SubstitutionParams, pmap: PhaseMap) -> AugmentedField:
    """Rank-one slot mixer p (x) p on phase-1 pixels (spectral_ops.py:227-237)."""
    return _aug_apply(native.FFTC_AUG_CHI, f, pmap, _coef(params))


def apply_local_A(f: AugmentedField, t: complex, params: SubstitutionParams, pmap: PhaseMap) -> AugmentedField:
    """A = (t - 1) chi'' + I (spectral_ops.py:240-250)."""
    return _aug_apply(native.FFTC_AUG_LOCAL_A, f, pmap, _coef(params, t))


def invert_shifted_A(f: AugmentedField, t: complex, sigma0: complex, params: SubstitutionParams,
                     pmap: PhaseMap) -> AugmentedField:
    """Pixel-local closed-form inverse of (A + sigma0 I) (spectral_ops.py:253-278)."""
    tt, s0 = complex(t), complex(sigma0)
    if 1.0 + s0 == 0:
        raise DegenerateParamError("shift sigma0 = -1 makes A + sigma0 I singular")
    if tt + s0 == 0:
        raise DegenerateParamError("shift sigma0 = -t makes A + sigma0 I singular")
    return _aug_apply(native.FFTC_AUG_INV_SHIFTED, f, pmap, _coef(params, tt, s0))


# -- solvers.py field helpers ------------------------------------------------------
def _e0_vector(e0, d: int) -> np.ndarray:
    if e0 is None:
        e0 = (1.0,) + (0.0,) * (d - 1)
    v = np.array([complex(x) for x in e0])
    if v.shape != (d,):
        raise ContractError(f"applied field e0 must have {d} components, got {len(v)}")
    return v


def _sigma_star(e0v: np.ndarray, jmean: np.ndarray) -> complex:
    e0sq = np.vdot(e0v, e0v).real
    if e0sq == 0:
        raise ContractError("applied field e0 must be nonzero")
    return complex(np.vdot(e0v, jmean)) / e0sq


def extract_sigma_star(e: VectorField, pmap: PhaseMap, sigma1: complex, e0=None) -> complex:
    """Effective conductivity along e0 from an electric field iterate (solvers.py:147-155)."""
    torch = _torch()
    grid = _grid(e)
    e0v = _e0_vector(e0, len(grid))
    if np.vdot(e0v, e0v).real == 0:
        raise ContractError("applied field e0 must be nonzero")
    prob = _problem(grid, pmap)
    src = _dev(e)
    j = torch.empty_like(src)
    s1 = np.array([complex(sigma1).real, complex(sigma1).imag])
    _check(native.lib().fftc_apply_sigma(C.byref(prob), s1.ctypes.data, src.data_ptr(), j.data_ptr(), _stream(torch)),
           "fftc_apply_sigma")
    return _sigma_star(e0v, _sum_vec(j, grid) / _npix(grid))


def extract_sigma_star_aug(f: AugmentedField, t: complex, params: SubstitutionParams, pmap: PhaseMap,
                           e0=None) -> complex:
    """Effective conductivity from an augmented iterate (solvers.py:158-171)."""
    e0v = _e0_vector(e0, len(_grid(f.Q)))
    if np.vdot(e0v, e0v).real == 0:
        raise ContractError("applied field e0 must be nonzero")
    flux = apply_local_A(f, t, params, pmap)
    return _sigma_star(e0v, gamma0(flux.Q))


def recover_physical_fields(f: AugmentedField, t: complex, params: SubstitutionParams,
                            pmap: PhaseMap) -> tuple[VectorField, VectorField]:
    """(E, J) = (Q, (A F)_Q) of an augmented solution (solvers.py:174-184)."""
    flux = apply_local_A(f, t, params, pmap)
    return VectorField.from_device(_dev(f.Q).clone()), flux.Q


def equilibrium_residual(j: VectorField) -> float:
    """||Gamma_1 j|| / ||<j>|| (solvers.py:187-192)."""
    den = float(np.linalg.norm(gamma0(j)))
    if den < _TINY:
        raise ContractError("mean flux vanishes; residual is undefined")
    return norm(gamma1(j)) / den


def equilibrium_residual_aug(jaug: AugmentedField, pmap: PhaseMap) -> float:
    """Augmented analogue: sqrt((sum|Gamma_1 Q|^2 + sum|S|^2 chi)/N) / ||<Q>|| (solvers.py:195-204)."""
    den = float(np.linalg.norm(gamma0_aug(jaug)))
    if den < _TINY:
        raise ContractError("mean flux vanishes; residual is undefined")
    grid = _grid(jaug.Q)
    g = _dev(gamma1(jaug.Q))
    total = _norm2(g, grid) + _norm2(_dev(jaug.S), grid, pmap, True)
    return math.sqrt(total / _npix(grid)) / den
