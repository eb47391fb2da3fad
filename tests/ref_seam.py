"""The INTEGRATION.md binding, as a maintainer would add it to the reference
-- TEST INFRASTRUCTURE (drop-in proof from the reference's side).

``install(fftcond)`` replaces the reference's seam, the private loops
``fftcond.solvers._solve_h`` / ``_solve_aug`` (reference solvers.py:280,
:366, reached through ``_DISPATCH`` :481-491), with calls into the C ABI's
host-buffer entry point ``fftc_solve_host`` (include/fftcond_b200.h) through
ctypes -- numpy only, no torch.  Everything above the seam stays the
reference's own code: ``SolverConfig`` validation, ``_reference_h`` /
``_reference_aug`` (which raise exactly as before), ``map_t`` / ``solve_p``,
and the result containers it builds.  ``tests/test_gpu_refsuite.py`` runs
the reference's own test files through this seam.
"""

from __future__ import annotations

import ctypes as C
import os

import numpy as np

LIB = os.environ.get("FFTC_LIB") or os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))),
                                                 "paper_2001_08289_b200", "libfftcond_b200.so")
_lib = None


class _Problem(C.Structure):
    _fields_ = [("d", C.c_int32), ("reserved", C.c_int32), ("n", C.c_int64 * 3), ("chi", C.c_void_p)]


class _Params(C.Structure):
    _fields_ = [("scheme", C.c_int32), ("reserved", C.c_int32), ("sigma1", C.c_double * 2),
                ("sigma0", C.c_double * 2), ("t", C.c_double * 2), ("p1", C.c_double * 2),
                ("p2", C.c_double * 2), ("p3", C.c_double * 2), ("e0", (C.c_double * 2) * 3),
                ("tol", C.c_double), ("max_iters", C.c_int64), ("gamma1_scale", C.c_double)]


class _Result(C.Structure):
    _fields_ = [("status", C.c_int32), ("degenerate_flux", C.c_int32), ("iterations", C.c_int64),
                ("sigma_star", C.c_double * 2), ("mean_E", (C.c_double * 2) * 3),
                ("mean_J", (C.c_double * 2) * 3), ("kernel_launches", C.c_int64),
                ("device_ms", C.c_double)]


def lib():
    global _lib
    if _lib is None:
        _lib = C.CDLL(LIB)
        _lib.fftc_last_error.restype = C.c_char_p
        _lib.fftc_solve_host.argtypes = [C.c_void_p, C.c_void_p, C.c_void_p, C.c_int64, C.c_void_p, C.c_void_p,
                                         C.c_void_p, C.c_void_p]
    return _lib


def install(fc):
    """Patch the reference package object ``fc`` (``import fftcond``) in place."""
    solvers, spectral_ops = fc.solvers, fc.spectral_ops
    status_of = {0: solvers.TerminationStatus.CONVERGED, 1: solvers.TerminationStatus.MAX_ITERS,
                 2: solvers.TerminationStatus.DIVERGED}

    def _solve_device(pmap, cfg, scheme_code, sigma0, t=1.0, p=(0, 0, 0)):
        chi = np.ascontiguousarray(pmap.chi, dtype=np.uint8)
        ny, nx = chi.shape
        pb = _Problem(d=2, n=(C.c_int64 * 3)(nx, ny, 1), chi=chi.ctypes.data)
        pr = _Params(scheme=scheme_code, tol=cfg.tol, max_iters=cfg.max_iters,
                     gamma1_scale=spectral_ops._gamma1_scale)
        for name, z in (("sigma1", cfg.sigma1), ("sigma0", sigma0), ("t", t), ("p1", p[0]), ("p2", p[1]),
                        ("p3", p[2])):
            getattr(pr, name)[:] = (complex(z).real, complex(z).imag)
        for c, z in enumerate(cfg.e0_vector()):
            pr.e0[c][:] = (z.real, z.imag)
        hist = np.empty((cfg.max_iters, 3))
        aug = np.empty((3, 2, ny, nx), np.complex128) if scheme_code >= 2 else None
        E = None if aug is not None else np.empty((2, ny, nx), np.complex128)  # substituted: E is aug's Q
        J = np.empty((2, ny, nx), np.complex128)
        res = _Result()
        rc = lib().fftc_solve_host(C.byref(pb), C.byref(pr), hist.ctypes.data, hist.shape[0],
                                   None if E is None else E.ctypes.data, J.ctypes.data,
                                   None if aug is None else aug.ctypes.data, C.byref(res))
        if rc:
            raise RuntimeError(lib().fftc_last_error().decode())
        history = solvers.ConvergenceHistory()
        for k in range(int(res.iterations)):
            history.append(k + 1, complex(hist[k, 0], hist[k, 1]), float(hist[k, 2]))
        VF = spectral_ops.VectorField
        aug_field = None
        if aug is not None:
            E = aug[0]
            aug_field = spectral_ops.AugmentedField(VF(aug[0]), VF(aug[1]), VF(aug[2]))
        return solvers.SolveResult(sigma_star=complex(res.sigma_star[0], res.sigma_star[1]), E_field=VF(E),
                                   J_field=VF(J), history=history, status=status_of[int(res.status)],
                                   degenerate_flux=bool(res.degenerate_flux), aug_field=aug_field)

    def _solve_h(pmap, cfg, accelerated):
        sigma0 = solvers._reference_h(cfg, accelerated)  # unchanged: raises as before
        return _solve_device(pmap, cfg, 1 if accelerated else 0, sigma0)

    def _solve_aug(pmap, cfg, accelerated):
        t = fc.transform.map_t(complex(cfg.sigma1), cfg.interval)
        params = fc.transform.solve_p(cfg.interval)
        sigma0 = solvers._reference_aug(cfg, t, accelerated)  # unchanged
        return _solve_device(pmap, cfg, 3 if accelerated else 2, sigma0, t, (params.p1, params.p2, params.p3))

    solvers._solve_h = _solve_h
    solvers._solve_aug = _solve_aug
    return fc
