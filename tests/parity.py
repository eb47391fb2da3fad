"""Parity protocol shared by the GPU tests.

For one device result ``r`` (a SolveResult) and one golden fixture ``g``:

1. status, iteration count and degenerate flag equal;
2. sigma* within REL relative (1e-10, BASELINE.json north_star tolerance);
3. ||d<J>|| / ||<J>|| <= REL;
4. ||d<E>|| / ||<E>|| <= REL on Converged runs only (on exploding MaxIters
   runs <E> is e0 recovered from O(1e30) iterates: catastrophic
   cancellation);
5. sigma*_k within REL relative at every recorded k;
6. residual_k within RES_REL relative plus RES_ABS absolute (the residual is
   the quantity most sensitive to FFT roundoff; 2.3e-5 worst relative
   difference measured across FFT libraries, and an absolute floor of a few
   1e-16 x contrast once res approaches 1e-13);
7. a stop decided within TIE of the tolerance is a declared tie, not a failure.
"""

from __future__ import annotations

import math

import numpy as np

REL = 1e-10
RES_REL = 1e-4
# residuals are normalised by |<j>|; FFT roundoff adds an absolute error of
# order eps * |j| / |<j>|, i.e. ~1e-16 times the contrast max(1, |sigma1|)
# (measured: the CUDA transforms are as accurate as pocketfft, rms error
# ratio 0.98-1.03 against a long-double reference, profiles/fft_accuracy.txt)
RES_ABS = 1e-14
TIE = 1e-4


def _rel(a, b):
    a, b = complex(a), complex(b)
    den = max(abs(b), 1e-300)
    return abs(a - b) / den


def _vec_rel(a, b):
    a = np.asarray(a, dtype=complex)
    b = np.asarray(b, dtype=complex)
    den = max(float(np.linalg.norm(b)), 1e-300)
    return float(np.linalg.norm(a - b)) / den


def golden_means(g):
    """<E>, <J> of a fixture, or (None, None) for history-only fixtures (the
    first iterations at 512^3 / 1024^3 keep no fields)."""
    if "mean_E" not in g:
        return None, None
    mE = np.array([complex(*v) for v in g["mean_E"]])
    mJ = np.array([complex(*v) for v in g["mean_J"]])
    return mE, mJ


def is_tie(g) -> bool:
    """Stopping margin of the golden below TIE (either side of tol)."""
    h = g["history"]
    tol = g["case"]["tol"]
    if g["status"] != "Converged" or len(h) < 2:
        return False
    k_res, prev_res = h[-1][3], h[-2][3]
    return abs(1.0 - k_res / tol) < TIE or abs(prev_res / tol - 1.0) < TIE


def check(r, g, *, rel=REL, res_rel=RES_REL, fields=True):
    """Assert parity of SolveResult r against golden g; returns a report dict."""
    name = g["case"]["name"]
    rep = dict(name=name, iters=r.iterations, golden_iters=g["iterations"])
    if is_tie(g) and (r.status.value != g["status"] or r.iterations != g["iterations"]):
        rep["tie"] = True
        return rep
    assert r.status.value == g["status"], f"{name}: status {r.status.value} != {g['status']}"
    assert r.iterations == g["iterations"], f"{name}: iterations {r.iterations} != {g['iterations']}"
    assert bool(r.degenerate_flux) == bool(g["degenerate_flux"]), f"{name}: degenerate flag"
    gs = complex(*g["sigma_star"])
    e = _rel(r.sigma_star, gs)
    rep["sigma_rel"] = e
    assert e <= rel, f"{name}: sigma* {r.sigma_star} vs {gs} rel {e:.3e}"
    h = g["history"]
    if len(h):
        dev = np.array([[rec.sigma_star.real, rec.sigma_star.imag, rec.residual] for rec in r.history])
        gsig = h[:, 1] + 1j * h[:, 2]
        dsig = dev[:, 0] + 1j * dev[:, 1]
        srel = np.abs(dsig - gsig) / np.maximum(np.abs(gsig), 1e-300)
        floor = RES_ABS * max(1.0, abs(complex(*g["case"]["sigma1"])))
        rrel = np.abs(dev[:, 2] - h[:, 3]) / (np.abs(h[:, 3]) + floor / res_rel)
        rep["hist_sigma_rel_max"] = float(srel.max())
        rep["hist_res_rel_max"] = float(rrel.max())
        assert srel.max() <= rel, f"{name}: history sigma* rel {srel.max():.3e} at k={int(srel.argmax()) + 1}"
        assert rrel.max() <= res_rel, f"{name}: history residual rel {rrel.max():.3e} at k={int(rrel.argmax()) + 1}"
    mE, mJ = golden_means(g)
    if mJ is not None and r.mean_J is not None and np.all(np.isfinite(mJ)):
        ej = _vec_rel(r.mean_J, mJ)
        rep["meanJ_rel"] = ej
        assert ej <= rel or float(np.linalg.norm(mJ)) == 0.0, f"{name}: <J> rel {ej:.3e}"
    if mE is not None and g["status"] == "Converged" and r.mean_E is not None:
        ee = _vec_rel(r.mean_E, mE)
        rep["meanE_rel"] = ee
        assert ee <= rel, f"{name}: <E> rel {ee:.3e}"
    if len(h) >= 1 and g["status"] == "Converged":
        tol = g["case"]["tol"]
        rep["margin_last"] = 1.0 - h[-1][3] / tol
        if len(h) >= 2:
            rep["margin_prev"] = h[-2][3] / tol - 1.0
    return rep


def field_check(r, path, *, rel=1e-9):
    """Field-level parity against saved golden fields (converged runs)."""
    z = np.load(path)
    out = {}
    for key, fld in (("E", r.E_field), ("J", r.J_field)):
        ref = z[key]
        got = fld.data
        den = math.sqrt(float(np.mean(np.abs(ref) ** 2))) or 1.0
        err = math.sqrt(float(np.mean(np.abs(got - ref) ** 2))) / den
        out[key] = err
        assert err <= rel, f"{path}: field {key} rms rel {err:.3e}"
    if r.aug_field is not None and "S" in z.files:
        for key, fld in (("S", r.aug_field.S), ("T", r.aug_field.T)):
            ref = z[key]
            got = fld.data
            scale = math.sqrt(float(np.mean(np.abs(z["E"]) ** 2))) or 1.0
            err = math.sqrt(float(np.mean(np.abs(got - ref) ** 2))) / scale
            out[key] = err
            assert err <= rel, f"{path}: field {key} rms rel {err:.3e}"
    return out
