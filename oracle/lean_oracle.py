"""Memory-lean, threaded form of the CPU oracle -- TEST INFRASTRUCTURE ONLY.

Same contract as ``oracle/fftcond_oracle.py`` (the checker, never the
product; only ``tests/``, ``smoke()`` and ``bench.py``'s CPU legs may use
it).  It exists because the plain restatement holds ~18 full d-vector
fields per augmented iteration: 115 GB at 512^3 and ~900 GB at 1024^3,
beyond both the dev container (62 GB) and the GPU box host (196 GB).

What changes is only WHERE values live, never HOW they are computed:

* fields are lists of per-component arrays; every pointwise operation of
  the reference loop (solvers.py:280-331, :366-443) is applied to one
  spatial component at a time with the same numpy expression, operand
  order and broadcast shapes as ``fftcond_oracle`` -- the augmented
  operator A (solvers.py:355-363) never mixes spatial components, so this
  is the same arithmetic element by element;
* J_raw = A(F_raw) is recomputed from F_raw when it is needed again instead
  of being stored (A is pointwise and deterministic);
* the d-dimensional FFT is the same sequence of 1-D numpy transforms numpy's
  ``_raw_fftnd`` performs (last axis first), each split over threads along
  an axis it does not transform (a line's transform does not depend on the
  other lines), written into preallocated buffers;
* reductions collect the per-row sums of every component and combine them
  with one ``math.fsum`` (exactly rounded, so the order of the rows does
  not matter), as ``total_real`` does (spectral_ops.py:33-55).

``tests/test_oracle.py`` pins this module bit for bit against
``fftcond_oracle.solve`` (histories, sigma*, <E>, <J>) on 2-D and 3-D cells.
"""

from __future__ import annotations

import math
import os
from concurrent.futures import ThreadPoolExecutor

import numpy as np

from . import fftcond_oracle as O

_POOL = None


def _pool(nthreads: int):
    global _POOL
    if _POOL is None or _POOL._max_workers != nthreads:
        _POOL = ThreadPoolExecutor(nthreads)
    return _POOL


def _nthreads() -> int:
    return int(os.environ.get("FFTC_ORACLE_THREADS", str(os.cpu_count() or 1)))


def _fft_axis(x: np.ndarray, out: np.ndarray, axis: int, inverse: bool):
    """out = numpy 1-D (i)fft of x along ``axis``, lines split over threads."""
    nd = x.ndim
    split = 0 if axis != 0 else 1
    n = x.shape[split]
    nt = max(1, min(_nthreads(), n))
    f = np.fft.ifft if inverse else np.fft.fft
    bounds = [(i * n // nt, (i + 1) * n // nt) for i in range(nt)]

    def job(b):
        sl = [slice(None)] * nd
        sl[split] = slice(*b)
        sl = tuple(sl)
        f(x[sl], axis=axis, out=out[sl])

    list(_pool(nt).map(job, bounds))


def fftn_(x: np.ndarray, inverse: bool, scratch: np.ndarray) -> np.ndarray:
    """numpy.fft.fftn / ifftn of one component over all its axes (x first,
    as numpy's _raw_fftnd does).  Uses ``scratch`` (same shape, complex128);
    the result lands in x or scratch, whichever is returned."""
    src, dst = x, scratch
    for axis in reversed(range(x.ndim)):
        _fft_axis(src, dst, axis, inverse)
        src, dst = dst, src
    return src


def _row_sums(values: np.ndarray) -> np.ndarray:
    return np.sum(values.reshape(-1, values.shape[-1]), axis=-1)


def _combine(rows: list) -> float:
    """total_real over the concatenation of several row-sum vectors."""
    allrows = np.concatenate(rows)
    if not np.all(np.isfinite(allrows)):
        return float(np.sum(allrows))
    return math.fsum(allrows.tolist())


def _mean_c(x: np.ndarray) -> complex:
    return O.total_complex(x) / x.size


def gamma1_(comps: list, scale: float = 1.0) -> list:
    """fftcond_oracle.gamma1 on a list of d component arrays (consumed: the
    transforms run in their storage).  Returns the d projected components.
    In-place ufunc forms of the same operations (add and the k-multiplies are
    the same IEEE operations on the same operands)."""
    d = len(comps)
    grid = comps[0].shape
    ks, inv = O.wave_vectors(grid)
    scratch = np.empty(grid, dtype=np.complex128)
    fh = []
    for c in range(d):
        r = fftn_(comps[c], False, scratch)
        if r is scratch:
            scratch = comps[c]
        fh.append(r)
    dot = ks[0] * fh[0]
    for c in range(1, d):
        np.multiply(ks[c], fh[c], out=scratch)
        np.add(dot, scratch, out=dot)  # dot = dot + ks[c] * fh[c]
    np.multiply(dot, inv if scale == 1.0 else inv * scale, out=dot)  # inv * 1.0 == inv
    out = []
    for c in range(d):
        np.multiply(ks[c], dot, out=fh[c])  # out[c] = ks[c] * dot
        r = fftn_(fh[c], True, scratch)
        if r is scratch:
            scratch = fh[c]
        out.append(r)
    return out


def solve(chi: np.ndarray, scheme: str, sigma1: complex, *, e0=None, tol: float = 1e-8,
          max_iters: int = 1000, alpha: float | None = None, beta: float | None = None,
          gamma1_scale: float = 1.0, keep_fields: bool = True) -> O.OracleResult:
    """``fftcond_oracle.solve`` for the schemes the 3-D configs use (basic,
    em_sub), in bounded memory.  Fields come back as (d, *grid) arrays when
    ``keep_fields`` (E = e or Q, J = j or Jq, aug = (Q, S, T))."""
    chi = np.asarray(chi, dtype=bool)
    d = chi.ndim
    if e0 is None:
        e0 = (1.0,) + (0.0,) * (d - 1)
    if scheme == "basic":
        return _loop_basic(chi, complex(sigma1), e0, tol, max_iters, gamma1_scale, keep_fields)
    if scheme == "em_sub":
        return _loop_em_sub(chi, complex(sigma1), e0, tol, max_iters, alpha, beta, gamma1_scale, keep_fields)
    raise ValueError(f"lean oracle covers basic and em_sub, not {scheme!r}")


def _e0(e0, grid):
    """e0 vector, |e0|^2 and the broadcast field, one full array per component
    (fftcond_oracle._applied)."""
    e0v = np.array([complex(v) for v in e0], dtype=np.complex128)
    return e0v, np.vdot(e0v, e0v).real, [np.full(grid, e0v[c], dtype=np.complex128) for c in range(len(e0v))]


def _loop_basic(chi, sigma1, e0, tol, max_iters, scale, keep):
    """fftcond_oracle._loop_h(accelerated=False), solvers.py:280-331."""
    s0 = O.reference_sigma0("basic", sigma1, None)
    grid = chi.shape
    npts = chi.size
    d = chi.ndim
    sig = np.where(chi, sigma1, 1.0 + 0j)
    e0v, e0sq, e0f = _e0(e0, grid)
    out = O.OracleResult()
    stop = O._Stop(tol)
    e = [x.copy() for x in e0f]  # holds e_raw, then e (pinned) in place
    del e0f
    g = None
    sstar = 0j
    with np.errstate(over="ignore", invalid="ignore"):
        for k in range(1, max_iters + 1):
            if k > 1:
                for c in range(d):  # e_raw = e - g / s0
                    g[c] = g[c] / s0
                    np.subtract(e[c], g[c], out=e[c])
                g = j = None
            delta = e0v - np.array([_mean_c(x) for x in e])
            for c in range(d):
                e[c] += delta[c]  # e = e_raw + delta (broadcast add, same values)
            j = [sig * e[c] for c in range(d)]
            jm = np.array([_mean_c(x) for x in j])
            den = float(np.linalg.norm(jm))
            sstar = complex(np.vdot(e0v, jm)) / e0sq
            if den < O.TINY and math.isfinite(den):
                out.degenerate_flux = True
                out.status = "Diverged"
                break
            jj = [x.copy() for x in j] if keep else j
            g = gamma1_(jj, scale)
            res = math.sqrt(_combine([_row_sums(np.abs(x) ** 2) for x in g]) / npts) / den
            if stop(out, k, sstar, res):
                break
    out.sigma_star = out.history[-1][1] if out.history else sstar
    if keep:
        out.E = np.stack(e)
        out.J = np.stack(j)
    return out


def _apply_A_c(q, s, tt, t, p, chi):
    """fftcond_oracle.apply_A restricted to one spatial component."""
    p1, p2, p3 = p
    u = np.where(chi, p1 * q + p2 * s + p3 * tt, 0.0)
    tm1 = t - 1.0
    return (tm1 * p1 * u + q, np.where(chi, tm1 * p2 * u + s, 0.0), np.where(chi, tm1 * p3 * u + tt, 0.0))


def _loop_em_sub(chi, sigma1, e0, tol, max_iters, alpha, beta, scale, keep):
    """fftcond_oracle._loop_aug(accelerated=True), solvers.py:366-443."""
    t = O.map_t(sigma1, alpha, beta)
    p = O.solve_p(alpha, beta)
    p1, p2, p3 = p
    s0 = O.reference_sigma0("em_sub", sigma1, t)
    grid = chi.shape
    npts = chi.size
    d = chi.ndim
    e0v, e0sq, e0f = _e0(e0, grid)
    chif = chi.astype(np.float64)
    out = O.OracleResult()
    stop = O._Stop(tol)
    zero = np.zeros(grid, dtype=np.complex128)
    fq = [x.copy() for x in e0f]
    fs = [zero.copy() for _ in range(d)]
    ft = [zero.copy() for _ in range(d)]
    inv_scale = 1.0 / (1.0 + s0)
    inv_c = (t - 1.0) / (t + s0)
    tau = (t - 1.0) * p1 * chif
    del chif
    sstar = 0j
    jq = None
    with np.errstate(over="ignore", invalid="ignore"):
        for k in range(1, max_iters + 1):
            if k == 1:
                # W = A(raw) + s0 raw (solvers.py:386-387), component by component
                for c in range(d):
                    aq, as_, at = _apply_A_c(fq[c], fs[c], ft[c], t, p, chi)
                    wq, ws, wt = aq + s0 * fq[c], as_ + s0 * fs[c], at + s0 * ft[c]
                    u = np.where(chi, p1 * wq + p2 * ws + p3 * wt, 0.0)
                    fq[c] = inv_scale * (wq - inv_c * p1 * u)
                    fs[c] = np.where(chi, inv_scale * (ws - inv_c * p2 * u), 0.0)
                    ft[c] = np.where(chi, inv_scale * (wt - inv_c * p3 * u), 0.0)
            else:
                # R = J_raw - s0 F_raw with J_raw = A(F_raw) recomputed
                rq = []
                for c in range(d):
                    jqc = _apply_A_c(fq[c], fs[c], ft[c], t, p, chi)[0]
                    rq.append(jqc - s0 * fq[c])
                g = gamma1_(rq, scale)
                del rq
                for c in range(d):
                    jqc, jsc, jtc = _apply_A_c(fq[c], fs[c], ft[c], t, p, chi)
                    rqc = jqc - s0 * fq[c]  # recomputed: same operands, same value
                    rs = jsc - s0 * fs[c]
                    rt = jtc - s0 * ft[c]
                    wq = 2.0 * s0 * e0f[c] - 2.0 * g[c] + rqc
                    ws = -rs
                    wt = rt
                    u = np.where(chi, p1 * wq + p2 * ws + p3 * wt, 0.0)
                    fq[c] = inv_scale * (wq - inv_c * p1 * u)
                    fs[c] = np.where(chi, inv_scale * (ws - inv_c * p2 * u), 0.0)
                    ft[c] = np.where(chi, inv_scale * (wt - inv_c * p3 * u), 0.0)
                del g
            delta = e0v - np.array([_mean_c(x) for x in fq])
            bshape = (1,) * len(grid)
            jq, js_rows = [], []
            for c in range(d):
                jqc, jsc, _ = _apply_A_c(fq[c], fs[c], ft[c], t, p, chi)
                dfc = delta[c:c + 1].reshape(bshape)
                jq.append(jqc + p1 * tau * dfc + dfc)
                jsd = jsc + p2 * tau * dfc
                js_rows.append(_row_sums(np.abs(jsd) ** 2 * chi))
                del jsd
            jm = np.array([_mean_c(x) for x in jq])
            den = float(np.linalg.norm(jm))
            sstar = complex(np.vdot(e0v, jm)) / e0sq
            if den < O.TINY and math.isfinite(den):
                out.degenerate_flux = True
                out.status = "Diverged"
                break
            jq_in = [x.copy() for x in jq] if keep else jq
            g = gamma1_(jq_in, scale)
            tot = _combine([_row_sums(np.abs(x) ** 2) for x in g])
            tot += _combine(js_rows)
            del g, jq_in
            res = math.sqrt(tot / npts) / den
            if stop(out, k, sstar, res):
                break
    out.sigma_star = out.history[-1][1] if out.history else sstar
    if keep:
        delta = e0v - np.array([_mean_c(x) for x in fq])
        bshape = (1,) * len(grid)
        Q = np.stack([fq[c] + delta[c:c + 1].reshape(bshape) for c in range(d)])
        out.E = Q
        out.J = np.stack(jq) if jq is not None else None
        out.aug = (Q, np.stack(fs), np.stack(ft))
    return out
