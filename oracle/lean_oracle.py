"""Memory-lean, multi-threaded form of the CPU oracle -- TEST INFRASTRUCTURE ONLY.

Same contract as ``oracle/fftcond_oracle.py`` (the checker, never the
product; only ``tests/``, ``smoke()`` and ``bench.py``'s CPU legs may use
it).  It exists because the plain restatement holds ~18 full d-vector
fields per augmented iteration: 115 GB at 512^3 and ~900 GB at 1024^3,
beyond both the dev container (62 GB) and the GPU box host (196 GB), and
because it runs on one core.

What changes is only WHERE values live and WHICH thread computes them,
never HOW they are computed:

* fields are lists of per-component arrays; every pointwise operation of
  the reference loop (solvers.py:280-331, :366-443) is applied to one
  spatial component and one slab of the outermost grid axis at a time,
  with the same numpy expression, operand order and broadcast shapes as
  ``fftcond_oracle`` -- pointwise ops give the same value for a voxel
  whatever else is in the array, and the augmented operator A
  (solvers.py:355-363) never mixes spatial components;
* slabs run on a thread pool (numpy releases the GIL inside its loops);
* J_raw = A(F_raw) is recomputed from F_raw when it is needed again instead
  of being stored (A is pointwise and deterministic);
* the d-dimensional FFT is the same sequence of 1-D numpy transforms numpy's
  ``_raw_fftnd`` performs (last axis first), each split over threads along
  an axis it does not transform (a line's transform does not depend on the
  other lines), written into preallocated buffers;
* reductions collect the per-row sums (rows run along x, inside one slab)
  of every slab and component and combine them with one ``math.fsum``
  (exactly rounded, so the order of the rows does not matter), as
  ``total_real`` does (spectral_ops.py:33-55).

``tests/test_oracle.py::test_lean_oracle_bitwise`` pins this module bit for
bit against ``fftcond_oracle.solve`` (histories, sigma*, fields) on 2-D and
3-D cells.  ``FFTC_ORACLE_THREADS`` caps the threads (default: all CPUs).
"""

from __future__ import annotations

import math
import os
import time
from concurrent.futures import ThreadPoolExecutor

import numpy as np

from . import fftcond_oracle as O

_POOLS: dict = {}


def nthreads() -> int:
    return max(1, int(os.environ.get("FFTC_ORACLE_THREADS", str(os.cpu_count() or 1))))


def _pool(n: int) -> ThreadPoolExecutor:
    if n not in _POOLS:
        _POOLS[n] = ThreadPoolExecutor(n)
    return _POOLS[n]


def _slabs(n: int, parts: int):
    parts = max(1, min(parts, n))
    return [slice(i * n // parts, (i + 1) * n // parts) for i in range(parts)]


def par(n0: int, fn) -> list:
    """fn(slice) over slabs of the outermost axis (length n0), in order, on
    the thread pool.  Slabs are small (16 per thread, at least one plane) so
    the temporaries of the pointwise expressions stay a small multiple of
    threads x slab instead of a multiple of the grid."""
    nt = nthreads()
    sls = _slabs(n0, 16 * nt)
    if nt == 1 or len(sls) == 1:
        return [fn(sl) for sl in sls]
    return list(_pool(nt).map(fn, sls))


def _cut(arr: np.ndarray, sl: slice) -> np.ndarray:
    """Slab of a grid array or of a broadcastable one (size-1 outer axis kept)."""
    return arr if arr.shape[0] == 1 else arr[sl]


# --------------------------------------------------------------------------
# transforms
# --------------------------------------------------------------------------

def _fft_axis(x: np.ndarray, out: np.ndarray, axis: int, inverse: bool):
    """out = numpy 1-D (i)fft of x along ``axis``, lines split over threads."""
    nd = x.ndim
    split = 0 if axis != 0 else 1
    f = np.fft.ifft if inverse else np.fft.fft

    def job(sl):
        idx = [slice(None)] * nd
        idx[split] = sl
        idx = tuple(idx)
        f(x[idx], axis=axis, out=out[idx])

    nt = nthreads()
    sls = _slabs(x.shape[split], nt)
    list(_pool(len(sls)).map(job, sls)) if len(sls) > 1 else job(sls[0])


def fftn_(x: np.ndarray, inverse: bool, scratch: np.ndarray) -> np.ndarray:
    """numpy.fft.fftn / ifftn of one component over all its axes (x first,
    as numpy's _raw_fftnd does).  Uses ``scratch`` (same shape, complex128);
    the result lands in x or scratch, whichever is returned."""
    src, dst = x, scratch
    for axis in reversed(range(x.ndim)):
        _fft_axis(src, dst, axis, inverse)
        src, dst = dst, src
    return src


def gamma1_(comps: list, scale: float = 1.0) -> list:
    """fftcond_oracle.gamma1 on a list of d component arrays (consumed: the
    transforms run in their storage).  Returns the d projected components.
    The k-multiplies and the dot product run slab by slab as in-place ufunc
    calls: the same IEEE operations on the same operands."""
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
    dot = np.empty(grid, dtype=np.complex128)
    invs = inv if scale == 1.0 else None  # inv * 1.0 == inv

    def dot_slab(sl):
        dt = dot[sl]
        np.multiply(_cut(ks[0], sl), fh[0][sl], out=dt)  # dot = ks[0] * fh[0]
        tmp = scratch[sl]
        for c in range(1, d):
            np.multiply(_cut(ks[c], sl), fh[c][sl], out=tmp)
            np.add(dt, tmp, out=dt)  # dot = dot + ks[c] * fh[c]
        np.multiply(dt, inv[sl] if invs is not None else inv[sl] * scale, out=dt)

    par(grid[0], dot_slab)
    out = []
    for c in range(d):
        par(grid[0], lambda sl: np.multiply(_cut(ks[c], sl), dot[sl], out=fh[c][sl]))  # out[c] = ks[c] * dot
        r = fftn_(fh[c], True, scratch)
        if r is scratch:
            scratch = fh[c]
        out.append(r)
    return out


# --------------------------------------------------------------------------
# reductions (spectral_ops.py:33-55)
# --------------------------------------------------------------------------

def _rows(values: np.ndarray) -> np.ndarray:
    return np.sum(values.reshape(-1, values.shape[-1]), axis=-1)


def _total(rowlists: list) -> float:
    """total_real over the concatenation of row-sum vectors (slabs in order)."""
    allrows = np.concatenate(rowlists)
    if not np.all(np.isfinite(allrows)):
        return float(np.sum(allrows))
    return math.fsum(allrows.tolist())


def _means(comps: list) -> np.ndarray:
    """component_means of a list of component arrays, slab-parallel."""
    out = []
    for x in comps:
        parts = par(x.shape[0], lambda sl: (_rows(x[sl].real), _rows(x[sl].imag)))
        out.append(complex(_total([p[0] for p in parts]), _total([p[1] for p in parts])) / x.size)
    return np.array(out)


def _sumsq(comps: list) -> float:
    """total_real(np.abs(g) ** 2) over all components."""
    rows = []
    for x in comps:
        rows += par(x.shape[0], lambda sl: _rows(np.abs(x[sl]) ** 2))
    return _total(rows)


# --------------------------------------------------------------------------
# the loops
# --------------------------------------------------------------------------

def solve(chi: np.ndarray, scheme: str, sigma1: complex, *, e0=None, tol: float = 1e-8,
          max_iters: int = 1000, alpha: float | None = None, beta: float | None = None,
          gamma1_scale: float = 1.0, keep_fields: bool = True, on_iter=None) -> O.OracleResult:
    """``fftcond_oracle.solve`` for the schemes the 3-D configs use (basic,
    em_sub), in bounded memory on all host threads.  Fields come back as
    (d, *grid) arrays when ``keep_fields`` (E = e or Q, J = j or Jq,
    aug = (Q, S, T)).  ``on_iter(k)`` is called at the end of iteration k
    (the bench's per-iteration CPU timing)."""
    chi = np.asarray(chi, dtype=bool)
    d = chi.ndim
    if e0 is None:
        e0 = (1.0,) + (0.0,) * (d - 1)
    if scheme == "basic":
        return _loop_basic(chi, complex(sigma1), e0, tol, max_iters, gamma1_scale, keep_fields, on_iter)
    if scheme == "em_sub":
        return _loop_em_sub(chi, complex(sigma1), e0, tol, max_iters, alpha, beta, gamma1_scale, keep_fields,
                            on_iter)
    raise ValueError(f"lean oracle covers basic and em_sub, not {scheme!r}")


def _e0(e0):
    e0v = np.array([complex(v) for v in e0], dtype=np.complex128)
    return e0v, np.vdot(e0v, e0v).real


def _zeros(grid, d):
    out = [np.empty(grid, dtype=np.complex128) for _ in range(d)]
    for x in out:
        par(grid[0], lambda sl: x[sl].fill(0))
    return out


def _loop_basic(chi, sigma1, e0, tol, max_iters, scale, keep, on_iter):
    """fftcond_oracle._loop_h(accelerated=False), solvers.py:280-331."""
    s0 = O.reference_sigma0("basic", sigma1, None)
    grid = chi.shape
    npts = chi.size
    d = chi.ndim
    n0 = grid[0]
    sig = np.empty(grid, dtype=np.complex128)
    par(n0, lambda sl: np.copyto(sig[sl], np.where(chi[sl], sigma1, 1.0 + 0j)))
    e0v, e0sq = _e0(e0)
    out = O.OracleResult()
    stop = O._Stop(tol)
    e = _zeros(grid, d)  # e_raw = e0f.copy(), then pinned e in place
    for c in range(d):
        par(n0, lambda sl: e[c][sl].fill(e0v[c]))
    g = None
    j = _zeros(grid, d)
    sstar = 0j
    if on_iter is not None:
        on_iter(0)
    with np.errstate(over="ignore", invalid="ignore"):
        for k in range(1, max_iters + 1):
            if k > 1:
                def upd(sl):  # e_raw = e - g / s0
                    for c in range(d):
                        np.subtract(e[c][sl], g[c][sl] / s0, out=e[c][sl])

                par(n0, upd)
                j = g  # reuse the storage
                g = None
            delta = e0v - _means(e)

            def pin(sl):  # e = e_raw + delta; j = sig * e
                for c in range(d):
                    np.add(e[c][sl], delta[c], out=e[c][sl])
                    np.multiply(sig[sl], e[c][sl], out=j[c][sl])

            par(n0, pin)
            jm = _means(j)
            den = float(np.linalg.norm(jm))
            sstar = complex(np.vdot(e0v, jm)) / e0sq
            if den < O.TINY and math.isfinite(den):
                out.degenerate_flux = True
                out.status = "Diverged"
                break
            jin = [x.copy() for x in j] if keep else j
            g = gamma1_(jin, scale)
            res = math.sqrt(_sumsq(g) / npts) / den
            stopped = stop(out, k, sstar, res)
            if on_iter is not None:
                on_iter(k)
            if stopped:
                break
    out.sigma_star = out.history[-1][1] if out.history else sstar
    if keep:
        out.E = np.stack(e)
        out.J = np.stack(j)
    return out


def _apply_A_c(q, s, tt, t, p, chi):
    """fftcond_oracle.apply_A restricted to one spatial component (and slab)."""
    p1, p2, p3 = p
    u = np.where(chi, p1 * q + p2 * s + p3 * tt, 0.0)
    tm1 = t - 1.0
    return (tm1 * p1 * u + q, np.where(chi, tm1 * p2 * u + s, 0.0), np.where(chi, tm1 * p3 * u + tt, 0.0))


def _loop_em_sub(chi, sigma1, e0, tol, max_iters, alpha, beta, scale, keep, on_iter):
    """fftcond_oracle._loop_aug(accelerated=True), solvers.py:366-443."""
    t = O.map_t(sigma1, alpha, beta)
    p = O.solve_p(alpha, beta)
    p1, p2, p3 = p
    s0 = O.reference_sigma0("em_sub", sigma1, t)
    grid = chi.shape
    npts = chi.size
    d = chi.ndim
    n0 = grid[0]
    e0v, e0sq = _e0(e0)
    out = O.OracleResult()
    stop = O._Stop(tol)
    fq, fs, ft = _zeros(grid, d), _zeros(grid, d), _zeros(grid, d)
    for c in range(d):
        par(n0, lambda sl: fq[c][sl].fill(e0v[c]))
    inv_scale = 1.0 / (1.0 + s0)
    inv_c = (t - 1.0) / (t + s0)
    tau = np.empty(grid, dtype=np.complex128)  # (t - 1) p1 chi, complex as in the reference expression
    par(n0, lambda sl: np.copyto(tau[sl], (t - 1.0) * p1 * chi[sl].astype(np.float64)))
    work = _zeros(grid, d)  # R_q, then Jq
    sstar = 0j
    bshape = (1,) * len(grid)

    def new_iterate(sl, wq_fn):
        """(Q, S, T)_raw = (A + s0)^-1 W on one slab (solvers.py:408-411)."""
        ch = chi[sl]
        for c in range(d):
            q, s, tt = fq[c][sl], fs[c][sl], ft[c][sl]
            wq, ws, wt = wq_fn(c, sl, q, s, tt)
            u = np.where(ch, p1 * wq + p2 * ws + p3 * wt, 0.0)
            q[...] = inv_scale * (wq - inv_c * p1 * u)
            s[...] = np.where(ch, inv_scale * (ws - inv_c * p2 * u), 0.0)
            tt[...] = np.where(ch, inv_scale * (wt - inv_c * p3 * u), 0.0)

    def w_init(c, sl, q, s, tt):  # W = A(raw) + s0 raw (solvers.py:386-387)
        aq, as_, at = _apply_A_c(q, s, tt, t, p, chi[sl])
        return aq + s0 * q, as_ + s0 * s, at + s0 * tt

    def w_step(c, sl, q, s, tt):  # solvers.py:398-403 with J_raw = A(F_raw) recomputed
        jqc, jsc, jtc = _apply_A_c(q, s, tt, t, p, chi[sl])
        rq = jqc - s0 * q
        rs = jsc - s0 * s
        rt = jtc - s0 * tt
        e0f = np.full(q.shape, e0v[c], dtype=np.complex128)
        return 2.0 * s0 * e0f - 2.0 * g[c][sl] + rq, -rs, rt

    g = None
    if on_iter is not None:
        on_iter(0)
    with np.errstate(over="ignore", invalid="ignore"):
        for k in range(1, max_iters + 1):
            if k == 1:
                par(n0, lambda sl: new_iterate(sl, w_init))
            else:
                def rq_slab(sl):
                    for c in range(d):
                        jqc = _apply_A_c(fq[c][sl], fs[c][sl], ft[c][sl], t, p, chi[sl])[0]
                        np.copyto(work[c][sl], jqc - s0 * fq[c][sl])

                par(n0, rq_slab)
                g = gamma1_(work, scale)
                par(n0, lambda sl: new_iterate(sl, w_step))
                work = g  # reuse the storage
                g = None
            delta = e0v - _means(fq)

            def pinned(sl):  # solvers.py:416-420 (+ the js part of the residual)
                ch = chi[sl]
                rows = []
                for c in range(d):
                    jqc, jsc, _ = _apply_A_c(fq[c][sl], fs[c][sl], ft[c][sl], t, p, ch)
                    dfc = delta[c:c + 1].reshape(bshape)
                    np.copyto(work[c][sl], jqc + p1 * tau[sl] * dfc + dfc)
                    rows.append(_rows(np.abs(jsc + p2 * tau[sl] * dfc) ** 2 * ch))
                return rows

            js_parts = par(n0, pinned)
            js_rows = [r for c in range(d) for r in (part[c] for part in js_parts)]
            jm = _means(work)
            den = float(np.linalg.norm(jm))
            sstar = complex(np.vdot(e0v, jm)) / e0sq
            if den < O.TINY and math.isfinite(den):
                out.degenerate_flux = True
                out.status = "Diverged"
                break
            jq_keep = [x.copy() for x in work] if keep else None
            gj = gamma1_(work, scale)
            tot = _sumsq(gj)
            tot += _total(js_rows)
            work = gj
            del gj
            res = math.sqrt(tot / npts) / den
            stopped = stop(out, k, sstar, res)
            if on_iter is not None:
                on_iter(k)
            if stopped:
                break
    out.sigma_star = out.history[-1][1] if out.history else sstar
    if keep:
        delta = e0v - _means(fq)
        Q = np.stack([fq[c] + delta[c:c + 1].reshape(bshape) for c in range(d)])
        out.E = Q
        out.J = np.stack(jq_keep) if jq_keep is not None else None
        out.aug = (Q, np.stack(fs), np.stack(ft))
    return out


def timed_iterations(chi, scheme, sigma1, iters: int, **kw) -> list:
    """Wall time of each of the first ``iters`` iterations (setup excluded:
    the clock starts when the loop does)
    of a solve with every iteration run (tol 1e-300): the CPU baseline."""
    marks = []
    solve(chi, scheme, sigma1, tol=1e-300, max_iters=iters, keep_fields=False,
          on_iter=lambda k: marks.append(time.perf_counter()), **kw)
    return [b - a for a, b in zip(marks[:-1], marks[1:])]
