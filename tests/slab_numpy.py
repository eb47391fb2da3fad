"""numpy stand-in for GpuSlab (TEST INFRASTRUCTURE): the same per-rank phase
semantics as fftc_slab_* (include/fftcond_b200.h), written with the oracle's
formulas (oracle/fftcond_oracle.py, restating solvers.py:280-443), so the
slab driver (paper_2001_08289_b200/slab.py) -- transposes, all-reduces,
delta pinning, monitor -- can be exercised on CPU over gloo."""

from __future__ import annotations

import math

import numpy as np
import torch

from oracle import fftcond_oracle as O

ALPHA, BETA = 0.25, 4.0


class NumpySlab:
    def __init__(self, chi_local, n_global, z0, nzl, y0, nyl, cfg):
        nz, ny, nx = n_global
        self.chi = np.asarray(chi_local, bool)
        self.n = n_global
        self.y0, self.nyl, self.nzl = y0, nyl, nzl
        self.Ng = nx * ny * nz
        self.scheme = cfg.scheme.value
        self.em_type = cfg.scheme.accelerated
        self.sub = cfg.scheme.substituted
        self.s1 = complex(cfg.sigma1)
        self.tol = cfg.tol
        self.max_iters = cfg.max_iters
        self.e0v = cfg.e0_vector(3)
        self.e0sq = float(np.vdot(self.e0v, self.e0v).real)
        if self.sub:
            self.t = O.map_t(self.s1, ALPHA, BETA)
            self.p = O.solve_p(ALPHA, BETA)
        else:
            self.t, self.p = None, None
        self.s0 = O.reference_sigma0(self.scheme, self.s1, self.t, cfg.sigma0_override)
        self.sig = np.where(self.chi, self.s1, 1.0 + 0j)
        shz, shy = (3, nzl, ny, nx), (3, nyl, nz, nx)
        self.Az = torch.zeros(shz, dtype=torch.complex128)
        self.Ay = torch.zeros(shy, dtype=torch.complex128)
        self.Bz = torch.zeros(shz, dtype=torch.complex128) if self.em_type else self.Az
        self.By = torch.zeros(shy, dtype=torch.complex128) if self.em_type else self.Ay
        self.delta = np.zeros(3, complex)
        self.hist = []
        self.res0 = None
        self.prev = None
        self.k = 1
        self.stopped = False
        self.status = 1
        self.degenerate = False
        self.last = 0j

    # -- helpers ---------------------------------------------------------------
    def _e0f(self):
        f = np.empty((3,) + self.chi.shape, complex)
        for c in range(3):
            f[c] = self.e0v[c]
        return f

    def _deltas(self, raw):
        out = np.zeros(8)
        for c in range(3):
            m = raw[c].sum() / self.Ng
            dl = self.e0v[c] - m
            out[2 * c], out[2 * c + 1] = dl.real, dl.imag
        return out

    def _flux(self):
        """(A channel, B channel, j for <j>, js for the residual) of the current iterate."""
        dl = self.delta.reshape(3, 1, 1, 1)
        if not self.sub:
            j = self.sig * (self.X0 + dl)
            if self.em_type:
                return (self.sig - self.s0) * self.X0, j, j, None
            return j, None, j, None
        jq_raw, js_raw, _ = O.apply_A(self.X0, self.X1, self.X2, self.t, self.p, self.chi)
        tau = (self.t - 1.0) * self.p[0] * self.chi.astype(float)
        jq = jq_raw + self.p[0] * tau * dl + dl
        js = js_raw + self.p[1] * tau * dl
        if self.em_type:
            return jq_raw - self.s0 * self.X0, jq, jq, js
        return jq, None, jq, js

    # -- phases ----------------------------------------------------------------
    def phase(self, ph):
        if ph == 0:
            e0f = self._e0f()
            if self.scheme == "basic":
                self.X0 = e0f
            elif self.scheme == "em":
                self.X0 = ((self.sig + self.s0) * e0f) / (self.sig + self.s0)
            else:
                self.X0, self.X1, self.X2 = e0f, np.zeros_like(e0f), np.zeros_like(e0f)
                if self.scheme == "em_sub":
                    aq, as_, at = O.apply_A(self.X0, self.X1, self.X2, self.t, self.p, self.chi)
                    self._em_sub_update(aq + self.s0 * self.X0, as_, at)
            return self._deltas(self.X0)
        if ph == 1:
            a, b, j, js = self._flux()
            self.Az.numpy()[...] = np.fft.fft(np.fft.fft(a, axis=3), axis=2)
            if b is not None:
                self.Bz.numpy()[...] = np.fft.fft(np.fft.fft(b, axis=3), axis=2)
            out = np.zeros(8)
            for c in range(3):
                m = j[c].sum() / self.Ng
                out[2 * c], out[2 * c + 1] = m.real, m.imag
            out[6] = float(np.sum(np.abs(js) ** 2 * self.chi)) if js is not None else 0.0
            return out
        if ph == 2:
            nz, ny, nx = self.n
            kx = np.fft.fftfreq(nx, 1 / nx)[None, None, :]
            ky = np.fft.fftfreq(ny, 1 / ny)[self.y0:self.y0 + self.nyl][:, None, None]
            kz = np.fft.fftfreq(nz, 1 / nz)[None, :, None]
            k2 = kx * kx + ky * ky + kz * kz
            inv = np.where(k2 != 0, 1.0 / np.where(k2 != 0, k2, 1), 0.0)
            ks = (kx, ky, kz)

            def proj(F):
                dot = (kx * F[0] + ky * F[1] + kz * F[2]) * inv
                return np.stack([np.broadcast_to(k * dot, dot.shape) for k in ks])

            A = np.fft.fft(self.Ay.numpy(), axis=2)
            if self.em_type:
                Bh = np.fft.fft(self.By.numpy(), axis=2)
                G = proj(Bh)
                self.Ay.numpy()[...] = np.fft.ifft(A - 2 * proj(A), axis=2) * nz
            else:
                G = proj(A)
                self.Ay.numpy()[...] = np.fft.ifft(G, axis=2) * nz
            out = np.zeros(8)
            out[0] = float(np.sum(np.abs(G) ** 2)) / self.Ng
            return out
        if ph == 3:
            # Az holds the unnormalised inverse z transform; numpy's inverse y/x
            # transforms divide by ny*nx, the remaining 1/nz completes 1/N
            g = np.fft.ifft(np.fft.ifft(self.Az.numpy(), axis=2), axis=3) / self.n[0]
            dl = self.delta.reshape(3, 1, 1, 1)
            if self.scheme == "basic":
                self.X0 = (self.X0 + dl) - g / self.s0
            elif self.scheme == "em":
                self.X0 = (2.0 * self.s0 * self._e0f() + g) / (self.sig + self.s0)
            elif self.scheme == "basic_sub":
                _, js = self._flux()[2:]
                self.X1 = np.where(self.chi, self.X1 - js / self.s0, 0.0)
                self.X0 = (self.X0 + dl) - g / self.s0
            else:
                jq_raw, js_raw, jt_raw = O.apply_A(self.X0, self.X1, self.X2, self.t, self.p, self.chi)
                ws = -(js_raw - self.s0 * self.X1)
                wt = jt_raw - self.s0 * self.X2
                self._em_sub_update(2.0 * self.s0 * self._e0f() + g, ws, wt)
            return self._deltas(self.X0)
        raise ValueError(ph)

    def _em_sub_update(self, wq, ws, wt):
        p1, p2, p3 = self.p
        s_ = 1.0 / (1.0 + self.s0)
        c_ = (self.t - 1.0) / (self.t + self.s0)
        u = np.where(self.chi, p1 * wq + p2 * ws + p3 * wt, 0.0)
        self.X0 = s_ * (wq - c_ * p1 * u)
        self.X1 = np.where(self.chi, s_ * (ws - c_ * p2 * u), 0.0)
        self.X2 = np.where(self.chi, s_ * (wt - c_ * p3 * u), 0.0)

    def set_delta(self, d6):
        self.delta = np.array([complex(d6[2 * c], d6[2 * c + 1]) for c in range(3)])

    def monitor(self, tot):
        jm = np.array([complex(tot[2 * c], tot[2 * c + 1]) for c in range(3)])
        den = float(np.linalg.norm(jm))
        sstar = complex(np.vdot(self.e0v, jm)) / self.e0sq
        self.last = sstar
        rec = np.zeros(7)
        if den < 1e-300 and math.isfinite(den):
            self.stopped, self.status, self.degenerate = True, 2, True
        else:
            res = math.sqrt((tot[7] + tot[6]) / self.Ng) / den
            if not (math.isfinite(res) and np.isfinite(sstar)):
                self.stopped, self.status = True, 2
            else:
                self.hist.append((sstar, res))
                if self.res0 is None:
                    self.res0 = res
                settled = self.prev is None or abs(sstar - self.prev) <= self.tol * abs(sstar)
                if res <= self.tol and settled:
                    self.stopped, self.status = True, 0
                elif self.res0 > 0 and res > 1e6 * self.res0:
                    self.stopped, self.status = True, 2
                else:
                    self.prev = sstar
                    if self.k >= self.max_iters:
                        self.stopped = True
                    self.k += 1
                rec[4], rec[5], rec[6] = sstar.real, sstar.imag, res
        rec[0], rec[1], rec[2], rec[3] = float(self.stopped), self.status, float(self.degenerate), len(self.hist)
        if not self.hist:
            rec[4], rec[5] = sstar.real, sstar.imag
        return rec

    def finalize(self):
        dl = self.delta.reshape(3, 1, 1, 1)
        if not self.sub:
            E = self.X0 + dl
            J = self.sig * E
        else:
            E = self.X0 + dl
            J = self._flux()[2]
        out = np.zeros(12)
        for c in range(3):
            me, mj = E[c].sum() / self.Ng, J[c].sum() / self.Ng
            out[2 * c], out[2 * c + 1], out[6 + 2 * c], out[6 + 2 * c + 1] = me.real, me.imag, mj.real, mj.imag
        return out
