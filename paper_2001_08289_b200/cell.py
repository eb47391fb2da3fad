"""Periodic unit-cell phase maps (the solver input).

``PhaseMap`` carries the phase-1 indicator chi of a periodic cell on a
pixel (d = 2) or voxel (d = 3) grid; axis order is (y, x) or (z, y, x), x
fastest, matching the reference's ``chi[j, i]`` convention
(``fftcond/geometry.py:20-39``).  The reference is 2-D only; d = 3 is the
extension the BASELINE 3-D configurations need.  Builders reproduce the
reference's centred square (``geometry.py:85-106``) and add its cube and
random-medium analogues.
"""

from __future__ import annotations

from fractions import Fraction

import numpy as np


class PhaseMap:
    """Immutable two-phase indicator; every axis even and >= 2."""

    __slots__ = ("_chi", "_dev")

    def __init__(self, chi):
        arr = np.array(chi, dtype=bool)
        if arr.ndim not in (2, 3):
            raise ValueError(f"indicator must be 2-D or 3-D, got shape {arr.shape}")
        if any(n < 2 or n % 2 for n in arr.shape):
            raise ValueError(f"grid dims must be even and >= 2, got {arr.shape}")
        arr.flags.writeable = False
        self._chi = arr
        self._dev = None  # device copy, created on first solve

    @property
    def chi(self) -> np.ndarray:
        return self._chi

    @property
    def dim(self) -> int:
        return self._chi.ndim

    @property
    def grid(self) -> tuple:
        return self._chi.shape

    @property
    def nx(self) -> int:
        return self._chi.shape[-1]

    @property
    def ny(self) -> int:
        return self._chi.shape[-2]

    @property
    def nz(self) -> int:
        return self._chi.shape[0] if self._chi.ndim == 3 else 1

    @property
    def volume_fraction(self) -> Fraction:
        return Fraction(int(self._chi.sum()), self._chi.size)

    def __eq__(self, other):
        if not isinstance(other, PhaseMap):
            return NotImplemented
        return self._chi.shape == other._chi.shape and bool(np.array_equal(self._chi, other._chi))

    def __hash__(self):
        return hash((self._chi.shape, self._chi.tobytes()))

    def __repr__(self):
        dims = "x".join(str(n) for n in reversed(self._chi.shape))
        return f"PhaseMap({dims}, f={float(self.volume_fraction):.4f})"


def volume_fraction(pmap: PhaseMap) -> Fraction:
    return pmap.volume_fraction


def build_uniform(n: int, phase1: bool = False, dim: int = 2) -> PhaseMap:
    """Single-phase n^dim cell."""
    return PhaseMap(np.full((n,) * dim, bool(phase1)))


def _even_side(n: int, side_fraction: float) -> int:
    if n < 2 or n % 2:
        raise ValueError(f"grid side must be even and >= 2, got {n}")
    if not 0.0 < side_fraction < 1.0:
        raise ValueError(f"side_fraction must lie in (0, 1), got {side_fraction}")
    m_real = side_fraction * n
    m = int(round(m_real))
    if abs(m_real - m) > 1e-9 * n or m % 2 or m <= 0:
        raise ValueError(
            f"side_fraction * n = {m_real!r} is not an even integer; "
            f"side {side_fraction} is not representable on an n={n} grid")
    return m


def build_square_array(n: int, side_fraction: float) -> PhaseMap:
    """Centred square inclusion of side side_fraction*n (an even integer)."""
    m = _even_side(n, side_fraction)
    chi = np.zeros((n, n), dtype=bool)
    lo = (n - m) // 2
    chi[lo:lo + m, lo:lo + m] = True
    return PhaseMap(chi)


def build_cube_array(n: int, side: int) -> PhaseMap:
    """Centred cubic inclusion of ``side`` voxels on an n^3 grid.

    BASELINE config 3 asks for side 0.63*N, which is not an even integer at
    N = 512 (322.56); callers pass the nearest even voxel count explicitly.
    """
    if n < 2 or n % 2:
        raise ValueError(f"grid side must be even and >= 2, got {n}")
    if side <= 0 or side > n or side % 2:
        raise ValueError(f"cube side must be an even integer in (0, {n}], got {side}")
    chi = np.zeros((n, n, n), dtype=bool)
    lo = (n - side) // 2
    chi[lo:lo + side, lo:lo + side, lo:lo + side] = True
    return PhaseMap(chi)


def build_disk_array(n: int, radius: float) -> PhaseMap:
    """Centred disk: pixel centres within ``radius`` of the cell centre."""
    if n < 2 or n % 2:
        raise ValueError(f"grid side must be even and >= 2, got {n}")
    if not 0.0 < radius < 0.5:
        raise ValueError(f"radius must lie in (0, 0.5), got {radius}")
    c = (np.arange(n) + 0.5) / n - 0.5
    return PhaseMap(c[None, :] ** 2 + c[:, None] ** 2 <= radius * radius)


def build_random_medium(n: int, dim: int = 3, *, seed: int, smoothing: float, fraction: float) -> PhaseMap:
    """Seeded random two-phase medium (BASELINE config 4 recipe).

    Uniform [0, 1) voxel field from ``numpy.random.default_rng(seed)``,
    periodic Gaussian smoothing of standard deviation ``smoothing`` voxels
    applied as the spectral multiplier exp(-2 pi^2 s^2 |k/n|^2), and phase 1
    where the smoothed field is at or below its ``fraction`` quantile.
    """
    rng = np.random.default_rng(seed)
    u = rng.random((n,) * dim)
    k = np.fft.fftfreq(n)
    k2 = np.zeros((n,) * dim)
    for ax in range(dim):
        shape = [1] * dim
        shape[ax] = n
        k2 = k2 + (k.reshape(shape)) ** 2
    s = np.fft.ifftn(np.fft.fftn(u) * np.exp(-2.0 * np.pi ** 2 * smoothing ** 2 * k2)).real
    thr = np.quantile(s, fraction)
    return PhaseMap(s <= thr)
