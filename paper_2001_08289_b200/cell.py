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

import os
from fractions import Fraction

import numpy as np


class PhaseMap:
    """Immutable two-phase indicator; every axis even and >= 2."""

    __slots__ = ("_chi", "__weakref__")

    def __init__(self, chi):
        arr = np.array(chi, dtype=bool)
        if arr.ndim not in (2, 3):
            raise ValueError(f"indicator must be 2-D or 3-D, got shape {arr.shape}")
        if any(n < 2 or n % 2 for n in arr.shape):
            raise ValueError(f"grid dims must be even and >= 2, got {arr.shape}")
        arr.flags.writeable = False
        self._chi = arr

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
    applied in Fourier space as the separable multiplier
    prod_axes exp(-2 pi^2 s^2 (k_a/n)^2) on the real-input transform (one
    half-spectrum, so 1024^3 fits in ~30 GB of host memory), and phase 1
    where the smoothed field is at or below its ``fraction`` quantile.
    Deterministic for a given numpy; ``c4_phase_map`` freezes the 1024^3
    instance as a bit-packed file with a committed SHA-256.
    """
    rng = np.random.default_rng(seed)
    u = rng.random((n,) * dim)
    U = np.fft.rfftn(u)
    del u
    k = np.fft.fftfreq(n)
    g = np.exp(-2.0 * np.pi ** 2 * smoothing ** 2 * k * k)
    for ax in range(dim):
        m = U.shape[ax]
        shape = [1] * dim
        shape[ax] = m
        U *= g[:m].reshape(shape)
    s = np.fft.irfftn(U, s=(n,) * dim)
    del U
    thr = np.quantile(s, fraction)
    return PhaseMap(s <= thr)


# BASELINE config 4 as frozen for this build: the 1024^3 instance of the
# recipe above is shared by the GPU runs and the CPU oracle through one
# bit-packed file (save_chi_bits), pinned by its SHA-256.  The file is 128 MiB
# (44 MB compressed), too large for the repository, so it is regenerated
# deterministically when absent and checked against this digest.
C4_SEED, C4_SMOOTHING, C4_FRACTION = 20260809, 4.0, 0.30
C4_CHI_SHA256 = {1024: "e9bfd9c4a8c7eb2f95ed6206beb6bc4ecddf1fa84134e7de5167ddce77b15f9b"}
C4_CHI_DIR = os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))), "data")


def c4_phase_map(n: int = 1024, directory: str | None = None) -> PhaseMap:
    """The config-4 random medium on an n^3 grid.  For n with a frozen digest
    the bit-packed file ``<directory>/c4_chi_<n>.fchi`` is loaded (written on
    first use) and verified; a digest mismatch raises instead of silently
    solving a different medium."""
    import hashlib

    digest = C4_CHI_SHA256.get(n)
    if digest is None:
        return build_random_medium(n, 3, seed=C4_SEED, smoothing=C4_SMOOTHING, fraction=C4_FRACTION)
    directory = directory or C4_CHI_DIR
    path = os.path.join(directory, f"c4_chi_{n}.fchi")
    if not os.path.exists(path):
        pm = build_random_medium(n, 3, seed=C4_SEED, smoothing=C4_SMOOTHING, fraction=C4_FRACTION)
        os.makedirs(directory, exist_ok=True)
        save_chi_bits(pm, path + ".tmp")
        os.replace(path + ".tmp", path)
    with open(path, "rb") as fh:
        h = hashlib.sha256()
        for block in iter(lambda: fh.read(1 << 24), b""):
            h.update(block)
    if h.hexdigest() != digest:
        raise ValueError(f"{path}: SHA-256 {h.hexdigest()} does not match the frozen config-4 medium {digest}")
    return load_chi_bits(path)


# -- phase-map files ---------------------------------------------------------------
RASTER_MAGIC = "P-PHASE"  # geometry.py:17


def save_raster(pmap: PhaseMap) -> str:
    """2-D plain-text raster of the reference (geometry.py:126-136):
    ``P-PHASE <nx> <ny>`` then ny rows of nx 0/1 tokens, row 0 first."""
    if pmap.dim != 2:
        raise ValueError("the P-PHASE text raster is 2-D; use save_chi_bits for 3-D cells")
    lines = [f"{RASTER_MAGIC} {pmap.nx} {pmap.ny}"]
    for row in pmap.chi:
        lines.append(" ".join("1" if v else "0" for v in row))
    return "\n".join(lines) + "\n"


def load_raster(text: str) -> PhaseMap:
    """Parse :func:`save_raster` output (geometry.py:139-189); faults raise
    RasterParseError naming line and column, as the reference does."""
    from .exceptions import RasterParseError

    lines = text.splitlines()
    if not lines or not lines[0].strip():
        raise RasterParseError("missing header", line=1)
    header = lines[0].split()
    if header[0] != RASTER_MAGIC:
        raise RasterParseError(f"expected magic {RASTER_MAGIC!r}", line=1, column=1)
    if len(header) != 3:
        raise RasterParseError(f"header needs 3 tokens, got {len(header)}", line=1, column=len(header))
    try:
        nx, ny = int(header[1]), int(header[2])
    except ValueError:
        raise RasterParseError("dimensions must be integers", line=1, column=2) from None
    if nx < 2 or ny < 2 or nx % 2 or ny % 2:
        raise RasterParseError(f"dims must be even and >= 2, got {nx} x {ny}", line=1, column=2)
    chi = np.zeros((ny, nx), dtype=bool)
    for j in range(ny):
        lineno = j + 2
        if j + 1 >= len(lines):
            raise RasterParseError(f"missing data row {j}", line=lineno)
        tokens = lines[j + 1].split()
        if len(tokens) != nx:
            raise RasterParseError(f"expected {nx} tokens, got {len(tokens)}", line=lineno,
                                   column=min(len(tokens), nx) + 1)
        for i, tok in enumerate(tokens):
            if tok == "1":
                chi[j, i] = True
            elif tok != "0":
                raise RasterParseError(f"token must be 0 or 1, got {tok!r}", line=lineno, column=i + 1)
    for extra, line in enumerate(lines[ny + 1:], start=ny + 2):
        if line.strip():
            raise RasterParseError("unexpected trailing content", line=extra)
    return PhaseMap(chi)


# Bit-packed binary phase map: the text raster costs ~2 bytes
# per voxel and is 2-D only; at 1024^3 this format is 128 MiB.
#   bytes 0-7   magic b"FFTCHI01"
#   bytes 8-11  uint32 LE d (2 or 3);  bytes 12-15 reserved (0)
#   bytes 16-39 int64 LE nx, ny, nz (nz = 1 for d = 2)
#   bytes 40-   chi in C order (z, y, x), 8 voxels per byte, least
#               significant bit first (numpy packbits bitorder="little")
CHI_BITS_MAGIC = b"FFTCHI01"


def save_chi_bits(pmap: PhaseMap, path) -> None:
    chi = pmap.chi
    nz = pmap.nz
    head = CHI_BITS_MAGIC + np.array([pmap.dim, 0], "<u4").tobytes() + np.array([pmap.nx, pmap.ny, nz], "<i8").tobytes()
    with open(path, "wb") as fh:
        fh.write(head)
        fh.write(np.packbits(chi.reshape(-1), bitorder="little").tobytes())


def load_chi_bits(path) -> PhaseMap:
    from .exceptions import RasterParseError

    with open(path, "rb") as fh:
        head = fh.read(40)
        if len(head) < 40 or head[:8] != CHI_BITS_MAGIC:
            raise RasterParseError("not a bit-packed phase map (bad magic)", line=1, column=1)
        d = int(np.frombuffer(head[8:12], "<u4")[0])
        nx, ny, nz = (int(v) for v in np.frombuffer(head[16:40], "<i8"))
        if d not in (2, 3) or (d == 2 and nz != 1) or min(nx, ny, nz) < 1:
            raise RasterParseError(f"bad header: d={d}, n=({nx}, {ny}, {nz})", line=1, column=2)
        count = nx * ny * nz
        body = np.frombuffer(fh.read(), dtype=np.uint8)
    if body.size != (count + 7) // 8:
        raise RasterParseError(f"expected {(count + 7) // 8} data bytes, got {body.size}", line=1, column=3)
    chi = np.unpackbits(body, count=count, bitorder="little").astype(bool)
    return PhaseMap(chi.reshape((nz, ny, nx) if d == 3 else (ny, nx)))
