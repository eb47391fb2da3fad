"""Field containers returned by the solver.

``VectorField`` mirrors the reference container (``fftcond/spectral_ops.py``
:58-93): ``data[c, ...]`` is component c (0 = x) on the grid, complex128.
Here the data may live on the GPU: a field produced by a solve keeps its
device tensor and is copied to host memory only when ``.data`` is read
(at 1024^3 one field is 48 GiB, so eager host copies are not an option).
``AugmentedField`` is the (Q, S, T) triple of the substituted schemes
(``spectral_ops.py:141-173``).
"""

from __future__ import annotations

import numpy as np

from .exceptions import SupportError

# Test hook, same role as the reference's spectral_ops._gamma1_scale
# (spectral_ops.py:29-30): scales the nonzero-mode multiplier of Gamma_1.
_gamma1_scale = 1.0


def _total(values: np.ndarray) -> float:
    """Deterministic host total (row sums, exactly rounded combine)."""
    import math

    rows = np.sum(values.reshape(-1, values.shape[-1]), axis=-1)
    if not np.all(np.isfinite(rows)):
        return float(np.sum(rows))
    return math.fsum(rows.tolist())


# Device fields up to this size come back through page-locked memory (torch's
# caching host allocator keeps the blocks for the next read): ~3x the
# bandwidth of a pageable copy.  Larger ones (1024^3: 48 GiB each) take the
# pageable path so the process does not pin a large share of host RAM.
PINNED_COPY_MAX_BYTES = 8 << 30


def _to_host(dev) -> np.ndarray:
    import torch

    if dev.numel() * dev.element_size() <= PINNED_COPY_MAX_BYTES:
        host = torch.empty(dev.shape, dtype=dev.dtype, pin_memory=True)
        host.copy_(dev)  # synchronous: the stream is drained when this returns
        return host.numpy()
    return dev.cpu().numpy()


class VectorField:
    """Complex d-vector samples on a periodic grid, host or device resident."""

    __slots__ = ("_host", "_dev")

    def __init__(self, data=None, *, device=None):
        self._host = None
        self._dev = device
        if data is not None:
            arr = np.asarray(data, dtype=np.complex128)
            if arr.ndim not in (3, 4) or arr.shape[0] != arr.ndim - 1:
                raise ValueError(f"expected shape (2, ny, nx) or (3, nz, ny, nx), got {arr.shape}")
            self._host = arr
        elif device is None:
            raise ValueError("VectorField needs host data or a device tensor")

    @classmethod
    def from_device(cls, tensor) -> "VectorField":
        return cls(None, device=tensor)

    @property
    def data(self) -> np.ndarray:
        if self._host is None:
            self._host = _to_host(self._dev)
            self._dev = None
        return self._host

    @data.setter
    def data(self, value):
        self._host = np.asarray(value, dtype=np.complex128)
        self._dev = None

    @property
    def device_tensor(self):
        """The device tensor if the field still lives on the GPU, else None."""
        return self._dev

    @property
    def shape(self) -> tuple:
        return tuple(self._host.shape if self._host is not None else self._dev.shape)

    @property
    def grid_shape(self) -> tuple:
        return self.shape[1:]

    @classmethod
    def zeros(cls, *grid) -> "VectorField":
        return cls(np.zeros((len(grid),) + tuple(grid), dtype=np.complex128))

    @classmethod
    def constant(cls, vec, *grid) -> "VectorField":
        v = np.asarray(vec, dtype=np.complex128).reshape(len(grid))
        out = np.empty((len(grid),) + tuple(grid), dtype=np.complex128)
        for c in range(len(grid)):
            out[c] = v[c]
        return cls(out)

    def mean(self) -> np.ndarray:
        d = self.data
        npts = int(np.prod(d.shape[1:]))
        return np.array([complex(_total(d[c].real), _total(d[c].imag)) / npts
                         for c in range(d.shape[0])])

    def copy(self) -> "VectorField":
        return VectorField(self.data.copy())


class AugmentedField:
    """(Q, S, T) triple; S and T vanish off the inclusion."""

    __slots__ = ("Q", "S", "T")

    def __init__(self, Q: VectorField, S: VectorField, T: VectorField):
        if not (Q.grid_shape == S.grid_shape == T.grid_shape):
            raise ValueError("Q, S, T must share one grid")
        self.Q, self.S, self.T = Q, S, T

    @classmethod
    def from_mean(cls, vec, *grid) -> "AugmentedField":
        return cls(VectorField.constant(vec, *grid), VectorField.zeros(*grid), VectorField.zeros(*grid))

    @property
    def grid_shape(self) -> tuple:
        return self.Q.grid_shape

    def copy(self) -> "AugmentedField":
        return AugmentedField(self.Q.copy(), self.S.copy(), self.T.copy())


def check_support(f: AugmentedField, chi: np.ndarray):
    outside = ~chi
    if np.any(f.S.data[:, outside]) or np.any(f.T.data[:, outside]):
        raise SupportError("S/T slots carry data on phase-2 pixels")
