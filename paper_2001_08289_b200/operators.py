"""Device operator API: Gamma_1 and raw transforms on GPU fields.

``gamma1(field)`` replaces the reference projection ``gamma1`` /
``_gamma1_arr`` (``fftcond/spectral_ops.py:120-133``): out = ifftn(k (k.F^)
/|k|^2 * scale), zero mode dropped, Nyquist kept, computed by the same
fused sweeps the solver uses (row FFT, column FFT with the projection in
registers, inverse passes).  ``fft_axes`` exposes the unnormalised per-axis
transforms for testing.  Inputs may be numpy arrays (copied to the device)
or CUDA tensors; outputs are CUDA tensors.
"""

from __future__ import annotations

import ctypes as C

import numpy as np

from . import fields as _fields
from . import native
from .exceptions import BackendError, ContractError


def _as_device(data):
    import torch

    if isinstance(data, torch.Tensor):
        t = data.to(device="cuda", dtype=torch.complex128)
    else:
        t = torch.from_numpy(np.ascontiguousarray(np.asarray(data, dtype=np.complex128))).to("cuda")
    return t.contiguous()


def _problem(shape) -> native.Problem:
    d = shape[0]
    grid = shape[1:]
    if len(grid) != d or d not in (2, 3):
        raise ContractError(f"expected a (d, *grid) field with d = 2 or 3, got {tuple(shape)}")
    L = native.lib()
    for n in grid:
        if not L.fftc_supported_length(int(n)):
            raise ContractError(f"grid axis of length {n} is not supported (even lengths >= 2)")
    p = native.Problem()
    p.d = d
    p.n[0] = grid[-1]
    p.n[1] = grid[-2]
    p.n[2] = grid[0] if d == 3 else 1
    return p


def gamma1(data, scale: float | None = None):
    """Gamma_1 of a (d, *grid) complex field on the GPU; returns a CUDA tensor."""
    import torch

    t = _as_device(data)
    out = torch.empty_like(t)
    p = _problem(tuple(t.shape))
    sc = _fields._gamma1_scale if scale is None else float(scale)
    rc = native.lib().fftc_gamma1(C.byref(p), t.data_ptr(), out.data_ptr(), sc,
                                  torch.cuda.current_stream().cuda_stream)
    if rc:
        raise BackendError(f"fftc_gamma1 failed ({rc}): {native.last_error()}")
    return out


def fft_axes(data, axes_mask: int, inverse: bool = False):
    """Unnormalised per-axis DFT (bit 0 = x, 1 = y, 2 = z) on a copy."""
    import torch

    t = _as_device(data).clone()
    p = _problem(tuple(t.shape))
    rc = native.lib().fftc_fft(C.byref(p), t.data_ptr(), int(bool(inverse)), int(axes_mask),
                               torch.cuda.current_stream().cuda_stream)
    if rc:
        raise BackendError(f"fftc_fft failed ({rc}): {native.last_error()}")
    return t
