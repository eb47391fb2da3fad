"""GPU operator tests: per-axis FFTs against numpy.fft and Gamma_1 against
the oracle restatement of the reference _gamma1_arr (spectral_ops.py:120-128),
plus the reference's Gamma_1 property tests (tests/test_spectral_ops.py:55-90)
run on the device projection."""

from __future__ import annotations

import numpy as np
import pytest

pytestmark = pytest.mark.gpu

SHAPES_2D = [(2, 2), (4, 8), (8, 8), (16, 32), (32, 16), (64, 64), (256, 128), (2048, 8), (8, 4096)]
SHAPES_3D = [(2, 16, 16), (4, 16, 16), (16, 16, 16), (16, 16, 2), (16, 2, 16), (8, 16, 32), (32, 16, 8),
             (2, 2, 2), (64, 32, 16)]
# even lengths outside the fused transforms: the general path (cuFFT)
SHAPES_2D += [(6, 10), (48, 30), (100, 2), (6, 8192)]
SHAPES_3D += [(6, 4, 10), (12, 12, 12), (2, 30, 8)]


def _rand(shape, seed=0):
    rng = np.random.default_rng(seed)
    d = len(shape)
    return rng.standard_normal((d,) + shape) + 1j * rng.standard_normal((d,) + shape)


@pytest.mark.parametrize("shape", SHAPES_2D + SHAPES_3D)
@pytest.mark.parametrize("inverse", [False, True])
def test_fft_each_axis(shape, inverse):
    from paper_2001_08289_b200.operators import fft_axes

    f = _rand(shape, 1)
    d = len(shape)
    for ax in range(d):
        got = fft_axes(f, 1 << ax, inverse).cpu().numpy()
        np_axis = -1 - ax
        ref = np.fft.ifft(f, axis=np_axis) * shape[np_axis] if inverse else np.fft.fft(f, axis=np_axis)
        err = np.abs(got - ref).max() / np.abs(ref).max()
        assert err < 1e-14, (shape, ax, inverse, err)


@pytest.mark.parametrize("shape", [(6, 10), (48, 30), (16, 32), (6, 4, 10), (12, 12, 12), (8, 16, 32)])
@pytest.mark.parametrize("inverse", [False, True])
def test_fft_all_axes(shape, inverse):
    from paper_2001_08289_b200.operators import fft_axes

    f = _rand(shape, 2)
    d = len(shape)
    got = fft_axes(f, (1 << d) - 1, inverse).cpu().numpy()
    axes = tuple(range(1, d + 1))
    ref = np.fft.ifftn(f, axes=axes) * np.prod(shape) if inverse else np.fft.fftn(f, axes=axes)
    err = np.abs(got - ref).max() / np.abs(ref).max()
    assert err < 1e-14, (shape, inverse, err)


@pytest.mark.parametrize("shape", SHAPES_2D + SHAPES_3D)
def test_gamma1_matches_oracle(shape):
    from oracle import fftcond_oracle as O
    from paper_2001_08289_b200.operators import gamma1

    f = _rand(shape, 2)
    got = gamma1(f).cpu().numpy()
    ref = O.gamma1(f)
    err = np.abs(got - ref).max() / max(np.abs(ref).max(), 1e-300)
    assert err < 1e-13, (shape, err)


def test_gamma1_scale_hook():
    from oracle import fftcond_oracle as O
    from paper_2001_08289_b200.operators import gamma1

    f = _rand((16, 16), 3)
    got = gamma1(f, scale=0.5).cpu().numpy()
    ref = O.gamma1(f, 0.5)
    assert np.abs(got - ref).max() < 1e-13 * np.abs(ref).max()


class TestGamma1Properties:
    """tests/test_spectral_ops.py:55-90 on the device projection."""

    N = 16

    def _norm(self, a):
        return float(np.sqrt(np.mean(np.abs(a) ** 2)))

    def test_kills_constants(self):
        from paper_2001_08289_b200.operators import gamma1

        f = np.empty((2, self.N, self.N), complex)
        f[0], f[1] = 2.0 + 1j, -0.5
        assert self._norm(gamma1(f).cpu().numpy()) < 1e-14

    def test_gradient_mode_fixed(self):
        from paper_2001_08289_b200.operators import gamma1

        x = (np.arange(self.N) + 0.5) / self.N
        f = np.zeros((2, self.N, self.N), complex)
        f[0] = 2 * np.pi * np.cos(2 * np.pi * x)[None, :]
        g = gamma1(f).cpu().numpy()
        assert self._norm(g - f) <= 1e-12 * self._norm(f)

    def test_divergence_free_killed(self):
        from paper_2001_08289_b200.operators import gamma1

        y = (np.arange(self.N) + 0.5) / self.N
        f = np.zeros((2, self.N, self.N), complex)
        f[0] = np.cos(2 * np.pi * y)[:, None]
        assert self._norm(gamma1(f).cpu().numpy()) <= 1e-12

    def test_idempotent_and_self_adjoint(self):
        from paper_2001_08289_b200.operators import gamma1

        f, h = _rand((self.N, self.N), 4), _rand((self.N, self.N), 5)
        g = gamma1(f).cpu().numpy()
        gg = gamma1(g).cpu().numpy()
        assert self._norm(gg - g) <= 1e-12 * self._norm(g)
        lhs = np.mean(np.sum(np.conj(g) * h, axis=0))
        rhs = np.mean(np.sum(np.conj(f) * gamma1(h).cpu().numpy(), axis=0))
        assert abs(lhs - rhs) <= 1e-12 * self._norm(f) * self._norm(h)

    def test_zero_mean_and_repeatable(self):
        from paper_2001_08289_b200.operators import gamma1

        f = _rand((self.N, self.N), 6)
        g1 = gamma1(f).cpu().numpy()
        g2 = gamma1(f).cpu().numpy()
        assert np.abs(g1.mean(axis=(1, 2))).max() <= 1e-13
        assert np.array_equal(g1, g2)  # bitwise repeatable (test_spectral_ops.py:318-324)
