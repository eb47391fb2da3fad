"""Golden vectors for the public operator surface, produced by the LIVE
reference (TEST INFRASTRUCTURE; runs only in the dev container, where
/root/reference exists).

Writes tests/golden/ops.npz (inputs and reference outputs per case) and
tests/golden/ops.json (scalar outputs and the reference selftest report).
Reference functions exercised: spectral_ops.py:96-278 (inner, norm, gamma0,
gamma1, inner_aug, norm_aug, gamma1_aug, apply_chi_aug, apply_local_A,
invert_shifted_A) and solvers.py:147-204 (extract_sigma_star(_aug),
recover_physical_fields, equilibrium_residual(_aug)); selftest.py:89-205.

    PYTHONPATH=/root/reference/pkg/src PYTHONDONTWRITEBYTECODE=1 python oracle/gen_golden_ops.py
"""

from __future__ import annotations

import json
import os
import sys

import numpy as np

REF = "/root/reference/pkg/src"
if REF not in sys.path:
    sys.path.insert(0, REF)

from fftcond import geometry as G  # noqa: E402
from fftcond import selftest as ST  # noqa: E402
from fftcond import solvers as SV  # noqa: E402
from fftcond import spectral_ops as SO  # noqa: E402
from fftcond import transform as TR  # noqa: E402

OUT = os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))), "tests", "golden")

CASES = [
    # name, ny, nx, chi recipe, seed, sigma1, e0, sigma0 shift
    ("sq16", 16, 16, "square", 11, 3.0 + 1.0j, (1.0, 0.0), 0.7 + 0.3j),
    ("rect32x64", 32, 64, "random", 12, -7.5 + 2.0j, (0.6, 0.8j), 2.0 - 1.0j),
    ("sq32", 32, 32, "square", 13, 10.0, (1.0, 1.0), 0.25),
]


def _rand(rng, ny, nx):
    return rng.standard_normal((2, ny, nx)) + 1j * rng.standard_normal((2, ny, nx))


def cplx(z):
    z = complex(z)
    return [z.real, z.imag]


def main():
    arrays, meta = {}, {"cases": [], "selftest": []}
    interval = TR.SpectralInterval(0.25, 4.0)
    params = TR.solve_p(interval)
    for name, ny, nx, recipe, seed, sigma1, e0, shift in CASES:
        rng = np.random.default_rng(seed)
        if recipe == "square":
            pmap = G.build_square_array(nx, 0.5)
        else:
            pmap = G.PhaseMap(rng.random((ny, nx)) < 0.4)
        chi = pmap.chi
        t = TR.map_t(sigma1, interval)
        f, g = _rand(rng, ny, nx), _rand(rng, ny, nx)
        F = [_rand(rng, ny, nx), np.where(chi, _rand(rng, ny, nx), 0.0), np.where(chi, _rand(rng, ny, nx), 0.0)]
        H = [_rand(rng, ny, nx), np.where(chi, _rand(rng, ny, nx), 0.0), np.where(chi, _rand(rng, ny, nx), 0.0)]
        vf, vg = SO.VectorField(f), SO.VectorField(g)
        aF = SO.AugmentedField(*(SO.VectorField(x) for x in F))
        aH = SO.AugmentedField(*(SO.VectorField(x) for x in H))
        p = f"{name}/"
        arrays[p + "chi"] = chi
        arrays[p + "f"], arrays[p + "g"] = f, g
        for k, x in enumerate(F):
            arrays[p + f"F{k}"] = x
        for k, x in enumerate(H):
            arrays[p + f"H{k}"] = x
        arrays[p + "gamma1_f"] = SO.gamma1(vf).data
        for tag, out in (("gamma1_aug", SO.gamma1_aug(aF, pmap)), ("chi_aug", SO.apply_chi_aug(aF, params, pmap)),
                         ("local_A", SO.apply_local_A(aF, t, params, pmap)),
                         ("inv_shifted", SO.invert_shifted_A(aF, t, shift, params, pmap))):
            arrays[p + tag + "_Q"], arrays[p + tag + "_S"], arrays[p + tag + "_T"] = out.Q.data, out.S.data, out.T.data
        E, J = SV.recover_physical_fields(aF, t, params, pmap)
        arrays[p + "recover_E"], arrays[p + "recover_J"] = E.data, J.data
        meta["cases"].append(dict(
            name=name, ny=ny, nx=nx, sigma1=cplx(sigma1), e0=[cplx(z) for z in e0], shift=cplx(shift), t=cplx(t),
            interval=[0.25, 4.0],
            inner=cplx(SO.inner(vf, vg)), norm=SO.norm(vf), gamma0=[cplx(z) for z in SO.gamma0(vf)],
            inner_aug=cplx(SO.inner_aug(aF, aH, pmap)), norm_aug=SO.norm_aug(aF, pmap),
            gamma0_aug=[cplx(z) for z in SO.gamma0_aug(aF)],
            sigma_star=cplx(SV.extract_sigma_star(vf, pmap, sigma1, e0)),
            sigma_star_aug=cplx(SV.extract_sigma_star_aug(aF, t, params, pmap, e0)),
            eq_residual=SV.equilibrium_residual(vf), eq_residual_aug=SV.equilibrium_residual_aug(aF, pmap),
        ))
    for r in ST.run_selftest():
        meta["selftest"].append(dict(name=r.name, passed=bool(r.passed), measured=float(r.measured),
                                     threshold=float(r.threshold)))
    np.savez_compressed(os.path.join(OUT, "ops.npz"), **arrays)
    with open(os.path.join(OUT, "ops.json"), "w") as fh:
        json.dump(meta, fh, indent=1)
    print(f"wrote {len(arrays)} arrays, {len(meta['cases'])} cases, {len(meta['selftest'])} selftest lines")


if __name__ == "__main__":
    main()
