"""TMA 3-D column passes (FFTC_TMA_COLS3=1) vs the strip kernels on grids
whose y/z lines use them; prints the history deltas per scheme."""
import os
import sys

sys.path.insert(0, os.path.join(os.path.dirname(__file__), ".."))
import numpy as np  # noqa: E402

import paper_2001_08289_b200 as fb  # noqa: E402

shapes = [tuple(int(v) for v in s.split("x")) for s in (sys.argv[1].split(",") if len(sys.argv) > 1 else
                                                        ["256x256x8", "512x256x4", "256x1024x2", "1024x256x2"])]
schemes = sys.argv[2].split(",") if len(sys.argv) > 2 else ["basic", "em", "basic_sub", "em_sub"]
VAR = "FFTC_TMA_COLS3"  # TMA tile passes ("1") vs the strip kernels ("0")
iv = fb.SpectralInterval(0.25, 4.0)
bad = 0
for shape in shapes:
    rng = np.random.default_rng(1)
    pm = fb.PhaseMap(rng.random(shape) < 0.3)
    for scheme in schemes:
        sk = fb.SchemeKind(scheme)
        cfg = fb.SolverConfig(scheme=sk, sigma1=10.0 + 2j, tol=1e-10, max_iters=300, e0=(0.6, 0.0, 0.8),
                              interval=iv if sk.substituted else None)
        os.environ[VAR] = "0"
        r0 = fb.solve(pm, cfg)
        os.environ[VAR] = "1"
        r1 = fb.solve(pm, cfg)
        h0 = np.array([[h.sigma_star.real, h.sigma_star.imag, h.residual] for h in r0.history])
        h1 = np.array([[h.sigma_star.real, h.sigma_star.imag, h.residual] for h in r1.history])
        n = min(len(h0), len(h1))
        z0, z1 = h0[:n, 0] + 1j * h0[:n, 1], h1[:n, 0] + 1j * h1[:n, 1]
        ds = float(np.max(np.abs(z1 - z0) / np.abs(z0))) if n else 0.0
        dr = float(np.max(np.abs(h1[:n, 2] - h0[:n, 2]) / h0[:n, 2])) if n else 0.0
        ok = r0.iterations == r1.iterations and ds < 1e-10 and dr < 1e-6
        bad += not ok
        print(f"{'x'.join(map(str, shape))} {scheme:9s} iters {r0.iterations} vs {r1.iterations}  dsigma {ds:.2e}  "
              f"dres {dr:.2e}  {'OK' if ok else 'MISMATCH'}", flush=True)
print("mismatches:", bad)
