"""Repeat 3-D solves whose y/z lines run the TMA tile passes on the z-blocked
work layout and compare histories bit for bit (race detector for
cols3_tma.cuh / the z-blocked row kernels).  Usage: python scripts/stress_3d_tma.py [reps]"""
import os
import sys

sys.path.insert(0, os.path.join(os.path.dirname(__file__), ".."))
import numpy as np  # noqa: E402

import paper_2001_08289_b200 as fb  # noqa: E402
from paper_2001_08289_b200 import native  # noqa: E402

reps = int(sys.argv[1]) if len(sys.argv) > 1 else 10
bad = total = 0
for shape, scheme in (((256, 256, 16), "em_sub"), ((512, 256, 8), "basic"), ((256, 512, 8), "em"),
                      ((256, 256, 32), "basic_sub")):
    rng = np.random.default_rng(11)
    pm = fb.PhaseMap(rng.random(shape) < 0.3)
    sk = fb.SchemeKind(scheme)
    cfg = fb.SolverConfig(scheme=sk, sigma1=10.0 + 2j, tol=1e-10, max_iters=400, e0=(0.6, 0.0, 0.8),
                          interval=fb.SpectralInterval(0.25, 4.0) if sk.substituted else None)
    ref = None
    for _ in range(reps):
        r = fb.solve(pm, cfg)
        assert native.last_layout() & 255 > 0, "z-blocked layout expected"
        h = [(x.sigma_star, x.residual) for x in r.history]
        if ref is None:
            ref = h
            continue
        total += 1
        if h != ref:
            bad += 1
            print("MISMATCH", shape, scheme, flush=True)
    print(shape, scheme, len(ref), "records", flush=True)
print(f"{bad} mismatching repeats of {total}")
