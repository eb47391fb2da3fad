"""Per-solve wall time of the device-resident path vs the public API (fb.solve
with a fresh host phase map), to locate host overhead in the e2e number."""
import os
import sys
import time

sys.path.insert(0, os.path.join(os.path.dirname(os.path.abspath(__file__)), ".."))
import numpy as np
import torch

import paper_2001_08289_b200 as fb
from paper_2001_08289_b200.solver import _solve_aug, _solve_h

n = int(sys.argv[1]) if len(sys.argv) > 1 else 2048
chi = np.zeros((n, n), dtype=bool)
chi[n // 4:3 * n // 4, n // 4:3 * n // 4] = True
pm_dev = fb.PhaseMap(chi)
for scheme in ("em", "em_sub"):
    sk = fb.SchemeKind(scheme)
    cfg = fb.SolverConfig(scheme=sk, sigma1=10.0, tol=1e-10, max_iters=20000,
                          interval=fb.SpectralInterval(0.25, 4.0) if sk.substituted else None)
    run = _solve_aug if sk.substituted else _solve_h
    for rep in range(3):
        torch.cuda.synchronize()
        t0 = time.perf_counter()
        r = run(pm_dev, cfg, sk.accelerated, want_fields=False)
        torch.cuda.synchronize()
        t1 = time.perf_counter()
        r2 = fb.solve(fb.PhaseMap(chi), cfg)
        _ = r2.sigma_star
        torch.cuda.synchronize()
        t2 = time.perf_counter()
        print(f"{scheme:7s} it={r.iterations:4d} device-path wall {1e3*(t1-t0):8.2f} ms (device {r.device_ms:8.2f})"
              f"  public API wall {1e3*(t2-t1):8.2f} ms", flush=True)
