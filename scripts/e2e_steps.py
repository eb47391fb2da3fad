"""Per-solve wall vs device time of the bench's e2e step (six C2 solves
through fb.solve with a fresh host phase map), to locate e2e variance."""
import os
import sys
import time

sys.path.insert(0, os.path.join(os.path.dirname(os.path.abspath(__file__)), ".."))
import numpy as np
import torch

import paper_2001_08289_b200 as fb

n = 2048
chi = np.asarray(fb.build_square_array(n, 0.5).chi)
cfgs = []
for sch, s1 in [("em", 0.1), ("em", 10.0), ("em", 1000.0), ("em_sub", 0.1), ("em_sub", 10.0), ("em_sub", 1000.0)]:
    sk = fb.SchemeKind(sch)
    cfgs.append(fb.SolverConfig(scheme=sk, sigma1=s1, tol=1e-10, max_iters=20000,
                                interval=fb.SpectralInterval(0.25, 4.0) if sk.substituted else None))
for step in range(4):
    pm = fb.PhaseMap(chi)
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    rows = []
    for cfg in cfgs:
        a = time.perf_counter()
        r = fb.solve(pm, cfg)
        _ = r.sigma_star
        torch.cuda.synchronize()
        rows.append((r.iterations, 1e3 * (time.perf_counter() - a), r.device_ms))
    tot = 1e3 * (time.perf_counter() - t0)
    print(f"step {step}: {tot:8.1f} ms  " + "  ".join(f"{it}:{w:.1f}/{d:.1f}" for it, w, d in rows), flush=True)
