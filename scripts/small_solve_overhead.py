"""Host overhead of one solve on small grids: wall time per fb.solve / device-path
solve vs the device time of its iteration loop (C1-sized problems)."""
import os
import sys
import time

sys.path.insert(0, os.path.join(os.path.dirname(os.path.abspath(__file__)), ".."))
import torch

import paper_2001_08289_b200 as fb
from paper_2001_08289_b200.solver import _solve_h

for n, scheme in ((256, "basic"), (256, "em"), (1024, "em")):
    pm = fb.build_square_array(n, 0.5)
    sk = fb.SchemeKind(scheme)
    cfg = fb.SolverConfig(scheme=sk, sigma1=10.0, tol=1e-8)
    for _ in range(3):
        fb.solve(pm, cfg)
    torch.cuda.synchronize()
    reps = 20
    t0 = time.perf_counter()
    for _ in range(reps):
        r = _solve_h(pm, cfg, sk.accelerated, want_fields=False)
    torch.cuda.synchronize()
    t1 = time.perf_counter()
    for _ in range(reps):
        r2 = fb.solve(pm, cfg)
        _ = r2.sigma_star
    torch.cuda.synchronize()
    t2 = time.perf_counter()
    print(f"{n}^2 {scheme:6s} it={r.iterations:4d} device {r.device_ms:7.3f} ms  device-path wall {1e3*(t1-t0)/reps:7.3f} ms"
          f"  public API wall {1e3*(t2-t1)/reps:7.3f} ms", flush=True)
