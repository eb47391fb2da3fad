"""Where the end-to-end C3 step goes: solve with fields, then each field's
read-back, timed separately (wall clock after a device synchronise)."""
import os
import sys
import time

sys.path.insert(0, os.path.join(os.path.dirname(__file__), ".."))
import numpy as np  # noqa: E402
import torch  # noqa: E402

import paper_2001_08289_b200 as fb  # noqa: E402

n = int(sys.argv[1]) if len(sys.argv) > 1 else 512
pm = fb.build_cube_array(n, 2 * int(round(0.63 * n / 2)))
chi = np.array(pm.chi)
cfg = fb.SolverConfig(scheme=fb.SchemeKind.EYRE_MILTON_SUB, sigma1=100.0, tol=1e-8, max_iters=20000,
                      e0=(1.0, 0.0, 0.0), interval=fb.SpectralInterval(0.25, 4.0))
for rep in range(3):
    t0 = time.perf_counter()
    p = fb.PhaseMap(chi)
    t1 = time.perf_counter()
    r = fb.solve(p, cfg)
    torch.cuda.synchronize()
    t2 = time.perf_counter()
    ts = []
    for f in (r.E_field, r.J_field, r.aug_field.S, r.aug_field.T):
        a = time.perf_counter()
        _ = f.data
        ts.append(time.perf_counter() - a)
    t3 = time.perf_counter()
    print(f"rep {rep}: phasemap {1e3*(t1-t0):.0f} ms, solve {1e3*(t2-t1):.0f} ms (device {r.device_ms:.0f} ms, "
          f"{r.iterations} it), readback {[round(1e3*x) for x in ts]} ms total {1e3*(t3-t2):.0f} ms", flush=True)
    del r, p
