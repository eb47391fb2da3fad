"""Per-call wall vs device time of repeated solves (host overhead check)."""
import sys, os, time
sys.path.insert(0, os.path.join(os.path.dirname(__file__), ".."))
import torch
import paper_2001_08289_b200 as fb
from paper_2001_08289_b200.solver import _solve_aug, _solve_h
n = int(sys.argv[1]) if len(sys.argv) > 1 else 2048
pm = fb.build_square_array(n, 0.5)
t0 = time.perf_counter(); import paper_2001_08289_b200.native as nat; nat.lib(); print("lib load", time.perf_counter()-t0)
for scheme, s1 in [("em", 10.0), ("em_sub", 10.0)] * 3:
    sk = fb.SchemeKind(scheme)
    cfg = fb.SolverConfig(scheme=sk, sigma1=s1, tol=1e-10, max_iters=20000,
                          interval=fb.SpectralInterval(0.25, 4.0) if sk.substituted else None)
    torch.cuda.synchronize(); t0 = time.perf_counter()
    r = (_solve_aug if sk.substituted else _solve_h)(pm, cfg, sk.accelerated, want_fields=False)
    torch.cuda.synchronize(); wall = (time.perf_counter() - t0) * 1e3
    print(f"{scheme:7s} it={r.iterations:4d} wall={wall:8.2f} ms device={r.device_ms:8.2f} ms launches={r.kernel_launches}", flush=True)
