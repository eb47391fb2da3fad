"""Small profiling target: one 3-D solve for a few iterations outside the CUDA
graph (FFTC_NO_GRAPH; ncu cannot profile kernels of a conditional graph).
Usage: FFTC_NO_GRAPH=1 python scripts/prof_3d_one.py [--n 512] [--scheme em_sub] [--iters 2] [--workload c3|c4]"""
import argparse
import os
import sys

sys.path.insert(0, os.path.join(os.path.dirname(__file__), ".."))
import paper_2001_08289_b200 as fb  # noqa: E402
from paper_2001_08289_b200 import cell  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--n", type=int, default=512)
ap.add_argument("--scheme", default="em_sub")
ap.add_argument("--iters", type=int, default=2)
ap.add_argument("--workload", default="c3")
a = ap.parse_args()
if a.workload == "c3":
    pm = fb.build_cube_array(a.n, 2 * int(round(0.63 * a.n / 2)))
    e0, s1 = (1.0, 0.0, 0.0), 100.0
else:
    pm = cell.c4_phase_map(a.n)
    e0, s1 = (3 ** -0.5,) * 3, 50.0
sk = fb.SchemeKind(a.scheme)
cfg = fb.SolverConfig(scheme=sk, sigma1=s1, tol=1e-300, max_iters=a.iters, e0=e0,
                      interval=fb.SpectralInterval(0.25, 4.0) if sk.substituted else None)
r = fb.solve(pm, cfg, fields=False)
print(a.workload, a.scheme, a.n, r.iterations, r.sigma_star, f"{r.device_ms:.1f} ms", r.kernel_launches, "launches")
