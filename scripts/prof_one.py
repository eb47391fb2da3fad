"""Small profiling target: one solve at 2048^2 for a few iterations."""
import sys, os, argparse
sys.path.insert(0, os.path.join(os.path.dirname(__file__), ".."))
import paper_2001_08289_b200 as fb
ap = argparse.ArgumentParser()
ap.add_argument("--scheme", default="em_sub"); ap.add_argument("--n", type=int, default=2048)
ap.add_argument("--iters", type=int, default=3); ap.add_argument("--sigma1", type=float, default=10.0)
a = ap.parse_args()
pm = fb.build_square_array(a.n, 0.5)
sk = fb.SchemeKind(a.scheme)
cfg = fb.SolverConfig(scheme=sk, sigma1=a.sigma1, tol=1e-300, max_iters=a.iters,
                      interval=fb.SpectralInterval(0.25, 4.0) if sk.substituted else None)
r = fb.solve(pm, cfg)
print(a.scheme, a.n, r.iterations, r.sigma_star, r.device_ms)
