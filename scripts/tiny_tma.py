import sys, os
sys.path.insert(0, os.path.join(os.path.dirname(__file__), ".."))
import paper_2001_08289_b200 as fb
from paper_2001_08289_b200.solver import _run_device
scheme = sys.argv[1] if len(sys.argv) > 1 else "basic"
os.environ["FFTC_NO_GRAPH"] = "1"
pm = fb.build_square_array(512, 0.5)
sk = fb.SchemeKind(scheme)
cfg = fb.SolverConfig(scheme=sk, sigma1=10.0, tol=1e-300, max_iters=2, interval=fb.SpectralInterval(0.25, 4) if sk.substituted else None)
r = _run_device(pm, cfg, want_fields=False)
print(scheme, r.iterations, r.sigma_star)
