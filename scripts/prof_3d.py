"""A few 3-D iterations for ncu (non-graph launches): n^3 cube, scheme."""
import os
import sys

sys.path.insert(0, os.path.join(os.path.dirname(__file__), ".."))
os.environ.setdefault("FFTC_NO_GRAPH", "1")
import paper_2001_08289_b200 as fb  # noqa: E402
from paper_2001_08289_b200.solver import _run_device  # noqa: E402

n = int(sys.argv[1]) if len(sys.argv) > 1 else 512
scheme = sys.argv[2] if len(sys.argv) > 2 else "basic"
sk = fb.SchemeKind(scheme)
pm = fb.build_cube_array(n, 2 * int(0.315 * n))
cfg = fb.SolverConfig(scheme=sk, sigma1=100.0, tol=1e-300, max_iters=3, e0=(1.0, 0.0, 0.0),
                      interval=fb.SpectralInterval(0.25, 4.0) if sk.substituted else None)
_run_device(pm, cfg, want_fields=False)
print("done")
