import sys, os
sys.path.insert(0, os.path.join(os.path.dirname(__file__), ".."))
import paper_2001_08289_b200 as fb
from paper_2001_08289_b200 import native
from paper_2001_08289_b200.solver import _run_device
n = int(sys.argv[1]) if len(sys.argv) > 1 else 2048
import time, torch
# warm the clocks: ~2 s of solves before measuring
pmw = fb.build_square_array(n, 0.5)
cw = fb.SolverConfig(scheme=fb.SchemeKind.EYRE_MILTON, sigma1=10.0, tol=1e-300, max_iters=50)
t0 = time.time()
while time.time() - t0 < 2.0:
    _run_device(pmw, cw, want_fields=False)
for scheme in ("basic", "em", "basic_sub", "em_sub"):
    pm = fb.build_square_array(n, 0.5)
    sk = fb.SchemeKind(scheme)
    cfg = fb.SolverConfig(scheme=sk, sigma1=10.0, tol=1e-300, max_iters=30, interval=fb.SpectralInterval(0.25, 4) if sk.substituted else None)
    _run_device(pm, cfg, want_fields=False)
    native.profile(True)
    r = _run_device(pm, cfg, want_fields=False)
    st = native.kernel_stats(); native.profile(False)
    print(n, f"{scheme:9s}", {k: f"{1e3*v[1]/v[0]:.1f}" for k, v in st.items() if k.startswith("sweep")}, flush=True)
