import sys, os
sys.path.insert(0, os.path.join(os.path.dirname(__file__), ".."))
import torch
import paper_2001_08289_b200 as fb
from paper_2001_08289_b200 import native
from paper_2001_08289_b200.solver import _run_device
for n, scheme in ((16, "em"), (256, "basic"), (1024, "em_sub")):
    pm = fb.build_square_array(n, 0.5)
    sk = fb.SchemeKind(scheme)
    cfg = fb.SolverConfig(scheme=sk, sigma1=10.0, tol=1e-10, max_iters=50, interval=fb.SpectralInterval(0.25, 4) if sk.substituted else None)
    _run_device(pm, cfg, want_fields=False)
    native.profile(True)
    r = _run_device(pm, cfg, want_fields=False)
    st = native.kernel_stats(); native.profile(False)
    print(n, scheme, r.iterations, {k: f"{1e3*v[1]/v[0]:.1f}us x{v[0]}" for k, v in st.items()}, flush=True)
