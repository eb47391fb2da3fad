"""Per-kernel device time of one 3-D iteration (profiled solve, max_iters
small, tol tiny), for each scheme at n^3.  Usage: python scripts/kernels_3d.py [n] [schemes]"""
import os
import sys
import time

sys.path.insert(0, os.path.join(os.path.dirname(__file__), ".."))
import paper_2001_08289_b200 as fb  # noqa: E402
from paper_2001_08289_b200 import native  # noqa: E402
from paper_2001_08289_b200.solver import _run_device  # noqa: E402

n = int(sys.argv[1]) if len(sys.argv) > 1 else 512
schemes = sys.argv[2].split(",") if len(sys.argv) > 2 else ["basic", "em_sub"]
pm = fb.build_cube_array(n, 2 * int(0.315 * n))
iv = fb.SpectralInterval(0.25, 4.0)
cw = fb.SolverConfig(scheme=fb.SchemeKind.BASIC, sigma1=10.0, tol=1e-300, max_iters=8, e0=(1.0, 0.0, 0.0))
t0 = time.time()
while time.time() - t0 < 2.0:
    _run_device(pm, cw, want_fields=False)
for scheme in schemes:
    sk = fb.SchemeKind(scheme)
    cfg = fb.SolverConfig(scheme=sk, sigma1=100.0, tol=1e-300, max_iters=6, e0=(1.0, 0.0, 0.0),
                          interval=iv if sk.substituted else None)
    native.profile(True)
    _run_device(pm, cfg, want_fields=False)
    st = native.kernel_stats()
    native.profile(False)
    tot = sum(v[1] for k, v in st.items() if k not in ("init", "finalize")) / 6
    vox = n ** 3
    print(f"{n}^3 {scheme:9s} iter {tot:.2f} ms = {vox / (tot / 1e3) / 1e9:.2f} G vox-it/s |",
          " ".join(f"{k} {1e3 * v[1] / v[0]:.0f}us x{v[0] // 6}" for k, v in st.items() if k not in ("init", "finalize")),
          flush=True)
