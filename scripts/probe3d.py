import sys, os
sys.path.insert(0, os.path.join(os.path.dirname(__file__), ".."))
import numpy as np
import paper_2001_08289_b200 as fb
from oracle import fftcond_oracle as O
for shape in [(2,16,16),(4,16,16),(16,16,16),(16,16,2),(16,2,16),(8,16,32),(32,16,8)]:
    chi = np.zeros(shape, bool)
    chi[tuple(slice(n//4, n//4 + n//2) for n in shape)] = True
    for scheme in ("basic", "em"):
        cfg = fb.SolverConfig(scheme=fb.SchemeKind(scheme), sigma1=10.0, tol=1e-8, max_iters=3, e0=(1.0, 0.3, 0.2))
        r = fb.solve(fb.PhaseMap(chi), cfg)
        o = O.solve(chi, scheme, 10.0, tol=1e-8, max_iters=3, e0=(1.0, 0.3, 0.2))
        print(shape, scheme, [f"{x.residual:.6f}" for x in r.history], [f"{x[2]:.6f}" for x in o.history], flush=True)
