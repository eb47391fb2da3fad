import sys, time
sys.path.insert(0, "/root/repo")
import numpy as np
import paper_2001_08289_b200 as fb
from oracle import fftcond_oracle as O
for n, scheme, s1 in [(8,"basic",2.0),(64,"basic",10.0),(64,"em",10.0),(64,"basic_sub",10.0),(64,"em_sub",10.0),(256,"basic",10.0)]:
    pm = fb.build_square_array(n, 0.5)
    sk = fb.SchemeKind(scheme)
    cfg = fb.SolverConfig(scheme=sk, sigma1=s1, tol=1e-10, interval=fb.SpectralInterval(0.25,4.0) if sk.substituted else None)
    t0=time.perf_counter(); r = fb.solve(pm, cfg); t1=time.perf_counter()
    o = O.solve(pm.chi, scheme, s1, tol=1e-10, alpha=0.25, beta=4.0)
    print(n, scheme, r.status.value, o.status, r.iterations, o.iterations, r.sigma_star, o.sigma_star, abs(r.sigma_star-o.sigma_star)/abs(o.sigma_star), f"{(t1-t0)*1e3:.1f}ms dev={r.device_ms:.2f}ms launches={r.kernel_launches}", flush=True)
    if r.iterations and o.iterations:
        print("   res1", r.history.records[0].residual, o.history[0][2], " last", r.history.records[-1].residual, o.history[-1][2])
