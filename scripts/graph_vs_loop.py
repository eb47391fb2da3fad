"""Device time of solves with the CUDA-graph WHILE loop vs the host-chunked loop."""
import sys, os, time
sys.path.insert(0, os.path.join(os.path.dirname(__file__), ".."))
import torch
import paper_2001_08289_b200 as fb
from paper_2001_08289_b200.solver import _run_device
B = fb.SpectralInterval(0.25, 4.0)
cases = [("c1", 256, "basic", 10.0, 1e-8), ("c2s", 2048, "em_sub", 10.0, 1e-10), ("c5pt", 1024, "em_sub", 19.207 + 4.118j, 1e-8),
         ("tiny", 16, "em", 10.0, 1e-10)]
for name, n, scheme, s1, tol in cases:
    pm = fb.build_square_array(n, 0.5)
    sk = fb.SchemeKind(scheme)
    cfg = fb.SolverConfig(scheme=sk, sigma1=s1, tol=tol, max_iters=20000, interval=B if sk.substituted else None)
    res = {}
    for mode in ("graph", "loop"):
        if mode == "loop": os.environ["FFTC_NO_GRAPH"] = "1"
        else: os.environ.pop("FFTC_NO_GRAPH", None)
        _run_device(pm, cfg, want_fields=False)
        ts = []
        for _ in range(3):
            torch.cuda.synchronize(); t0 = time.perf_counter()
            r = _run_device(pm, cfg, want_fields=False)
            torch.cuda.synchronize(); ts.append((time.perf_counter() - t0) * 1e3)
        res[mode] = (r.iterations, r.sigma_star, min(ts), r.device_ms, r.kernel_launches)
    g, l = res["graph"], res["loop"]
    print(f"{name:5s} n={n:5d} it={g[0]}/{l[0]} same_sigma={g[1]==l[1]} wall graph {g[2]:9.2f} ms loop {l[2]:9.2f} ms  "
          f"per-iter graph {1e3*g[2]/g[0]:8.1f} us loop {1e3*l[2]/l[0]:8.1f} us  launches {g[4]}/{l[4]}", flush=True)
