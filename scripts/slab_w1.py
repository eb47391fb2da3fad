"""Single GPU: the monolithic 3-D solve vs the slab path at world 1 with the
fused transposes (z pass on the y-slab copy, where z lines are near)."""
import os
import sys
import time

sys.path.insert(0, os.path.join(os.path.dirname(__file__), ".."))
import torch  # noqa: E402

import paper_2001_08289_b200 as fb  # noqa: E402
from paper_2001_08289_b200.slab import solve_slab  # noqa: E402


class SelfComm:
    rank, world = 0, 1

    def all_reduce(self, t, group=None):
        pass

    def all_to_all_single(self, out, inp, group=None):
        out.copy_(inp)

    def barrier(self):
        torch.cuda.current_stream().synchronize()

    def all_gather_object(self, obj):
        return [obj]


n = int(sys.argv[1]) if len(sys.argv) > 1 else 512
scheme = sys.argv[2] if len(sys.argv) > 2 else "basic"
pm = fb.build_random_medium(n, 3, seed=20260809, smoothing=4.0, fraction=0.3)
sk = fb.SchemeKind(scheme)
cfg = fb.SolverConfig(scheme=sk, sigma1=50.0, tol=1e-300, max_iters=int(sys.argv[3]) if len(sys.argv) > 3 else 30,
                      e0=(3 ** -0.5,) * 3, interval=fb.SpectralInterval(0.25, 4.0) if sk.substituted else None)
variants = {"monolithic": lambda: fb.solve(pm, cfg, fields=False),
            "slab-w1-fused": lambda: solve_slab(pm.chi, cfg, comm=SelfComm(), fused=True),
            "slab-w1-a2a": lambda: solve_slab(pm.chi, cfg, comm=SelfComm(), fused=False)}
# one variant per process (argv[4]) at large sizes: the stream-ordered pool keeps its memory
only = sys.argv[4].split(",") if len(sys.argv) > 4 else list(variants)
for name, fn in ((k, v) for k, v in variants.items() if k in only):
    fn()
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    r = fn()
    torch.cuda.synchronize()
    dt = time.perf_counter() - t0
    it = r.iterations if hasattr(r, "iterations") else r["iterations"]
    fused = r.get("fused") if isinstance(r, dict) else None
    print(f"{n}^3 {scheme} {name:14s} {1e3 * dt / it:8.2f} ms/iter ({it} iters, fused={fused})", flush=True)
    if os.environ.get("SLAB_STATS"):  # per-kernel device time of one more run (profile mode: events around every launch)
        from paper_2001_08289_b200 import native
        native.profile(True)
        fn()
        st = native.kernel_stats()
        native.profile(False)
        print("   ", " ".join(f"{k} {1e3 * v[1] / max(v[0], 1):.0f}us x{v[0]}" for k, v in st.items()), flush=True)
