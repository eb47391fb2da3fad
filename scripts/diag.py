"""Diagnose parity of selected golden cases on the GPU (prints per-k deltas)."""
import sys, os
sys.path.insert(0, os.path.join(os.path.dirname(__file__), "..", "tests"))
sys.path.insert(0, os.path.join(os.path.dirname(__file__), ".."))
import numpy as np
from golden_io import load_group
from test_gpu_parity import run_case
for spec in sys.argv[1:]:
    grp, name = spec.split(":")
    g = load_group(grp)[name]
    r = run_case(g["case"])
    h = g["history"]
    dev = np.array([[rec.sigma_star.real, rec.sigma_star.imag, rec.residual] for rec in r.history])
    print(f"== {name}: dev {r.status.value} {r.iterations} | gold {g['status']} {g['iterations']} | s* {r.sigma_star} vs {g['sigma_star']}")
    n = min(len(h), len(dev))
    if n:
        gs = h[:n,1]+1j*h[:n,2]; ds = dev[:n,0]+1j*dev[:n,1]
        srel = np.abs(ds-gs)/np.maximum(np.abs(gs),1e-300); rrel = np.abs(dev[:n,2]-h[:n,3])/np.abs(h[:n,3])
        for k in sorted(set([0,1,2,3,n//4,n//2,3*n//4,n-3,n-2,n-1])):
            if 0 <= k < n:
                print(f"  k={k+1:5d} gold s*={gs[k]:.6e} res={h[k,3]:.6e} | dev s*={ds[k]:.6e} res={dev[k,2]:.6e} | srel={srel[k]:.2e} rrel={rrel[k]:.2e}")
    print("  meanE dev", r.mean_E, "gold", g["mean_E"])
    print("  meanJ dev", r.mean_J, "gold", g["mean_J"])
