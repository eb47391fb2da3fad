"""BASELINE configs 3 and 4 on one GPU: C3 512^3 cube em_sub sigma1=100, C4 1024^3
random medium (basic, and em_sub if it fits).  Reports iterations, sigma*,
device time and voxel-iterations/s."""
import sys, os, time, json, argparse
sys.path.insert(0, os.path.join(os.path.dirname(__file__), ".."))
import numpy as np, torch
import paper_2001_08289_b200 as fb
from paper_2001_08289_b200.solver import _solve_aug, _solve_h

ap = argparse.ArgumentParser()
ap.add_argument("--n3", type=int, default=512); ap.add_argument("--n4", type=int, default=1024)
ap.add_argument("--which", default="c3,c4"); ap.add_argument("--max-iters", type=int, default=20000)
a = ap.parse_args()
B = fb.SpectralInterval(0.25, 4.0)
out = {}

def run(name, pm, scheme, s1, e0):
    sk = fb.SchemeKind(scheme)
    cfg = fb.SolverConfig(scheme=sk, sigma1=s1, e0=e0, tol=1e-8, max_iters=a.max_iters, interval=B if sk.substituted else None)
    torch.cuda.synchronize(); t0 = time.perf_counter()
    r = (_solve_aug if sk.substituted else _solve_h)(pm, cfg, sk.accelerated, want_fields=False)
    torch.cuda.synchronize(); wall = time.perf_counter() - t0
    n = pm.chi.size
    rec = dict(scheme=scheme, grid=list(pm.grid), status=r.status.value, iterations=r.iterations,
               sigma_star=[r.sigma_star.real, r.sigma_star.imag], device_ms=r.device_ms, wall_s=wall,
               gvox_it_per_s=n * r.iterations / (r.device_ms / 1e3) / 1e9,
               mem_peak_gb=torch.cuda.max_memory_allocated() / 1e9)
    print(name, json.dumps(rec), flush=True)
    out[name] = rec

if "c3" in a.which:
    n = a.n3
    side = int(round(0.63 * n)) & ~1          # 322 at 512 (0.63*512 = 322.56 not representable)
    run(f"c3_{n}_em_sub", fb.build_cube_array(n, side), "em_sub", 100.0, (1.0, 0.0, 0.0))
if "c4" in a.which:
    n = a.n4
    t0 = time.perf_counter()
    rng = np.random.default_rng(20260809)
    u = torch.from_numpy(rng.random((n, n, n))).cuda()
    k = torch.fft.fftfreq(n, device="cuda", dtype=torch.float64)
    k2 = k[:, None, None] ** 2 + k[None, :, None] ** 2 + k[None, None, :] ** 2
    s = torch.fft.ifftn(torch.fft.fftn(u) * torch.exp(-2.0 * np.pi ** 2 * 16.0 * k2)).real
    del u, k2
    thr = torch.kthvalue(s.flatten().cpu(), int(0.30 * s.numel())).values.item()
    chi = (s <= thr).cpu().numpy()
    del s; torch.cuda.empty_cache()
    print(f"c4 chi built in {time.perf_counter()-t0:.1f}s, f={chi.mean():.4f}", flush=True)
    pm = fb.PhaseMap(chi)
    e0 = (1 / np.sqrt(3),) * 3
    run(f"c4_{n}_basic", pm, "basic", 50.0, e0)
    if "em_sub" in a.which:
        run(f"c4_{n}_em_sub", pm, "em_sub", 50.0, e0)
json.dump(out, open("gpurun_out/run_3d.json", "w"), indent=1)
