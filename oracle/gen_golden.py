"""Generate golden fixtures from the LIVE reference -- TEST INFRASTRUCTURE ONLY.

Runs only in the dev container, where ``/root/reference/pkg/src`` is
importable.  Every fixture is the output of the unmodified reference
``fftcond.solve`` (solvers.py:489-491) on a seeded/synthetic input, frozen
as JSON under ``tests/golden/``.  3-D fixtures (``group == "3d"``) cannot
come from the reference (it is 2-D only, geometry.py:33-34); they come from
``oracle/fftcond_oracle.py`` and say so in their ``source`` field.

Usage:  python oracle/gen_golden.py <group> [<group> ...] [--jobs N]
Groups: edge, c1, c2small, c5small, c2full, c5full, 3d, fields, general, big,
        c3red, c4red, c3first, c3full, c4first
"""

from __future__ import annotations

import argparse
import json
import math
import os
import sys
import time
from concurrent.futures import ProcessPoolExecutor

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
REPO = os.path.dirname(HERE)
# FFTC_GOLDEN_DIR: write fixtures elsewhere (the GPU box host writes under
# gpurun_out/); FFTC_REF_SRC: where the live reference is importable from --
# the read-only tree here, or its unmodified install under baseline/_ref on
# the GPU box host (pip install --target)
GOLDEN = os.environ.get("FFTC_GOLDEN_DIR") or os.path.join(REPO, "tests", "golden")
REF_SRC = os.environ.get("FFTC_REF_SRC") or (
    "/root/reference/pkg/src" if os.path.isdir("/root/reference/pkg/src") else os.path.join(REPO, "baseline", "_ref"))

ALPHA, BETA = 0.25, 4.0  # configs/compare.cfg:14-15 (the reference's only interval)
SEED = 20260809  # selftest.py:38


def c5_points(count: int = 256, seed: int = SEED):
    """Config-5 sweep points: Re in [-50, 50] minus [-beta, -alpha], Im in [0.01, 10]."""
    rng = np.random.default_rng(seed)
    pts = []
    while len(pts) < count:
        re = rng.uniform(-50.0, 50.0)
        im = rng.uniform(0.01, 10.0)
        if -BETA <= re <= -ALPHA:
            continue
        pts.append(complex(re, im))
    return pts


def _chi(geom):
    kind = geom["kind"]
    if kind == "square":
        n = geom["n"]
        m = geom["side"]
        chi = np.zeros((n, n), dtype=bool)
        lo = (n - m) // 2
        chi[lo:lo + m, lo:lo + m] = True
        return chi
    if kind == "uniform":
        return np.full((geom["ny"], geom["nx"]), bool(geom["phase1"]))
    if kind == "laminate_x":  # strips varying along x (tests/test_solvers.py:48-55)
        chi = np.zeros((geom["n"], geom["n"]), dtype=bool)
        chi[:, ::2] = True
        return chi
    if kind == "laminate_y":
        chi = np.zeros((geom["n"], geom["n"]), dtype=bool)
        chi[::2, :] = True
        return chi
    if kind == "rect":  # centred rectangle on an ny x nx grid
        ny, nx, my, mx = geom["ny"], geom["nx"], geom["my"], geom["mx"]
        chi = np.zeros((ny, nx), dtype=bool)
        chi[(ny - my) // 2:(ny - my) // 2 + my, (nx - mx) // 2:(nx - mx) // 2 + mx] = True
        return chi
    if kind == "random":
        rng = np.random.default_rng(geom["seed"])
        return rng.random((geom["ny"], geom["nx"])) < geom["frac"]
    if kind == "cube":
        n, m, d = geom["n"], geom["side"], 3
        chi = np.zeros((n,) * d, dtype=bool)
        lo = (n - m) // 2
        chi[lo:lo + m, lo:lo + m, lo:lo + m] = True
        return chi
    if kind == "embed2d":  # z-invariant stack of a 2-D square cell
        c2 = _chi(geom["base"])
        return np.repeat(c2[None], geom["nz"], axis=0)
    if kind == "random3d":
        rng = np.random.default_rng(geom["seed"])
        return rng.random((geom["n"],) * 3) < geom["frac"]
    if kind == "c4medium":  # BASELINE config-4 recipe (cell.build_random_medium; frozen file at 1024^3)
        sys.path.insert(0, REPO)
        from paper_2001_08289_b200 import cell

        return np.asarray(cell.c4_phase_map(geom["n"]).chi)
    raise ValueError(kind)


def cplx(z):
    z = complex(z)
    return [z.real, z.imag]


def run_case(case):
    """Solve one case and return the fixture dict."""
    sys.path.insert(0, REF_SRC)
    sys.path.insert(0, REPO)
    chi = _chi(case["geom"])
    t0 = time.perf_counter()
    if chi.ndim == 2 and not case.get("force_oracle"):
        import fftcond as fc
        from fftcond.spectral_ops import _mean_vec

        sch = fc.SchemeKind(case["scheme"])
        kw = dict(scheme=sch, sigma1=complex(*case["sigma1"]), tol=case["tol"],
                  max_iters=case["max_iters"])
        if sch.substituted:
            kw["interval"] = fc.SpectralInterval(ALPHA, BETA)
        if case.get("e0") is not None:
            kw["e0"] = tuple(complex(*v) for v in case["e0"])
        if case.get("sigma0_override") is not None:
            kw["sigma0_override"] = complex(*case["sigma0_override"])
        r = fc.solve(fc.PhaseMap(chi), fc.SolverConfig(**kw))
        hist = [[h.iteration, h.sigma_star.real, h.sigma_star.imag, h.residual]
                for h in r.history]
        E, J = r.E_field.data, r.J_field.data
        out = dict(status=r.status.value, degenerate_flux=bool(r.degenerate_flux),
                   iterations=r.iterations, sigma_star=cplx(r.sigma_star), history=hist,
                   mean_E=[cplx(v) for v in _mean_vec(E)], mean_J=[cplx(v) for v in _mean_vec(J)],
                   source=f"reference fftcond (live, {REF_SRC})")
        aug = r.aug_field
        fields = dict(E=E, J=J)
        if aug is not None:
            fields.update(S=aug.S.data, T=aug.T.data)
    elif case.get("lean"):
        # bounded-memory threaded restatement, bit-identical to fftcond_oracle
        # (tests/test_oracle.py::test_lean_oracle_bitwise)
        from oracle import fftcond_oracle as O
        from oracle import lean_oracle as LO

        e0 = None if case.get("e0") is None else [complex(*v) for v in case["e0"]]
        keep = bool(case.get("keep_fields", True))
        r = LO.solve(chi, case["scheme"], complex(*case["sigma1"]), e0=e0, tol=case["tol"],
                     max_iters=case["max_iters"], alpha=ALPHA, beta=BETA, keep_fields=keep)
        hist = [[k, s.real, s.imag, res] for k, s, res in r.history]
        out = dict(status=r.status, degenerate_flux=bool(r.degenerate_flux),
                   iterations=r.iterations, sigma_star=cplx(r.sigma_star), history=hist,
                   source="oracle/lean_oracle.py (bounded-memory form of the d-generic restatement; "
                          "no 3-D reference exists)")
        fields = {}
        if keep:
            out["mean_E"] = [cplx(v) for v in O.component_means(r.E)]
            out["mean_J"] = [cplx(v) for v in O.component_means(r.J)]
            fields = dict(E=r.E, J=r.J)
            if r.aug is not None:
                fields.update(S=r.aug[1], T=r.aug[2])
    else:
        from oracle import fftcond_oracle as O

        e0 = None if case.get("e0") is None else [complex(*v) for v in case["e0"]]
        ov = None if case.get("sigma0_override") is None else complex(*case["sigma0_override"])
        r = O.solve(chi, case["scheme"], complex(*case["sigma1"]), e0=e0, tol=case["tol"],
                    max_iters=case["max_iters"], alpha=ALPHA, beta=BETA, sigma0_override=ov)
        hist = [[k, s.real, s.imag, res] for k, s, res in r.history]
        out = dict(status=r.status, degenerate_flux=bool(r.degenerate_flux),
                   iterations=r.iterations, sigma_star=cplx(r.sigma_star), history=hist,
                   mean_E=[cplx(v) for v in O.component_means(r.E)],
                   mean_J=[cplx(v) for v in O.component_means(r.J)],
                   source="oracle/fftcond_oracle.py d-generic restatement (no 3-D reference exists)")
        fields = dict(E=r.E, J=r.J)
        if r.aug is not None:
            fields.update(S=r.aug[1], T=r.aug[2])
    out["cpu_seconds"] = time.perf_counter() - t0
    # size-independent field summaries: sum |F|^2 over the grid, per component
    out["field_sumsq"] = {k: [float(np.sum(np.abs(v[c]) ** 2)) for c in range(v.shape[0])]
                          for k, v in fields.items()}
    if chi.ndim == 3 and chi.shape[0] >= 128:
        import hashlib

        out["chi_sha256"] = hashlib.sha256(np.packbits(chi.reshape(-1), bitorder="little").tobytes()).hexdigest()
    out["case"] = case
    if case.get("save_fields"):
        path = os.path.join(GOLDEN, "fields", case["name"] + ".npz")
        os.makedirs(os.path.dirname(path), exist_ok=True)
        np.savez_compressed(path, chi=chi, **fields)
        out["fields_file"] = os.path.relpath(path, GOLDEN)
    return out


def C(name, geom, scheme, sigma1, tol=1e-8, max_iters=1000, **kw):
    s = complex(sigma1)
    return dict(name=name, geom=geom, scheme=scheme, sigma1=[s.real, s.imag], tol=tol,
                max_iters=max_iters, **kw)


def sq(n, frac_side=0.5):
    m = int(round(n * frac_side))
    return dict(kind="square", n=n, side=m)


def groups():
    g = {}
    edge = []
    for sch in ("basic", "em", "basic_sub", "em_sub"):
        edge.append(C(f"edge_phase2_{sch}", dict(kind="uniform", nx=8, ny=8, phase1=False), sch, 3.0))
        edge.append(C(f"edge_contrastfree_{sch}", sq(8), sch, 1.0, save_fields=True))
        edge.append(C(f"edge_tiny2_{sch}", dict(kind="random", ny=2, nx=2, frac=0.5, seed=3), sch, 2.0,
                      tol=1e-12, max_iters=500))
        edge.append(C(f"edge_4x4_{sch}", dict(kind="square", n=4, side=2), sch, 2.0, tol=1e-12,
                      max_iters=500, save_fields=True))
        edge.append(C(f"edge_rect16x32_{sch}", dict(kind="rect", ny=16, nx=32, my=8, mx=12), sch,
                      3.0 + 1.0j, tol=1e-11, max_iters=2000, save_fields=True))
        edge.append(C(f"edge_rect32x8_{sch}", dict(kind="rect", ny=32, nx=8, my=10, mx=4), sch,
                      7.0, tol=1e-11, max_iters=2000, save_fields=True))
        edge.append(C(f"edge_e0y_{sch}", sq(16), sch, 5.0, tol=1e-11, max_iters=2000,
                      e0=[[0.0, 0.0], [1.0, 0.0]]))
        edge.append(C(f"edge_e0complex_{sch}", sq(16), sch, 2.0 - 0.5j, tol=1e-11, max_iters=2000,
                      e0=[[0.6, 0.2], [-0.3, 0.7]], save_fields=True))
        edge.append(C(f"edge_random32_{sch}", dict(kind="random", ny=32, nx=32, frac=0.3, seed=SEED),
                      sch, 20.0, tol=1e-10, max_iters=5000, save_fields=True))
        edge.append(C(f"edge_maxiters_{sch}", sq(16), sch, 50.0, tol=1e-14, max_iters=3))
    edge.append(C("edge_laminate_series", dict(kind="laminate_x", n=8), "basic", 3.0, tol=1e-12))
    edge.append(C("edge_laminate_parallel", dict(kind="laminate_y", n=8), "basic", 3.0, tol=1e-12))
    edge.append(C("edge_geom_series", dict(kind="uniform", nx=8, ny=8, phase1=True), "basic_sub",
                  2.0, tol=1e-13, max_iters=200))
    edge.append(C("edge_dense8", sq(8), "basic", 2.0, tol=1e-13, max_iters=2000, save_fields=True))
    edge.append(C("edge_degenerate", sq(8), "basic", -3.0, max_iters=10))
    edge.append(C("edge_diverge_guard", sq(16), "basic", 2.0, max_iters=500,
                  sigma0_override=[0.01, 0.0]))
    edge.append(C("edge_em_override", sq(8), "em", -0.5, max_iters=30, sigma0_override=[1.0, 0.0]))
    edge.append(C("edge_insulating_emsub", sq(32), "em_sub", 0.0, tol=2e-3, max_iters=100))
    edge.append(C("edge_em_sub_negative", sq(64), "em_sub", -30.065 + 4.945j, max_iters=1000))
    g["edge"] = edge

    g["c1"] = [C("c1_basic_256_s10", sq(256), "basic", 10.0, tol=1e-8)]

    small = []
    for n in (64, 256):
        for sch in ("basic", "em", "basic_sub", "em_sub"):
            for s1 in (0.1, 10.0, 1000.0):
                small.append(C(f"c2s_{sch}_{n}_s{s1:g}", sq(n), sch, s1, tol=1e-10, max_iters=20000))
    g["c2small"] = small

    g["c2full"] = [C(f"c2_{sch}_2048_s{s1:g}", sq(2048), sch, s1, tol=1e-10, max_iters=20000)
                   for s1 in (0.1, 10.0, 1000.0) for sch in ("em", "em_sub")]

    pts = c5_points()
    g["c5small"] = [C(f"c5s_64_p{i:03d}", sq(64), "em_sub", s, tol=1e-8, max_iters=1000)
                    for i, s in enumerate(pts)]
    g["c5full"] = [C(f"c5_1024_p{i:03d}", sq(1024), "em_sub", s, tol=1e-8, max_iters=1000)
                   for i, s in enumerate(pts)]

    three = []
    for sch in ("basic", "em", "basic_sub", "em_sub"):
        three.append(C(f"3d_embed_{sch}", dict(kind="embed2d", nz=2, base=sq(16)), sch, 10.0,
                       tol=1e-10, max_iters=5000))
        three.append(C(f"3d_cube16_{sch}", dict(kind="cube", n=16, side=10), sch, 100.0,
                       tol=1e-8, max_iters=5000, e0=[[1, 0], [0, 0], [0, 0]], save_fields=True))
        three.append(C(f"3d_random16_{sch}", dict(kind="random3d", n=16, frac=0.3, seed=SEED), sch,
                       50.0, tol=1e-8, max_iters=5000,
                       e0=[[1 / math.sqrt(3), 0]] * 3))
    three.append(C("3d_cube32_em_sub", dict(kind="cube", n=32, side=20), "em_sub", 100.0, tol=1e-8,
                   max_iters=5000))
    three.append(C("3d_cube64_em_sub", dict(kind="cube", n=64, side=40), "em_sub", 100.0, tol=1e-8,
                   max_iters=5000))
    three.append(C("3d_random64_basic", dict(kind="random3d", n=64, frac=0.3, seed=SEED), "basic",
                   50.0, tol=1e-8, max_iters=5000, e0=[[1 / math.sqrt(3), 0]] * 3))
    for c in three:
        c["force_oracle"] = True
    g["3d"] = three

    # BASELINE configs 3 and 4 at their recipes: full solves on reduced grids
    # (SURVEY 8c), first iterations at the stated sizes (c3first here,
    # c4first on the GPU box host: 1024^3 needs ~165 GB)
    ex = [[1.0, 0.0], [0.0, 0.0], [0.0, 0.0]]
    ed = [[1 / math.sqrt(3), 0.0]] * 3
    c3side = lambda n: 2 * int(round(0.63 * n / 2))  # noqa: E731  (nearest even side; 322 at 512)
    g["c3red"] = [C(f"c3_cube{n}_em_sub", dict(kind="cube", n=n, side=c3side(n)), "em_sub", 100.0, tol=1e-8,
                    max_iters=20000, e0=ex, lean=True) for n in (128, 256)]
    g["c4red"] = [C(f"c4_random{n}_{sch}", dict(kind="c4medium", n=n), sch, 50.0, tol=1e-8, max_iters=20000,
                    e0=ed, lean=True) for n in (128, 256) for sch in ("basic", "em_sub")]
    g["c3first"] = [C("c3_cube512_em_sub_first4", dict(kind="cube", n=512, side=c3side(512)), "em_sub", 100.0,
                      tol=1e-8, max_iters=4, e0=ex, lean=True, keep_fields=False)]
    g["c3full"] = [C("c3_cube512_em_sub", dict(kind="cube", n=512, side=c3side(512)), "em_sub", 100.0,
                     tol=1e-8, max_iters=20000, e0=ex, lean=True, keep_fields=False)]
    g["c4first"] = [C("c4_random1024_basic_first3", dict(kind="c4medium", n=1024), "basic", 50.0, tol=1e-8,
                      max_iters=3, e0=ed, lean=True, keep_fields=False)]

    # grids outside the fused transforms' power-of-two lengths (the general
    # path: pointwise kernels around cuFFT); 2-D from the live reference
    gen = []
    for sch in ("basic", "em", "basic_sub", "em_sub"):
        gen.append(C(f"gen_sq6_{sch}", dict(kind="square", n=6, side=2), sch, 10.0, tol=1e-10, max_iters=2000))
        gen.append(C(f"gen_sq48_{sch}", sq(48), sch, 10.0, tol=1e-10, max_iters=5000))
        gen.append(C(f"gen_sq96_{sch}_s1000", sq(96), sch, 1000.0, tol=1e-8, max_iters=20000))
        gen.append(C(f"gen_rect40x24_{sch}", dict(kind="rect", ny=40, nx=24, my=10, mx=8), sch, 3.0 + 1.0j,
                     tol=1e-10, max_iters=5000))
        gen.append(C(f"gen_random30x50_{sch}", dict(kind="random", ny=30, nx=50, frac=0.3, seed=SEED), sch,
                     20.0 + 5.0j, tol=1e-10, max_iters=5000))
    three_gen = []
    for sch in ("basic", "em", "basic_sub", "em_sub"):
        three_gen.append(C(f"gen3d_random12_{sch}", dict(kind="random3d", n=12, frac=0.3, seed=SEED), sch, 50.0,
                           tol=1e-8, max_iters=5000, e0=[[1 / math.sqrt(3), 0]] * 3))
        three_gen.append(C(f"gen3d_cube24_{sch}", dict(kind="cube", n=24, side=14), sch, 100.0, tol=1e-8,
                           max_iters=5000, e0=[[1, 0], [0, 0], [0, 0]]))
    for c in three_gen:
        c["force_oracle"] = True
    g["general"] = gen + three_gen

    # the largest fused lengths (4096) and beyond (8192: the general path)
    big = [C("big_rect4096x64_em_sub", dict(kind="rect", ny=64, nx=4096, my=32, mx=2048), "em_sub", 10.0,
             tol=1e-8, max_iters=2000),
           C("big_rect64x4096_basic", dict(kind="rect", ny=4096, nx=64, my=2048, mx=32), "basic", 10.0 + 1.0j,
             tol=1e-8, max_iters=2000),
           C("big_sq4096_em_sub_3it", sq(4096), "em_sub", 10.0, tol=1e-300, max_iters=3),
           C("big_sq4096_em_3it", sq(4096), "em", 1000.0, tol=1e-300, max_iters=3),
           C("big_rect8x8192_basic_sub", dict(kind="rect", ny=8, nx=8192, my=4, mx=4096), "basic_sub", 10.0,
             tol=1e-8, max_iters=2000)]
    g["big"] = big
    return g


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("groups", nargs="+")
    ap.add_argument("--jobs", type=int, default=max(1, (os.cpu_count() or 2) - 1))
    ap.add_argument("--only", default=None, help="substring filter on case names")
    a = ap.parse_args()
    allg = groups()
    for grp in a.groups:
        cases = [c for c in allg[grp] if a.only is None or a.only in c["name"]]
        out_path = os.path.join(GOLDEN, f"{grp}.json")
        existing = {}
        if os.path.exists(out_path):
            with open(out_path) as f:
                existing = {r["case"]["name"]: r for r in json.load(f)}
        todo = [c for c in cases if c["name"] not in existing]
        print(f"[{grp}] {len(todo)} cases to run ({len(existing)} cached)", flush=True)
        with ProcessPoolExecutor(max_workers=a.jobs) as ex:
            for res in ex.map(run_case, todo):
                existing[res["case"]["name"]] = res
                print(f"  {res['case']['name']}: {res['status']} it={res['iterations']} "
                      f"s*={res['sigma_star']} ({res['cpu_seconds']:.1f}s)", flush=True)
                ordered = [existing[c["name"]] for c in allg[grp] if c["name"] in existing]
                with open(out_path + ".tmp", "w") as f:
                    json.dump(ordered, f, indent=0)
                os.replace(out_path + ".tmp", out_path)


if __name__ == "__main__":
    main()
