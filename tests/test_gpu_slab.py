"""GPU: the slab-decomposed 3-D path (fftc_slab_* kernels + the slab driver)
at world size 1 against the 3-D golden fixtures, and against the monolithic
fftc_solve on a larger random medium."""

from __future__ import annotations

import numpy as np
import pytest

from golden_io import load_group
from parity import REL

pytestmark = pytest.mark.gpu
ALPHA, BETA = 0.25, 4.0


def _cfg(case):
    import paper_2001_08289_b200 as fb

    sk = fb.SchemeKind(case["scheme"])
    kw = dict(scheme=sk, sigma1=complex(*case["sigma1"]), tol=case["tol"], max_iters=case["max_iters"])
    if sk.substituted:
        kw["interval"] = fb.SpectralInterval(ALPHA, BETA)
    if case.get("e0") is not None:
        kw["e0"] = tuple(complex(*v) for v in case["e0"])
    return fb.SolverConfig(**kw)


@pytest.mark.parametrize("name", ["3d_cube16_basic", "3d_cube16_em", "3d_cube16_basic_sub", "3d_cube16_em_sub",
                                  "3d_random16_em_sub", "3d_embed_basic", "3d_cube32_em_sub"])
def test_slab_world1_matches_golden(name):
    from paper_2001_08289_b200.slab import solve_slab
    from test_gpu_parity import _chi

    g = load_group("3d")[name]
    r = solve_slab(_chi(g["case"]["geom"]), _cfg(g["case"]))
    assert r["status"].value == g["status"] and r["iterations"] == g["iterations"]
    gs = complex(*g["sigma_star"])
    assert abs(r["sigma_star"] - gs) <= REL * abs(gs)
    h = g["history"]
    dev = np.array([s for s, _ in r["history"]])
    assert np.max(np.abs(dev - (h[:, 1] + 1j * h[:, 2])) / np.abs(h[:, 1] + 1j * h[:, 2])) <= REL


def test_slab_world1_matches_monolithic_64():
    import paper_2001_08289_b200 as fb
    from paper_2001_08289_b200.slab import solve_slab

    pm = fb.build_random_medium(64, 3, seed=20260809, smoothing=4.0, fraction=0.3)
    for scheme in ("basic", "em_sub"):
        sk = fb.SchemeKind(scheme)
        cfg = fb.SolverConfig(scheme=sk, sigma1=50.0, tol=1e-8, max_iters=2000, e0=(1 / 3 ** 0.5,) * 3,
                              interval=fb.SpectralInterval(ALPHA, BETA) if sk.substituted else None)
        a = fb.solve(pm, cfg)
        b = solve_slab(pm.chi, cfg)
        assert a.iterations == b["iterations"]
        assert abs(a.sigma_star - b["sigma_star"]) <= 1e-12 * abs(a.sigma_star)


class _Shared:
    def __init__(self, world):
        import threading

        self.barrier = threading.Barrier(world)
        self.buf = [None] * world


class ThreadComm:
    """torch.distributed stand-in for `world` host threads sharing ONE GPU:
    each simulated rank runs the real slab driver and GPU kernels on its own
    stream; the collectives are host-synchronised torch ops (every kernel has
    finished before an exchange starts, so no kernel waits on another rank).
    Sums run in rank order, as a deterministic all-reduce."""

    def __init__(self, shared, rank, world):
        self.s, self.rank, self.world = shared, rank, world

    @staticmethod
    def _sync():
        import torch

        torch.cuda.current_stream().synchronize()

    def all_reduce(self, t, group=None):
        self._sync()
        self.s.buf[self.rank] = t.clone()
        self.s.barrier.wait()
        tot = self.s.buf[0].clone()
        for q in range(1, self.world):
            tot += self.s.buf[q]
        self._sync()
        self.s.barrier.wait()
        t.copy_(tot)
        self._sync()

    def barrier(self):
        self._sync()
        self.s.barrier.wait()

    def all_gather_object(self, obj):
        self.s.buf[self.rank] = obj
        self.s.barrier.wait()
        out = list(self.s.buf)
        self.s.barrier.wait()
        return out

    def all_to_all_single(self, out, inp, group=None):
        import torch

        self._sync()
        self.s.buf[self.rank] = inp
        self.s.barrier.wait()
        out.copy_(torch.cat([self.s.buf[q].chunk(self.world, 0)[self.rank] for q in range(self.world)], 0))
        self._sync()
        self.s.barrier.wait()


def _run_threads(chi, cfg, world, fused=True):
    import threading

    import torch

    from paper_2001_08289_b200.slab import solve_slab

    shared, out, errs = _Shared(world), [None] * world, []

    def rank_main(r):
        try:
            torch.cuda.set_device(0)
            with torch.cuda.stream(torch.cuda.Stream()):
                out[r] = solve_slab(chi, cfg, comm=ThreadComm(shared, r, world), fused=fused)
        except BaseException as e:  # noqa: BLE001 -- reported below
            errs.append(e)
            shared.barrier.abort()

    th = [threading.Thread(target=rank_main, args=(r,)) for r in range(world)]
    for t in th:
        t.start()
    for t in th:
        t.join(timeout=600)
    assert not errs, errs
    return out


@pytest.mark.parametrize("fused", [False, True], ids=["alltoall", "fused"])
@pytest.mark.parametrize("shape, scheme, world", [((256, 256, 8), "em_sub", 2), ((256, 256, 8), "basic", 4),
                                                  ((512, 256, 8), "em", 2), ((64, 64, 64), "basic_sub", 4),
                                                  ((256, 1024, 8), "em", 2)])
def test_slab_threads_match_monolithic(shape, scheme, world, fused):
    """z-slab decomposition at world 2 / 4 on the GPU kernels (rank-local
    slabs with y0/z0 offsets, TMA tile column passes where the line lengths
    allow) against the single-GPU solve: identical iteration counts and
    histories to roundoff, identical records on every rank."""
    import paper_2001_08289_b200 as fb

    rng = np.random.default_rng(11)
    chi = rng.random(shape) < 0.3
    sk = fb.SchemeKind(scheme)
    cfg = fb.SolverConfig(scheme=sk, sigma1=20.0 + 1j, tol=1e-9, max_iters=300, e0=(0.0, 0.6, 0.8),
                          interval=fb.SpectralInterval(ALPHA, BETA) if sk.substituted else None)
    mono = fb.solve(fb.PhaseMap(chi), cfg)
    recs = _run_threads(chi, cfg, world, fused)
    # fused transposes need the TMA tile passes: y and z lines of 256..1024 and
    # nx a multiple of their tile widths; the 64^3 case keeps the all-to-alls
    # (y lines of 1024 run single-component tiles of four columns, z lines of 1024 vector tiles of two)
    def tile_ok(n, y_lines):
        return 256 <= n <= 1024 and shape[2] % (8 if n <= 256 else 4 if n <= 512 else (4 if y_lines else 2)) == 0

    assert all(r["fused"] == (fused and tile_ok(shape[0], False) and tile_ok(shape[1], True)) for r in recs)
    for r in recs:
        assert r["world"] == world and r["iterations"] == mono.iterations
        assert r["status"] == mono.status
        dev = np.array([s for s, _ in r["history"]])
        ref = np.array([h.sigma_star for h in mono.history])
        assert np.max(np.abs(dev - ref) / np.abs(ref)) <= 1e-12
    assert all(r["history"] == recs[0]["history"] for r in recs)
