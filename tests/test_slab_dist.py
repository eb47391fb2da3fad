"""CPU: the z-slab decomposed 3-D driver (paper_2001_08289_b200/slab.py) with
world_size 1 and 2 over gloo -- transposes, all-reduced partials, delta pin
and monitor -- reproduces the single-process oracle solve.  Per-rank compute
is the numpy backend (tests/slab_numpy.py, test infrastructure)."""

from __future__ import annotations

import os
import socket

import numpy as np
import pytest
import torch.distributed as dist
import torch.multiprocessing as mp

ALPHA, BETA = 0.25, 4.0
CASES = [("basic", 10.0), ("em", 10.0), ("basic_sub", 5.0), ("em_sub", 10.0)]


def _chi():
    rng = np.random.default_rng(7)
    return rng.random((8, 8, 4)) < 0.3


def _cfg(scheme, s1):
    import paper_2001_08289_b200 as fb

    sk = fb.SchemeKind(scheme)
    return fb.SolverConfig(scheme=sk, sigma1=s1, tol=1e-10, max_iters=400, e0=(1.0, 0.5, 0.25),
                           interval=fb.SpectralInterval(ALPHA, BETA) if sk.substituted else None)


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _worker(rank, world, port, q):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        from paper_2001_08289_b200.slab import solve_slab
        from slab_numpy import NumpySlab

        out = {}
        for scheme, s1 in CASES:
            r = solve_slab(_chi(), _cfg(scheme, s1), backend_factory=NumpySlab)
            out[scheme] = (r["iterations"], r["sigma_star"], r["status"].value, [h[1] for h in r["history"]])
        q.put((rank, out))
    finally:
        dist.destroy_process_group()


def _oracle(scheme, s1):
    from oracle import fftcond_oracle as O

    return O.solve(_chi(), scheme, s1, tol=1e-10, max_iters=400, alpha=ALPHA, beta=BETA, e0=(1.0, 0.5, 0.25))


@pytest.mark.parametrize("scheme,s1", CASES)
def test_slab_world1_matches_oracle(scheme, s1):
    from paper_2001_08289_b200.slab import solve_slab
    from slab_numpy import NumpySlab

    r = solve_slab(_chi(), _cfg(scheme, s1), backend_factory=NumpySlab)
    o = _oracle(scheme, s1)
    assert r["iterations"] == o.iterations and r["status"].value == o.status
    assert abs(r["sigma_star"] - o.sigma_star) <= 1e-12 * abs(o.sigma_star)


def test_slab_world2_gloo_matches_oracle():
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, 2, port, q)) for r in range(2)]
    for p in procs:
        p.start()
    got = dict(q.get(timeout=300) for _ in procs)
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    for scheme, s1 in CASES:
        o = _oracle(scheme, s1)
        for rank in (0, 1):
            it, s, st, res = got[rank][scheme]
            assert it == o.iterations and st == o.status, (scheme, rank, it, o.iterations)
            assert abs(s - o.sigma_star) <= 1e-12 * abs(o.sigma_star), (scheme, s, o.sigma_star)
            ores = [h[2] for h in o.history]
            assert np.allclose(res, ores, rtol=1e-8, atol=1e-14)
        assert got[0][scheme][1] == got[1][scheme][1]  # every rank reports the same sigma*
