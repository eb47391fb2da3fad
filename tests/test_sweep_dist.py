"""CPU, world_size 2 over gloo: the sweep driver shards independent solves
round robin and gathers every record on every rank, in order, identical to a
single-process run.  The per-rank solver is the CPU oracle (test
infrastructure) standing in for the GPU batch call."""

from __future__ import annotations

import os
import socket

import numpy as np
import pytest
import torch.distributed as dist
import torch.multiprocessing as mp

ALPHA, BETA = 0.25, 4.0


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _oracle_solver(pmap, cfgs):
    import paper_2001_08289_b200 as fb
    from oracle import fftcond_oracle as O

    out = []
    for c in cfgs:
        r = O.solve(pmap.chi, c.scheme.value, complex(c.sigma1), tol=c.tol, max_iters=c.max_iters,
                    alpha=ALPHA, beta=BETA)
        h = fb.ConvergenceHistory()
        for k, s, res in r.history:
            h.append(k, s, res)
        out.append(fb.SolveResult(sigma_star=r.sigma_star, E_field=None, J_field=None, history=h,
                                  status=fb.TerminationStatus(r.status), degenerate_flux=r.degenerate_flux,
                                  mean_E=O.component_means(r.E), mean_J=O.component_means(r.J), device_ms=0.0))
    return out


def _cfgs():
    import paper_2001_08289_b200 as fb
    from paper_2001_08289_b200.sweep import c5_points

    pts = c5_points(6)
    return [fb.SolverConfig(scheme=fb.SchemeKind.EYRE_MILTON_SUB, sigma1=s, tol=1e-8, max_iters=60,
                            interval=fb.SpectralInterval(ALPHA, BETA)) for s in pts]


def _worker(rank, world, port, q):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        import paper_2001_08289_b200 as fb
        from paper_2001_08289_b200.sweep import solve_sweep

        recs = solve_sweep(fb.build_square_array(16, 0.5), _cfgs(), local_solver=_oracle_solver)
        q.put((rank, [(r["sigma_star"], r["iterations"], r["status"].value) for r in recs]))
    finally:
        dist.destroy_process_group()


def test_shard_is_a_partition():
    from paper_2001_08289_b200.sweep import shard

    for n in (0, 1, 5, 256):
        for w in (1, 2, 3, 8):
            parts = [shard(n, r, w) for r in range(w)]
            flat = sorted(i for p in parts for i in p)
            assert flat == list(range(n))


def test_c5_points_recipe():
    from paper_2001_08289_b200.sweep import c5_points

    pts = c5_points()
    assert len(pts) == 256
    assert all(-50 <= p.real <= 50 and not (-4 <= p.real <= -0.25) and 0.01 <= p.imag <= 10 for p in pts)
    from golden_io import load_group

    g = load_group("c5small")
    first = g["c5s_64_p000"]["case"]["sigma1"]
    assert complex(*first) == pts[0]


def test_sweep_world2_gloo_matches_single_process():
    import paper_2001_08289_b200 as fb
    from paper_2001_08289_b200.sweep import solve_sweep

    ref = solve_sweep(fb.build_square_array(16, 0.5), _cfgs(), local_solver=_oracle_solver)
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, 2, port, q)) for r in range(2)]
    for p in procs:
        p.start()
    got = dict(q.get(timeout=240) for _ in procs)
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    want = [(r["sigma_star"], r["iterations"], r["status"].value) for r in ref]
    assert got[0] == want and got[1] == want
