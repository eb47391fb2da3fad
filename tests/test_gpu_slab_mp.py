"""GPU, two processes: the z-slab decomposed 3-D solve with the fused
transposes, ranks in separate processes sharing their slab buffers through
CUDA IPC (fftc_ipc_*), host collectives over gloo.  Both processes use the
one GPU this pool provides; no kernel waits on another rank -- the phases are
ordered by the host-level barrier and all-reduce -- so this exercises the
real multi-process plumbing (handle exchange, peer mapping, kernels writing
into another process's buffers) that NVLink peers use between GPUs."""

from __future__ import annotations

import os
import socket

import numpy as np
import pytest

pytestmark = pytest.mark.gpu
ALPHA, BETA = 0.25, 4.0


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _case(shape, scheme):
    import paper_2001_08289_b200 as fb

    rng = np.random.default_rng(5)
    chi = rng.random(shape) < 0.3
    sk = fb.SchemeKind(scheme)
    cfg = fb.SolverConfig(scheme=sk, sigma1=20.0 + 1j, tol=1e-9, max_iters=300, e0=(0.0, 0.6, 0.8),
                          interval=fb.SpectralInterval(ALPHA, BETA) if sk.substituted else None)
    return chi, cfg


def _worker(rank, world, port, shape, scheme, q):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    import torch
    import torch.distributed as dist

    torch.cuda.set_device(0)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        from paper_2001_08289_b200.slab import solve_slab

        chi, cfg = _case(shape, scheme)
        r = solve_slab(chi, cfg, fused=True)
        q.put((rank, r["fused"], r["iterations"], r["status"].value, [s for s, _ in r["history"]]))
    except BaseException as e:  # noqa: BLE001 -- reported to the parent
        q.put((rank, "error", repr(e), None, None))
    finally:
        dist.destroy_process_group()


@pytest.mark.parametrize("shape, scheme", [((256, 256, 8), "em_sub"), ((512, 256, 8), "basic")])
def test_two_process_fused_slab_matches_monolithic(shape, scheme):
    import torch.multiprocessing as mp

    import paper_2001_08289_b200 as fb

    chi, cfg = _case(shape, scheme)
    mono = fb.solve(fb.PhaseMap(chi), cfg)
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, 2, port, shape, scheme, q)) for r in range(2)]
    for p in procs:
        p.start()
    got = dict((m[0], m[1:]) for m in (q.get(timeout=600) for _ in procs))
    for p in procs:
        p.join(timeout=120)
    for r in (0, 1):
        fused, iters, status, hist = got[r]
        assert fused is True, got[r]
        assert iters == mono.iterations and status == mono.status.value
        ref = np.array([h.sigma_star for h in mono.history])
        assert np.max(np.abs(np.array(hist) - ref) / np.abs(ref)) <= 1e-12
    assert got[0][3] == got[1][3]
