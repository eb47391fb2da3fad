"""Batched solves: a sigma1 sweep (BASELINE config 5) or any list of configs
on one phase map, optionally sharded over the ranks of a torch.distributed
process group.

Sharding is by independent solve (round robin over ranks) -- there is no
data-path collective; the per-point records (status, iterations, sigma*,
history, <E>, <J>) are gathered once at the end with all_gather_object.
This is the batched form of the reference's sequential drivers
(cli.cmd_compare, cli.py:352-408; analysis.misestimation_report,
analysis.py:166-201) and of config 5's "batched over sweep points across
8 GPUs".
"""

from __future__ import annotations

import ctypes as C
from typing import Callable, Sequence

import numpy as np

from . import native
from .cell import PhaseMap
from .exceptions import BackendError
from .solver import SolverConfig, SolveResult, _check_grid, _device_chi, _params, _problem, _result_from, _torch


def _rank_world(group):
    try:
        import torch.distributed as dist

        if dist.is_available() and dist.is_initialized():
            return dist.get_rank(group), dist.get_world_size(group)
    except Exception:
        pass
    return 0, 1


def shard(n: int, rank: int, world: int) -> list[int]:
    """Indices of the points owned by `rank` (round robin: balances the mix
    of fast converging and MaxIters points of a sweep)."""
    return list(range(rank, n, world))


def _solve_local_gpu(pmap: PhaseMap, cfgs: Sequence[SolverConfig]) -> list[SolveResult]:
    """All configs of this rank through one fftc_solve_batch call."""
    if not cfgs:
        return []
    pars = [_params(c, pmap.dim) for c in cfgs]  # host validation first
    torch = _torch()
    _check_grid(pmap)
    chi = _device_chi(pmap, torch)
    prob = _problem(pmap, chi)
    cap = max(int(c.max_iters) for c in cfgs)
    hist = np.empty((len(cfgs), cap, 3), dtype=np.float64)
    parr = (native.Params * len(cfgs))(*pars)
    res = (native.Result * len(cfgs))()
    rc = native.lib().fftc_solve_batch(C.byref(prob), parr, len(cfgs), hist.ctypes.data, cap, res,
                                       torch.cuda.current_stream().cuda_stream)
    if rc:
        raise BackendError(f"fftc_solve_batch failed ({rc}): {native.last_error()}")
    return [_result_from(res[i], hist[i], pmap.dim) for i in range(len(cfgs))]


def _record(r: SolveResult) -> dict:
    return dict(sigma_star=r.sigma_star, status=r.status, iterations=r.iterations,
                degenerate_flux=r.degenerate_flux, device_ms=r.device_ms,
                history=np.array([[h.sigma_star.real, h.sigma_star.imag, h.residual] for h in r.history]),
                mean_E=r.mean_E, mean_J=r.mean_J)


def solve_sweep(pmap: PhaseMap, cfgs: Sequence[SolverConfig], *, group=None,
                local_solver: Callable | None = None) -> list[dict]:
    """Solve every config; returns one record per config, in order, on every rank.

    `local_solver(pmap, cfgs) -> list[SolveResult]` defaults to the GPU batch
    path; tests substitute a CPU solver to exercise the sharding on gloo.
    """
    rank, world = _rank_world(group)
    mine = shard(len(cfgs), rank, world)
    solver = local_solver or _solve_local_gpu
    local = solver(pmap, [cfgs[i] for i in mine])
    recs = {i: _record(r) for i, r in zip(mine, local)}
    if world > 1:
        import torch.distributed as dist

        gathered = [None] * world
        dist.all_gather_object(gathered, recs, group=group)
        for part in gathered:
            recs.update(part)
    return [recs[i] for i in range(len(cfgs))]


def c5_points(count: int = 256, seed: int = 20260809, alpha: float = 0.25, beta: float = 4.0) -> list[complex]:
    """BASELINE config 5 sweep points: Re in [-50, 50] excluding [-beta, -alpha],
    Im in [0.01, 10], seeded uniform draws with rejection (same recipe as the
    golden generator oracle/gen_golden.py)."""
    rng = np.random.default_rng(seed)
    pts = []
    while len(pts) < count:
        re = rng.uniform(-50.0, 50.0)
        im = rng.uniform(0.01, 10.0)
        if -beta <= re <= -alpha:
            continue
        pts.append(complex(re, im))
    return pts
