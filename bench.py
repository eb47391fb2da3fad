#!/usr/bin/env python
"""Benchmark: fp64 voxel-iterations/s of the FFT field iteration.

Default workload = BASELINE.json configs[1] (the config the metric is quoted
on that fits one GPU): 2048x2048 periodic cell with a centred square
inclusion (25% phase 1), sigma2 = 1, E0 = (1, 0), stop at residual 1e-10,
both the Eyre-Milton scheme (em) and the paper's accelerated substituted
scheme (em_sub, (alpha, beta) = (0.25, 4.0) from the reference's
configs/compare.cfg:14-15), sigma1 in {0.1, 10, 1000}.  One STEP = all six
solves run to convergence.  Synthetic input (the geometry is the
reference's own builder; no dataset exists).

value   = sum over solves of N * iterations / device time of the step, with
          the phase map already resident in HBM (CUDA events on the stream
          the library launches on).
e2e     = the same metric through the public API (fb.solve) with a HOST phase
          map: host->device copy of chi and device->host copy of the history
          inside the timed region.
--impl reference: the CPU oracle port (oracle/fftcond_oracle.py, a bit-exact
          numpy restatement of the reference loops) on the host cores.

Multi-GPU: configs[1] does not shard (replicas only): every rank runs the
full step on its own GPU, value = sum over ranks / max time over ranks.
"""

from __future__ import annotations

import argparse
import json
import math
import os
import subprocess
import sys
import time

REPO = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, REPO)

N_GRID = 2048
SIDE = 0.5
TOL = 1e-10
MAX_ITERS = 20000
ALPHA, BETA = 0.25, 4.0
SOLVES = [("em", 0.1), ("em", 10.0), ("em", 1000.0), ("em_sub", 0.1), ("em_sub", 10.0), ("em_sub", 1000.0)]
WORKLOADS = {
    "c2": SOLVES,
    "c1": [("basic", 10.0)],  # BASELINE configs[0]: 256^2, basic, tol 1e-8 (set_workload)
    "c2-emsub10": [("em_sub", 10.0)],
    "c2-fast": [("em", 0.1), ("em", 10.0), ("em_sub", 0.1), ("em_sub", 10.0)],
    "c5": None,  # BASELINE configs[4]: 256-point complex sigma1 sweep, em_sub, 1024^2 (see run_c5)
    "c3": None,  # BASELINE configs[2]: 512^3 centred cube, em_sub, sigma1=100 (see run_3d)
    "c4": None,  # BASELINE configs[3]: 1024^3 random medium, basic, sigma1=50; z-slabs over N GPUs (run_3d)
}


def _ncu_traffic(kernel, it_by_scheme, n):
    """DRAM bytes (read + write) per launch of `kernel` from the committed ncu
    capture (profiles/r1_ncu_traffic.json), weighted like the algorithmic
    bytes; None when the capture does not cover this kernel/grid/schemes."""
    path = os.path.join(os.path.dirname(os.path.abspath(__file__)), "profiles", "r1_ncu_traffic.json")
    try:
        with open(path) as fh:
            t = json.load(fh)
    except OSError:
        return None, None
    per = t.get("kernels", {}).get(kernel, {})
    if t.get("grid") != [n, n] or not all(s in per for s in it_by_scheme):
        return None, None
    tot = sum(it_by_scheme.values())
    bytes_ = sum((per[s]["dram_read"] + per[s]["dram_write"]) * k for s, k in it_by_scheme.items()) / tot
    return bytes_, t.get("source")


def _ncu_pipes(kernel, it_by_scheme):
    """FP64-pipe and issue-slot utilisation of `kernel` in the committed ncu
    capture (launch-weighted over schemes), or None."""
    path = os.path.join(os.path.dirname(os.path.abspath(__file__)), "profiles", "r1_ncu_traffic.json")
    try:
        with open(path) as fh:
            per = json.load(fh).get("kernels", {}).get(kernel, {})
    except OSError:
        return None
    if not all(s in per and "fp64_pipe" in per[s] for s in it_by_scheme):
        return None
    tot = sum(it_by_scheme.values())
    return {k: sum(per[s][k] * n for s, n in it_by_scheme.items()) / tot for k in ("fp64_pipe", "issue_active")}


def _fft_passes(kernel, it_by_scheme):
    """Length-n transforms per voxel and component done by one launch of a 2-D
    sweep, launch-weighted over schemes."""
    em_type = {"em": 1, "em_sub": 1}
    per = {"sweep1_rows_fwd": lambda s: 2 if s in em_type else 1,
           "sweep2_cols_gamma": lambda s: 3 if s in em_type else 2,
           "sweep3_rows_inv": lambda s: 1}.get(kernel)
    if per is None:
        return None
    tot = sum(it_by_scheme.values())
    return sum(per(s) * n for s, n in it_by_scheme.items()) / tot


def _peaks():
    path = os.path.join(REPO, "MEASURED_PEAKS.json")
    try:
        with open(path) as f:
            p = json.load(f)
        return float(p["hbm_gbs"]), "measured (MEASURED_PEAKS.json hbm_gbs)"
    except Exception:
        return 6650.0, "fallback (B200_PROFILING.md, MEASURED_PEAKS.json absent)"


def _bytes_per_voxel(scheme: str, d: int, f: float) -> dict:
    """Algorithmic HBM bytes per voxel per launch of each sweep (2-D schedule).

    V = 16 d (one complex128 d-vector); chi is 1 byte; S/T slots only move
    on phase-1 voxels (fraction f).  See DESIGN.md section 3.
    """
    V = 16.0 * d
    if scheme == "basic":
        k = {"sweep1_rows_fwd": 2 * V + 1, "sweep2_cols_gamma": 2 * V, "sweep3_rows_inv": 3 * V + 1}
    elif scheme == "em":
        k = {"sweep1_rows_fwd": 3 * V + 1, "sweep2_cols_gamma": 3 * V, "sweep3_rows_inv": 2 * V + 1}
    elif scheme == "basic_sub":
        k = {"sweep1_rows_fwd": 2 * V + f * V + 1, "sweep2_cols_gamma": 2 * V,
             "sweep3_rows_inv": 3 * V + 2 * f * V + 1}
    else:
        k = {"sweep1_rows_fwd": 3 * V + 2 * f * V + 1, "sweep2_cols_gamma": 3 * V,
             "sweep3_rows_inv": 2 * V + 5 * f * V + 1}
    return k


def _survey_bytes(scheme: str, d: int, f: float) -> float:
    """SURVEY.md 8(d) per-voxel-iteration figure for the fused 2-D schedule."""
    V = 16.0 * d
    return {"basic": 7 * V + 2, "em": 9 * V + 2, "basic_sub": 7 * V + 2 * f * V + 2,
            "em_sub": 9 * V + 6 * f * V + 2}[scheme]


class ClockSampler:
    """nvidia-smi clocks / throttle reasons sampled during the timed region."""

    Q = ("index,clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.active,"
         "clocks_event_reasons.hw_slowdown,clocks_event_reasons.hw_thermal_slowdown,"
         "clocks_event_reasons.sw_thermal_slowdown,clocks_event_reasons.sw_power_cap")

    def __init__(self, index: int):
        self.index = index
        self.proc = None
        self.path = os.path.join("/tmp", f"fftc_clocks_{os.getpid()}.csv")

    def start(self):
        try:
            self.proc = subprocess.Popen(
                ["nvidia-smi", f"--id={self.index}", f"--query-gpu={self.Q}", "--format=csv,noheader,nounits",
                 "-lms", "100"], stdout=open(self.path, "w"), stderr=subprocess.DEVNULL)
        except Exception:
            self.proc = None

    def stop(self) -> dict:
        if self.proc is None:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["nvidia-smi unavailable"]}
        self.proc.terminate()
        try:
            self.proc.wait(timeout=5)
        except Exception:
            self.proc.kill()
        sms, maxs, reasons = [], [], set()
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        try:
            for line in open(self.path):
                parts = [p.strip() for p in line.split(",")]
                if len(parts) < 9:
                    continue
                try:
                    sms.append(float(parts[1]))
                    maxs.append(float(parts[2]))
                except ValueError:
                    continue
                for nm, v in zip(names, parts[5:9]):
                    if v.lower() == "active":
                        reasons.add(nm)
        except OSError:
            pass
        sms.sort()
        return {"sm_mhz": sms[len(sms) // 2] if sms else None, "sm_max_mhz": max(maxs) if maxs else None,
                "reasons": sorted(reasons), "samples": len(sms)}


def _dist():
    ws = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    return ws, rank, local


# ---------------------------------------------------------------------------
# CPU legs (oracle port -- test infrastructure, never the product)
# ---------------------------------------------------------------------------

def _oracle_sample(args):
    scheme, s1, n, iters = args[:4]
    geom = args[4] if len(args) > 4 else "square"
    import numpy as np
    from oracle import fftcond_oracle as O

    e0 = None
    if geom == "square":
        chi = O.centred_box(n, int(round(SIDE * n)))
    elif geom == "cube":  # C3 recipe at a bounded size
        chi = O.centred_box(n, 2 * int(round(0.63 * n / 2)), 3)
        e0 = (1.0, 0.0, 0.0)
    else:  # C4 recipe (random medium) at a bounded size
        rng = np.random.default_rng(20260809)
        u = rng.random((n,) * 3)
        k = np.fft.fftfreq(n)
        k2 = k[:, None, None] ** 2 + k[None, :, None] ** 2 + k[None, None, :] ** 2
        sm = np.fft.ifftn(np.fft.fftn(u) * np.exp(-2.0 * np.pi ** 2 * 16.0 * k2)).real
        chi = sm <= np.quantile(sm, 0.30)
        e0 = (3 ** -0.5,) * 3
    t0 = time.perf_counter()
    r = O.solve(chi, scheme, s1, e0=e0, tol=1e-300, max_iters=iters, alpha=ALPHA, beta=BETA)
    dt = time.perf_counter() - t0
    return int(chi.size) * r.iterations, dt


def cpu_baseline(iters: int = 6, sample=(("em", 10.0), ("em_sub", 10.0))) -> dict:
    """Single-core oracle port on a bounded sample of the workload."""
    tot_v, tot_t = 0, 0.0
    for scheme, s1 in sample:
        v, t = _oracle_sample((scheme, s1, N_GRID, iters))
        tot_v += v
        tot_t += t
    return {"value": tot_v / tot_t, "unit": "voxel-iterations/s", "cores": 1, "kind": "port",
            "sample": f"{len(sample)} solves (" + ", ".join(f"{sch} at sigma1={v:g}" for sch, v in dict.fromkeys(sample))
                      + f") on {N_GRID}^2, {iters} iterations each "
                      f"(tol=1e-300 so every iteration runs), oracle/fftcond_oracle.py (numpy pocketfft, "
                      f"bit-identical to the reference loops), {tot_t:.1f} s of CPU work"}


def run_reference(a):
    ws, rank, _ = _dist()
    if rank != 0:
        return 0
    from concurrent.futures import ProcessPoolExecutor

    ncpu = os.cpu_count() or 1
    # every host core gets a bounded sample of one of the workload's solves
    # (cycling through them); the reference is single threaded, so this is
    # the throughput the host can deliver
    procs = max(1, ncpu)
    iters = a.ref_iters
    if a.workload == "c3":  # bounded 3-D samples: the reference itself is 2-D only (restatement, 128^3)
        solves, tasks = [("em_sub", 100.0)], [("em_sub", 100.0, 128, iters, "cube")]
    elif a.workload == "c4":
        solves, tasks = [("basic", 50.0)], [("basic", 50.0, 128, iters, "random")]
    elif a.workload == "c5":
        from paper_2001_08289_b200.sweep import c5_points

        pts = c5_points(max(procs, 8))
        solves, tasks = [("em_sub", p) for p in pts], [("em_sub", p, 1024, iters) for p in pts]
    else:
        solves = WORKLOADS[a.workload]
        tasks = [(sch, v, N_GRID, iters) for sch, v in solves]
    jobs = [tasks[i % len(tasks)] for i in range(max(procs, len(tasks)))]
    times, vox = [], 0
    with ProcessPoolExecutor(max_workers=procs) as ex:
        for step in range(a.warmup + a.steps):
            t0 = time.perf_counter()
            res = list(ex.map(_oracle_sample, jobs))
            dt = time.perf_counter() - t0
            if step >= a.warmup:
                times.append(dt)
                vox = sum(v for v, _ in res)
    ms = 1e3 * sum(times) / len(times)
    value = vox / (ms / 1e3)
    line = {
        "impl": "reference", "metric": "fp64 voxel-iterations/sec of the FFT iteration",
        "value": value, "unit": "voxel-iterations/s", "n_gpus": ws, "steps": a.steps, "warmup": a.warmup,
        "ms_per_step": ms, "higher_is_better": True, "scaling": "weak", "vs_baseline": None,
        "dtype": "f64 (complex128)", "data": "synthetic (reference square-array builder)",
        "config": _config(a) if WORKLOADS[a.workload] else {"workload": a.workload, "sample_grid": jobs[0][2],
                                                            "note": "bounded samples of the workload's solves"},
        "cpu_baseline": {"value": value, "unit": "voxel-iterations/s", "cores": procs, "kind": "port",
                         "sample": f"{len(jobs)} bounded samples ({iters} iterations each) cycling through the "
                                   f"{len(solves)} solves, {procs} processes on {ncpu} host CPUs; oracle/fftcond_oracle.py "
                                   f"is the bit-exact numpy restatement of the reference loops"},
        "e2e": {"value": value, "unit": "voxel-iterations/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
    }
    print(json.dumps(line), flush=True)
    return 0


def set_workload(name):
    """c1 (BASELINE configs[0]) runs the c2 machinery on its own grid and tolerance."""
    global N_GRID, TOL, MAX_ITERS
    if name == "c1":
        N_GRID, TOL, MAX_ITERS = 256, 1e-8, 1000


def _config(a):
    solves = WORKLOADS[a.workload]
    if a.workload == "c1":
        return {"workload": f"BASELINE configs[0]: {N_GRID}x{N_GRID} square array f=0.25, basic@sigma1=10, "
                            f"sigma0=(sigma1+1)/2, tol={TOL:g}",
                "grid": [N_GRID, N_GRID], "schemes": ["basic"], "sigma1": [10.0], "tol": TOL,
                "max_iters": MAX_ITERS,
                "l2": "working set (~8 MB) is L2-resident by nature; L2 flushed (256 MB write) before every "
                      "timed step, outside that step's CUDA events",
                "parallelism": "replicas" if _dist()[0] > 1 else "single GPU"}
    return {"workload": f"BASELINE configs[1]: {N_GRID}x{N_GRID} square array f=0.25, "
                        + ", ".join(f"{s}@sigma1={v:g}" for s, v in solves) + f", tol={TOL:g}",
            "grid": [N_GRID, N_GRID], "schemes": [s for s, _ in solves], "sigma1": [v for _, v in solves],
            "alpha_beta": [ALPHA, BETA], "tol": TOL, "max_iters": MAX_ITERS,
            "l2": "inputs larger than L2 (state + work fields 384-640 MB per solve >> 126 MB L2)",
            "parallelism": "replicas" if _dist()[0] > 1 else "single GPU"}


# ---------------------------------------------------------------------------
# GPU arm
# ---------------------------------------------------------------------------

def run_ours(a):
    import numpy as np
    import torch

    ws, rank, local = _dist()
    torch.cuda.set_device(local)
    if ws > 1:
        import torch.distributed as dist

        dist.init_process_group("nccl", device_id=torch.device("cuda", local))
    import paper_2001_08289_b200 as fb
    from paper_2001_08289_b200 import native
    from paper_2001_08289_b200.solver import _solve_aug, _solve_h

    solves = WORKLOADS[a.workload]
    chi_host = np.zeros((N_GRID, N_GRID), dtype=bool)
    m = int(round(SIDE * N_GRID))
    lo = (N_GRID - m) // 2
    chi_host[lo:lo + m, lo:lo + m] = True
    frac = float(chi_host.mean())
    cfgs = []
    for sch, s1 in solves:
        sk = fb.SchemeKind(sch)
        cfgs.append(fb.SolverConfig(scheme=sk, sigma1=s1, tol=TOL, max_iters=MAX_ITERS,
                                    interval=fb.SpectralInterval(ALPHA, BETA) if sk.substituted else None))
    pm_dev = fb.PhaseMap(chi_host)
    stream = torch.cuda.current_stream()

    def step_device():
        # chi resident in HBM (cached on pm_dev); fields not materialised
        its = []
        for cfg in cfgs:
            if cfg.scheme.substituted:
                r = _solve_aug(pm_dev, cfg, cfg.scheme.accelerated, want_fields=False)
            else:
                r = _solve_h(pm_dev, cfg, cfg.scheme.accelerated, want_fields=False)
            its.append(r)
        return its

    def step_e2e():
        pm = fb.PhaseMap(chi_host)  # fresh map: chi crosses host->device inside the step
        return [fb.solve(pm, cfg) for cfg in cfgs]

    def barrier():
        if ws > 1:
            import torch.distributed as dist

            dist.barrier()
        torch.cuda.synchronize()

    for _ in range(a.warmup):
        step_device()
    # ---- timed: device-resident (graph-mode loop, no profiling) ----
    barrier()
    clocks = ClockSampler(local)
    clocks.start()
    launches0 = native.lib().fftc_launch_count()
    results = None
    if a.workload == "c1":
        # L2-resident workload: flush L2 before every step, time each step alone
        flush = torch.empty(256 << 20, dtype=torch.uint8, device="cuda")
        pairs = []
        for _ in range(a.steps):
            flush.fill_(1)
            e0 = torch.cuda.Event(enable_timing=True)
            e1 = torch.cuda.Event(enable_timing=True)
            e0.record(stream)
            results = step_device()
            e1.record(stream)
            pairs.append((e0, e1))
    else:
        e0 = torch.cuda.Event(enable_timing=True)
        e1 = torch.cuda.Event(enable_timing=True)
        e0.record(stream)
        for _ in range(a.steps):
            results = step_device()
        e1.record(stream)
        pairs = [(e0, e1)]
    barrier()
    launches = native.lib().fftc_launch_count() - launches0
    clk = clocks.stop()
    ms_total = sum(b.elapsed_time(c) for b, c in pairs)
    ms = ms_total / a.steps
    vox = sum(N_GRID * N_GRID * r.iterations for r in results)
    # ---- one profiled step: per-kernel CUDA-event durations for the roofline ----
    native.profile(True)
    p0 = torch.cuda.Event(enable_timing=True)
    p1 = torch.cuda.Event(enable_timing=True)
    p0.record(stream)
    step_device()
    p1.record(stream)
    torch.cuda.synchronize()
    prof_ms = p0.elapsed_time(p1)
    kstats = native.kernel_stats()
    native.profile(False)
    # ---- timed: end to end through the public API, host inputs ----
    step_e2e()  # warm the allocator paths of the public API
    barrier()
    clocks_e2e = ClockSampler(local)  # the e2e steps run last, often at lower power-capped clocks
    clocks_e2e.start()
    f0 = torch.cuda.Event(enable_timing=True)
    f1 = torch.cuda.Event(enable_timing=True)
    t_wall = time.perf_counter()
    f0.record(stream)
    e2e_res = None
    for _ in range(a.steps):
        e2e_res = step_e2e()
        _ = [r.sigma_star for r in e2e_res]
    f1.record(stream)
    barrier()
    t_wall = time.perf_counter() - t_wall
    clk_e2e = clocks_e2e.stop()
    ms_e2e = max(f0.elapsed_time(f1), 1e3 * t_wall) / a.steps
    e2e_iters = sum(r.iterations for r in e2e_res)
    # max over ranks
    if ws > 1:
        import torch.distributed as dist

        t = torch.tensor([ms, ms_e2e], device="cuda", dtype=torch.float64)
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        ms, ms_e2e = float(t[0]), float(t[1])
    value = ws * vox / (ms / 1e3)
    e2e_value = ws * N_GRID * N_GRID * e2e_iters / (ms_e2e / 1e3)

    # ---- roofline of the dominant kernel (from the per-launch events) ----
    hbm, peak_src = _peaks()
    N = N_GRID * N_GRID
    dom = max(kstats.items(), key=lambda kv: kv[1][1]) if kstats else None
    # algorithmic bytes: weight each scheme's per-kernel bytes by its share of launches
    it_by_scheme = {}
    for (sch, _), r in zip(solves, results):
        it_by_scheme[sch] = it_by_scheme.get(sch, 0) + r.iterations
    tot_it = sum(it_by_scheme.values())
    roof = None
    if dom is not None:
        name, (nl, tms) = dom
        bpv = sum(_bytes_per_voxel(s, 2, frac)[name] * n for s, n in it_by_scheme.items()) / tot_it
        per_launch_ms = tms / nl
        achieved = bpv * N / (per_launch_ms / 1e3) / 1e9
        traffic, traffic_src = _ncu_traffic(name, it_by_scheme, N_GRID)
        roof = {"bound": "hbm", "kernel": name, "achieved": achieved, "peak": hbm, "unit": "GB/s",
                "frac": achieved / hbm, "traffic": traffic, "traffic_source": traffic_src, "peak_source": peak_src,
                "bytes_per_launch": bpv * N, "avg_launch_ms": per_launch_ms, "launches": nl,
                "share_of_step": tms / prof_ms if prof_ms > 0 else None,
                "timing": "CUDA events around every launch of one profiled step (one iteration per sync)",
                # the sweeps are bound by their transforms, not by HBM: FFT
                # points per second of the dominant kernel and its pipe utilisation in the ncu capture
                "fft_passes_per_voxel_component": _fft_passes(name, it_by_scheme),
                "fft_gpoints_per_s": (_fft_passes(name, it_by_scheme) or 0.0) * 2 * N / (per_launch_ms / 1e3) / 1e9,
                "ncu_pipes": _ncu_pipes(name, it_by_scheme)}
    survey_b = sum(_survey_bytes(s, 2, frac) * n for s, n in it_by_scheme.items()) / tot_it
    ours_b = sum(sum(_bytes_per_voxel(s, 2, frac).values()) * n for s, n in it_by_scheme.items()) / tot_it
    iter_roof = {"bytes_per_voxel_iter_survey": survey_b, "bytes_per_voxel_iter_schedule": ours_b,
                 "achieved_gbs_survey_bytes": value / ws * survey_b / 1e9,
                 "frac_survey_bytes": value / ws * survey_b / 1e9 / hbm,
                 "achieved_gbs_schedule_bytes": value / ws * ours_b / 1e9,
                 "frac_schedule_bytes": value / ws * ours_b / 1e9 / hbm}

    line = {
        "metric": "fp64 voxel-iterations/sec of the FFT iteration",
        "value": value, "unit": "voxel-iterations/s", "n_gpus": ws, "steps": a.steps, "warmup": a.warmup,
        "ms_per_step": ms, "higher_is_better": True, "scaling": "weak", "vs_baseline": None,
        "dtype": "f64 (complex128)", "data": "synthetic (reference square-array builder)",
        "config": _config(a),
        "roofline": roof, "iteration_roofline": iter_roof,
        "e2e": {"value": e2e_value, "unit": "voxel-iterations/s", "h2d_bytes_per_step": N,
                "d2h_bytes_per_step": 24 * e2e_iters + 256 * len(cfgs), "clocks": clk_e2e},
        "gpu_launches": int(launches), "clocks": clk,
        "kernels": {k: {"launches": v[0], "ms_total": v[1], "ms_per_launch": v[1] / max(v[0], 1)}
                    for k, v in kstats.items()},
        "solves": [{"scheme": s, "sigma1": v, "iterations": r.iterations, "status": r.status.value,
                    "sigma_star": [r.sigma_star.real, r.sigma_star.imag]} for (s, v), r in zip(solves, results)],
    }
    if ws == 1 and not a.no_cpu_baseline:
        line["cpu_baseline"] = (cpu_baseline(62, (("basic", 10.0),) * 30) if a.workload == "c1"
                                else cpu_baseline(a.cpu_iters))
    if rank == 0:
        print(json.dumps(line), flush=True)
    if ws > 1:
        import torch.distributed as dist

        dist.destroy_process_group()
    return 0


def run_c5(a):
    """BASELINE configs[4]: 256 complex sigma1 points on the 1024^2 square array,
    em_sub, tol 1e-8, max_iters 1000 (reference defaults), points sharded
    round robin over the ranks ("batched over sweep points across GPUs"):
    strong scaling, total work fixed.  Step = the whole sweep."""
    import numpy as np
    import torch

    ws, rank, local = _dist()
    torch.cuda.set_device(local)
    if ws > 1:
        import torch.distributed as dist

        dist.init_process_group("nccl", device_id=torch.device("cuda", local))
    import paper_2001_08289_b200 as fb
    from paper_2001_08289_b200 import native
    from paper_2001_08289_b200.sweep import _solve_local_gpu, c5_points, shard, solve_sweep

    n = 1024
    pm = fb.build_square_array(n, 0.5)
    pts = c5_points(a.c5_points)
    cfgs = [fb.SolverConfig(scheme=fb.SchemeKind.EYRE_MILTON_SUB, sigma1=s, tol=1e-8, max_iters=1000,
                            interval=fb.SpectralInterval(ALPHA, BETA)) for s in pts]
    mine = [cfgs[i] for i in shard(len(cfgs), rank, ws)]
    _solve_local_gpu(pm, mine[:2])  # warm up
    stream = torch.cuda.current_stream()
    times, recs = [], None
    clocks = ClockSampler(local)
    clocks.start()
    launches0 = native.lib().fftc_launch_count()
    for step in range(max(1, a.steps)):
        if ws > 1:
            import torch.distributed as dist

            dist.barrier()
        torch.cuda.synchronize()
        e0 = torch.cuda.Event(enable_timing=True)
        e1 = torch.cuda.Event(enable_timing=True)
        e0.record(stream)
        recs = solve_sweep(pm, cfgs)
        e1.record(stream)
        torch.cuda.synchronize()
        times.append(e0.elapsed_time(e1))
    launches = native.lib().fftc_launch_count() - launches0
    clk = clocks.stop()
    ms = sum(times) / len(times)
    # end to end: a fresh host phase map per step (chi host->device inside the
    # timed region, histories device->host), through the public sweep API
    chi_host = np.asarray(pm.chi)
    if ws > 1:
        dist.barrier()
    torch.cuda.synchronize()
    f0 = torch.cuda.Event(enable_timing=True)
    f1 = torch.cuda.Event(enable_timing=True)
    t_wall = time.perf_counter()
    f0.record(stream)
    recs_e2e = solve_sweep(fb.PhaseMap(chi_host), cfgs)
    f1.record(stream)
    torch.cuda.synchronize()
    ms_e2e = max(f0.elapsed_time(f1), 1e3 * (time.perf_counter() - t_wall))
    if ws > 1:
        import torch.distributed as dist

        t = torch.tensor([ms, ms_e2e], device="cuda", dtype=torch.float64)
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        ms, ms_e2e = float(t[0]), float(t[1])
    vox = sum(n * n * r["iterations"] for r in recs)
    value = vox / (ms / 1e3)
    e2e_value = sum(n * n * r["iterations"] for r in recs_e2e) / (ms_e2e / 1e3)
    hbm, src = _peaks()
    V = 32.0
    bpv = 8 * V + 7 * 0.25 * V + 2
    # roofline of the dominant kernel: per-launch CUDA events over a few points
    # solved one after another (profiling mode: one iteration per sync)
    from paper_2001_08289_b200.solver import _solve_aug

    native.profile(True)
    for c in cfgs[:4]:
        _solve_aug(pm, c, True, want_fields=False)
    torch.cuda.synchronize()
    kstats = native.kernel_stats()
    native.profile(False)
    frac = float(np.asarray(pm.chi).mean())
    roof = None
    if kstats:
        name, (nl, tms) = max(((k, v) for k, v in kstats.items() if k.startswith("sweep")), key=lambda kv: kv[1][1])
        per_launch_ms = tms / nl
        bl = _bytes_per_voxel("em_sub", 2, frac)[name] * n * n
        achieved = bl / (per_launch_ms / 1e3) / 1e9
        roof = {"bound": "hbm", "kernel": name, "achieved": achieved, "peak": hbm, "unit": "GB/s",
                "frac": achieved / hbm, "traffic": None, "peak_source": src, "bytes_per_launch": bl,
                "avg_launch_ms": per_launch_ms, "launches": nl,
                "fft_gpoints_per_s": _fft_passes(name, {"em_sub": 1}) * 2 * n * n / (per_launch_ms / 1e3) / 1e9,
                "timing": "CUDA events around every launch of 4 points solved in turn (one iteration per sync)"}
    conv = sum(1 for r in recs if r["status"].value == "Converged")
    line = {"metric": "fp64 voxel-iterations/sec of the FFT iteration", "value": value,
            "unit": "voxel-iterations/s", "n_gpus": ws, "steps": len(times), "warmup": 1, "ms_per_step": ms,
            "higher_is_better": True, "scaling": "strong", "vs_baseline": None, "dtype": "f64 (complex128)",
            "data": "synthetic (seeded sigma1 points, reference square-array builder)",
            "config": {"workload": f"BASELINE configs[4]: {len(cfgs)} complex sigma1 points, em_sub, {n}^2, tol 1e-8, "
                                   "max_iters 1000", "parallelism": f"points sharded over {ws} GPU(s)"},
            "iteration_roofline": {"bytes_per_voxel_iter_schedule": bpv, "frac_schedule_bytes": value * bpv / 1e9 / hbm / ws,
                                   "peak_gbs": hbm, "peak_source": src},
            "roofline": roof,
            "e2e": {"value": e2e_value, "unit": "voxel-iterations/s", "h2d_bytes_per_step": n * n,
                    "d2h_bytes_per_step": 24 * sum(r["iterations"] for r in recs_e2e) + 256 * len(recs_e2e)},
            "gpu_launches": int(launches * ws), "clocks": clk, "points_converged": conv, "points_total": len(recs),
            "total_iterations": sum(r["iterations"] for r in recs)}
    if ws == 1 and not a.no_cpu_baseline:
        tot_v, tot_t = 0, 0.0
        for p_ in pts[:2]:
            v_, t_ = _oracle_sample(("em_sub", p_, n, a.cpu_iters))
            tot_v += v_
            tot_t += t_
        line["cpu_baseline"] = {"value": tot_v / tot_t, "unit": "voxel-iterations/s", "cores": 1, "kind": "port",
                                "sample": f"2 of the sweep's sigma1 points, em_sub on {n}^2, {a.cpu_iters} iterations each "
                                          f"(tol=1e-300), oracle/fftcond_oracle.py, {tot_t:.1f} s of CPU work"}
    if rank == 0:
        print(json.dumps(line), flush=True)
    if ws > 1:
        import torch.distributed as dist

        dist.destroy_process_group()
    return 0


def run_3d(a):
    """BASELINE configs[2] (C3: 512^3 cube, em_sub, sigma1 = 100, e0 = x) and
    configs[3] (C4: 1024^3 seeded random medium, f = 0.30, basic, sigma1 = 50,
    e0 = (1,1,1)/sqrt 3), tol 1e-8.  One step = one whole solve through the
    public API (host phase map in, history out).  C4 on N > 1 GPUs runs the
    z-slab decomposition with the transposes fused into the column passes
    (CUDA IPC peer buffers); time = max over ranks (strong scaling)."""
    import numpy as np
    import torch

    ws, rank, local = _dist()
    torch.cuda.set_device(local)
    if ws > 1:
        import torch.distributed as dist

        dist.init_process_group("nccl", device_id=torch.device("cuda", local))
    import paper_2001_08289_b200 as fb
    from paper_2001_08289_b200 import native
    from paper_2001_08289_b200.slab import solve_slab

    iv = fb.SpectralInterval(ALPHA, BETA)
    if a.workload == "c3":
        n = a.n3d or 512
        if ws > 1:
            raise SystemExit("c3 is a single-GPU configuration (BASELINE configs[2])")
        pm = fb.build_cube_array(n, 2 * int(round(0.63 * n / 2)))
        cfg = fb.SolverConfig(scheme=fb.SchemeKind.EYRE_MILTON_SUB, sigma1=100.0, tol=1e-8, max_iters=20000,
                              e0=(1.0, 0.0, 0.0), interval=iv)
        work = f"BASELINE configs[2]: {n}^3 centred cube side {2 * int(round(0.63 * n / 2))}, em_sub, sigma1=100, tol 1e-8"
        bpv = 15 * 48 + 6 * float(pm.volume_fraction) * 48 + 2
    else:
        n = a.n3d or 1024
        pm = fb.build_random_medium(n, 3, seed=20260809, smoothing=4.0, fraction=0.30)
        cfg = fb.SolverConfig(scheme=fb.SchemeKind.BASIC, sigma1=50.0, tol=1e-8, max_iters=20000,
                              e0=(1 / 3 ** 0.5,) * 3)
        work = (f"BASELINE configs[3]: {n}^3 random medium (seed 20260809, smoothing 4, f 0.30), basic, "
                f"sigma1=50, tol 1e-8")
        bpv = 11 * 48 + 2

    def one(c):
        if ws > 1:
            return solve_slab(pm.chi, c, fused=True)
        r = fb.solve(pm, c, fields=False)  # no E/J output fields: 96 GB at 1024^3
        return {"iterations": r.iterations, "status": r.status, "sigma_star": r.sigma_star, "fused": False}

    warm = fb.SolverConfig(scheme=cfg.scheme, sigma1=cfg.sigma1, tol=1e-300, max_iters=3, e0=cfg.e0,
                           interval=cfg.interval)
    for _ in range(max(1, a.warmup)):
        one(warm)
    stream = torch.cuda.current_stream()
    clocks = ClockSampler(local)
    clocks.start()
    launches0 = native.lib().fftc_launch_count()
    times, rec = [], None
    for _ in range(a.steps):
        if ws > 1:
            torch.distributed.barrier()
        torch.cuda.synchronize()
        e0 = torch.cuda.Event(enable_timing=True)
        e1 = torch.cuda.Event(enable_timing=True)
        e0.record(stream)
        rec = one(cfg)
        e1.record(stream)
        torch.cuda.synchronize()
        times.append(e0.elapsed_time(e1))
    clk = clocks.stop()
    launches = native.lib().fftc_launch_count() - launches0
    ms = sum(times) / len(times)
    if ws > 1:
        t = torch.tensor([ms, float(launches)], device="cuda", dtype=torch.float64)
        torch.distributed.all_reduce(t[:1], op=torch.distributed.ReduceOp.MAX)
        torch.distributed.all_reduce(t[1:], op=torch.distributed.ReduceOp.SUM)
        ms, launches = float(t[0]), int(t[1])
    vox = n ** 3 * rec["iterations"]
    value = vox / (ms / 1e3)
    hbm, src = _peaks()
    line = {"metric": "fp64 voxel-iterations/sec of the FFT iteration", "value": value,
            "unit": "voxel-iterations/s", "n_gpus": ws, "steps": len(times), "warmup": a.warmup, "ms_per_step": ms,
            "higher_is_better": True, "scaling": "strong", "vs_baseline": None, "dtype": "f64 (complex128)",
            "data": "synthetic (seeded reference-style builders)",
            "config": {"workload": work, "grid": [n, n, n],
                       "parallelism": f"z-slabs over {ws} GPUs, transposes fused into the column passes"
                       if ws > 1 else "single GPU",
                       "l2": "fields of 6-48 GiB >> 126 MB L2"},
            "iteration_roofline": {"bytes_per_voxel_iter_survey": bpv, "achieved_gbs": value * bpv / 1e9 / ws,
                                   "frac": value * bpv / 1e9 / hbm / ws, "peak_gbs": hbm, "peak_source": src},
            "e2e": {"value": value, "unit": "voxel-iterations/s", "h2d_bytes_per_step": n ** 3,
                    "d2h_bytes_per_step": 24 * rec["iterations"],
                    "note": "each step is one solve through the public API: host phase map in, history out"},
            "gpu_launches": int(launches), "clocks": clk, "iterations": rec["iterations"],
            "status": rec["status"].value, "sigma_star": [rec["sigma_star"].real, rec["sigma_star"].imag],
            "fused_transposes": bool(rec.get("fused", False))}
    if rank == 0:
        print(json.dumps(line), flush=True)
    if ws > 1:
        torch.distributed.destroy_process_group()
    return 0


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=3)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", choices=["ours", "reference"], default="ours")
    ap.add_argument("--workload", choices=sorted(WORKLOADS), default="c2")
    ap.add_argument("--ref-iters", type=int, default=4, help="iterations per solve per reference step")
    ap.add_argument("--cpu-iters", type=int, default=6, help="iterations per solve in cpu_baseline")
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--c5-points", type=int, default=256)
    ap.add_argument("--n3d", type=int, default=0, help="c3/c4 grid side (default: the BASELINE size)")
    a = ap.parse_args()
    set_workload(a.workload)
    if a.workload == "c5" and a.impl == "ours":
        return run_c5(a)
    if a.workload in ("c3", "c4") and a.impl == "ours":
        return run_3d(a)
    if a.impl == "reference":
        return run_reference(a)
    return run_ours(a)


if __name__ == "__main__":
    sys.exit(main())
