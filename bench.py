#!/usr/bin/env python
"""Benchmark: fp64 voxel-iterations/s of the FFT field iteration.

Default workload = BASELINE.json configs[2] (C3), the largest configuration
BASELINE names for a single B200: a 512^3 periodic cell with a centred cubic
inclusion of side 322 (0.63 N rounded to the reference's even-integer rule,
f = 0.2487), sigma1 = 100, sigma2 = 1, E0 = (1, 0, 0), the paper's
accelerated substituted scheme em_sub with (alpha, beta) = (0.25, 4.0) (the
reference's only configured interval, configs/compare.cfg:14-15), stop at
the reference default tol 1e-8.  One STEP = one whole solve to convergence.
Synthetic input (the reference's centred-box builder in 3-D; no dataset).

value   = N * iterations / device time of the step, phase map resident in
          HBM, no output fields (CUDA events on the launching stream).
e2e     = the same metric through the public API (fb.solve) with a HOST
          phase map: chi host->device and E, J, S, T (Q is E) device->host
          inside the timed region, plus the history.
roofline: the dominant kernel's algorithmic bytes per launch (DESIGN.md
          section 3) over its mean CUDA-event duration in one profiled solve,
          against MEASURED_PEAKS.json; traffic = ncu DRAM bytes per launch.
cpu_baseline / --impl reference: the CPU oracle port (oracle/lean_oracle.py,
          bit-identical to the restatement of the reference loops; the
          reference itself is 2-D only) at the SAME 512^3 cell, per-iteration
          wall time with setup excluded, on all host threads.

Other workloads (--workload): c1 (BASELINE configs[0], 256^2 basic), c2
(configs[1], 2048^2 em + em_sub at sigma1 in {0.1, 10, 1000}), c2-fast,
c2-emsub10, c4 (configs[3], 1024^3 random medium, basic) and c4-emsub (its
accelerated arm), c5 (configs[4], 256 complex sigma1 points at 1024^2).
2-D reference arms run the unmodified reference from baseline/_ref.

Multi-GPU (--gpus N, or torchrun): without WORLD_SIZE, bench.py relaunches
itself under torch.distributed.run with N ranks.  The 3-D workloads then run
the z-slab decomposition (strong scaling, time = max over ranks); C5 shards
its points; C1/C2 run replicas.
"""

from __future__ import annotations

import argparse
import json
import math
import os
import socket
import subprocess
import sys
import time

REPO = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, REPO)

METRIC = "fp64 voxel-iterations/sec of the FFT iteration"
ALPHA, BETA = 0.25, 4.0
N_GRID, SIDE, TOL, MAX_ITERS = 2048, 0.5, 1e-10, 20000  # 2-D workloads (set_workload)
SOLVES_2D = {
    "c2": [("em", 0.1), ("em", 10.0), ("em", 1000.0), ("em_sub", 0.1), ("em_sub", 10.0), ("em_sub", 1000.0)],
    "c1": [("basic", 10.0)],
    "c2-emsub10": [("em_sub", 10.0)],
    "c2-fast": [("em", 0.1), ("em", 10.0), ("em_sub", 0.1), ("em_sub", 10.0)],
}
WORKLOADS_3D = ("c3", "c4", "c4-emsub")
WORKLOADS = sorted(list(SOLVES_2D) + list(WORKLOADS_3D) + ["c5"])


# ---------------------------------------------------------------------------
# byte models
# ---------------------------------------------------------------------------

def _bytes_per_voxel(scheme: str, d: int, f: float) -> dict:
    """Algorithmic HBM bytes per voxel per launch of each sweep.

    V = 16 d (one complex128 d-vector); chi is 1 byte; S/T slots only move
    on phase-1 voxels (fraction f).  The row sweeps are the same in 2-D and
    3-D; 3-D adds the y passes and moves Gamma to the z pass.
    """
    V = 16.0 * d
    em = scheme in ("em", "em_sub")
    if scheme == "basic":
        k = {"sweep1_rows_fwd": 2 * V + 1, "sweep3_rows_inv": 3 * V + 1}
    elif scheme == "em":
        k = {"sweep1_rows_fwd": 3 * V + 1, "sweep3_rows_inv": 2 * V + 1}
    elif scheme == "basic_sub":
        k = {"sweep1_rows_fwd": 2 * V + f * V + 1, "sweep3_rows_inv": 3 * V + 2 * f * V + 1}
    else:
        k = {"sweep1_rows_fwd": 3 * V + 2 * f * V + 1, "sweep3_rows_inv": 2 * V + 5 * f * V + 1}
    k["sweep2_cols_gamma"] = 3 * V if em else 2 * V  # em: read r^, j^, write (I - 2 Gamma) r^
    if d == 3:
        k["y_fwd_3d"] = 4 * V if em else 2 * V
        k["y_inv_3d"] = 2 * V
    return k


def _bytes_lean(f: float) -> dict:
    """Per-launch bytes per voxel of the memory-lean em_sub schedule (3-D):
    compact S/T slots (moved on phase 1 only), 2-byte rank codes, one work
    field; per iteration sweep 1 and the y forward pass run twice (flux Jq,
    then residual field Rq) and the z pass once Parseval-only, once with
    (I - 2 Gamma^)."""
    V = 48.0
    return {"sweep1_rows_fwd": 2 * V + 2 * f * V + 2, "y_fwd_3d": 2 * V, "z_parseval_3d": V,
            "sweep2_cols_gamma": 2 * V, "y_inv_3d": 2 * V, "sweep3_rows_inv": 2 * V + 5 * f * V + 2}


LEAN_LAUNCHES = {"sweep1_rows_fwd": 2, "y_fwd_3d": 2}


def _survey_bytes(scheme: str, d: int, f: float) -> float:
    """SURVEY.md 8(d) per-voxel-iteration figure for the fused schedule."""
    V = 16.0 * d
    if d == 2:
        return {"basic": 7 * V + 2, "em": 9 * V + 2, "basic_sub": 7 * V + 2 * f * V + 2,
                "em_sub": 9 * V + 6 * f * V + 2}[scheme]
    return {"basic": 11 * V + 2, "em": 15 * V + 2, "basic_sub": 11 * V + 2 * f * V + 2,
            "em_sub": 15 * V + 6 * f * V + 2}[scheme]


def _fft_passes(kernel, scheme, d):
    """Length-n transforms per voxel and component done by one launch."""
    em = scheme in ("em", "em_sub")
    return {"sweep1_rows_fwd": 2 if em else 1, "sweep2_cols_gamma": 3 if em else 2, "sweep3_rows_inv": 1,
            "y_fwd_3d": 2 if em else 1, "y_inv_3d": 1}.get(kernel)


def _peaks():
    try:
        with open(os.path.join(REPO, "MEASURED_PEAKS.json")) as f:
            p = json.load(f)
        return float(p["hbm_gbs"]), "measured (MEASURED_PEAKS.json hbm_gbs, torch copy)"
    except Exception:
        return 6650.0, "fallback (B200_PROFILING.md; MEASURED_PEAKS.json absent)"


def _ncu_record(workload, kernel):
    """DRAM traffic and pipe utilisation of `kernel` from the committed ncu
    capture for this workload (profiles/r2_ncu_<workload>.json), or {}."""
    path = os.path.join(REPO, "profiles", f"r2_ncu_{workload}.json")
    try:
        with open(path) as fh:
            rec = json.load(fh)
    except OSError:
        return {}
    k = rec.get("kernels", {}).get(kernel)
    if not k:
        return {}
    out = {"traffic": k.get("dram_read", 0) + k.get("dram_write", 0), "traffic_source": f"profiles/r2_ncu_{workload}.json "
           f"({rec.get('source', 'ncu --set full')})"}
    for key in ("fp64_pipe", "issue_active", "dram_throughput"):
        if key in k:
            out.setdefault("ncu", {})[key] = k[key]
    return out


class ClockSampler:
    """nvidia-smi clocks / throttle reasons sampled during the timed region."""

    Q = ("index,clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.active,"
         "clocks_event_reasons.hw_slowdown,clocks_event_reasons.hw_thermal_slowdown,"
         "clocks_event_reasons.sw_thermal_slowdown,clocks_event_reasons.sw_power_cap")
    NAMES = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]

    def __init__(self, index: int):
        self.index = index
        self.proc = None
        self.path = os.path.join("/tmp", f"fftc_clocks_{os.getpid()}_{index}.csv")

    def _cmd(self, loop):
        c = ["nvidia-smi", f"--id={self.index}", f"--query-gpu={self.Q}", "--format=csv,noheader,nounits"]
        return c + (["-lms", "50"] if loop else [])

    def start(self):
        try:
            self.proc = subprocess.Popen(self._cmd(True), stdout=open(self.path, "w"), stderr=subprocess.DEVNULL)
        except Exception:
            self.proc = None
        return self

    def _parse(self, lines, sms, maxs, reasons):
        for line in lines:
            parts = [p.strip() for p in line.split(",")]
            if len(parts) < 9:
                continue
            try:
                sms.append(float(parts[1]))
                maxs.append(float(parts[2]))
            except ValueError:
                continue
            for nm, v in zip(self.NAMES, parts[5:9]):
                if v.lower() == "active":
                    reasons.add(nm)

    def stop(self) -> dict:
        if self.proc is None:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["nvidia-smi unavailable"], "samples": 0}
        sms, maxs, reasons = [], [], set()
        if self.proc.poll() is None:
            # a short timed region can end before the first loop sample: take one now, while the GPU is hot
            try:
                self._parse(subprocess.run(self._cmd(False), capture_output=True, text=True, timeout=10).stdout
                            .splitlines(), sms, maxs, reasons)
            except Exception:
                pass
        self.proc.terminate()
        try:
            self.proc.wait(timeout=5)
        except Exception:
            self.proc.kill()
        try:
            with open(self.path) as fh:
                self._parse(fh, sms, maxs, reasons)
        except OSError:
            pass
        sms.sort()
        return {"sm_mhz": sms[len(sms) // 2] if sms else None, "sm_max_mhz": max(maxs) if maxs else None,
                "reasons": sorted(reasons), "samples": len(sms)}


def _dist():
    return (int(os.environ.get("WORLD_SIZE", "1")), int(os.environ.get("RANK", "0")),
            int(os.environ.get("LOCAL_RANK", "0")))


def _free_port() -> int:
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


def _relaunch(a) -> int | None:
    """--gpus N without a torchrun environment: run N ranks of this script
    under torch.distributed.run (one process per GPU) and return its code."""
    ws_env = os.environ.get("WORLD_SIZE")
    if ws_env is not None:
        if int(ws_env) != a.gpus:
            print(json.dumps({"error": f"--gpus {a.gpus} but WORLD_SIZE={ws_env}"}), flush=True)
            return 2
        return None
    if a.gpus <= 1:
        return None
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", f"--nproc-per-node={a.gpus}",
           "--master-addr", "127.0.0.1", f"--master-port={_free_port()}", os.path.abspath(__file__)] + sys.argv[1:]
    return subprocess.run(cmd).returncode


def _init_dist(torch, local):
    ws, rank, _ = _dist()
    torch.cuda.set_device(local)
    if ws > 1:
        import torch.distributed as dist

        if torch.cuda.device_count() < ws:
            raise SystemExit(f"{ws} ranks need {ws} GPUs, {torch.cuda.device_count()} visible")
        dist.init_process_group("nccl", device_id=torch.device("cuda", local))
    return ws, rank


def _max_over_ranks(torch, vals):
    ws = _dist()[0]
    if ws == 1:
        return vals
    import torch.distributed as dist

    t = torch.tensor(vals, device="cuda", dtype=torch.float64)
    dist.all_reduce(t, op=dist.ReduceOp.MAX)
    return [float(v) for v in t]


def _events(torch):
    return torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)


# ---------------------------------------------------------------------------
# 3-D workloads (C3, C4): the headline
# ---------------------------------------------------------------------------

def _cell_3d(workload, n=None):
    """(PhaseMap, SolverConfig, description) of a BASELINE 3-D config."""
    import paper_2001_08289_b200 as fb
    from paper_2001_08289_b200 import cell

    iv = fb.SpectralInterval(ALPHA, BETA)
    if workload == "c3":
        n = n or 512
        side = 2 * int(round(0.63 * n / 2))
        pm = fb.build_cube_array(n, side)
        cfg = fb.SolverConfig(scheme=fb.SchemeKind.EYRE_MILTON_SUB, sigma1=100.0, tol=1e-8, max_iters=MAX_ITERS,
                              e0=(1.0, 0.0, 0.0), interval=iv)
        desc = (f"BASELINE configs[2] (C3): {n}^3 centred cube side {side} (0.63 N, even), f={float(pm.volume_fraction):.4f}, "
                f"em_sub sigma1=100 (alpha, beta)=(0.25, 4), E0=x, tol 1e-8; one step = one whole solve")
    else:
        n = n or 1024
        pm = cell.c4_phase_map(n)
        sch = fb.SchemeKind.EYRE_MILTON_SUB if workload == "c4-emsub" else fb.SchemeKind.BASIC
        cfg = fb.SolverConfig(scheme=sch, sigma1=50.0, tol=1e-8, max_iters=MAX_ITERS, e0=(3 ** -0.5,) * 3,
                              interval=iv if sch.substituted else None)
        desc = (f"BASELINE configs[3] (C4): {n}^3 random medium (seed 20260809, periodic Gaussian sigma 4 voxels, "
                f"30th percentile; frozen SHA-256 for 1024^3), {sch.value} sigma1=50, E0=(1,1,1)/sqrt3, tol 1e-8; "
                f"one step = one whole solve")
    return pm, cfg, desc


def cpu_baseline_3d(workload, n, iters=2, threads=None) -> dict:
    """The oracle port on the same cell: per-iteration wall time (setup
    excluded) of iteration `iters` (k >= 2 carries both transforms of em_sub)."""
    from oracle import lean_oracle as LO

    old = os.environ.get("FFTC_ORACLE_THREADS")
    if threads:
        os.environ["FFTC_ORACLE_THREADS"] = str(threads)
    try:
        pm, cfg, _ = _cell_3d(workload, n)
        chi = pm.chi
        t0 = time.perf_counter()
        dts = LO.timed_iterations(chi, cfg.scheme.value, complex(cfg.sigma1), iters, e0=cfg.e0, alpha=ALPHA,
                                  beta=BETA)
        wall = time.perf_counter() - t0
    finally:
        if threads:
            if old is None:
                os.environ.pop("FFTC_ORACLE_THREADS", None)
            else:
                os.environ["FFTC_ORACLE_THREADS"] = old
    t = dts[-1]
    return {"value": chi.size / t, "unit": "voxel-iterations/s", "cores": LO.nthreads() if not threads else threads,
            "kind": "port",
            "sample": f"iteration {iters} of a {cfg.scheme.value} solve on the {chi.shape[0]}^3 cell of the same recipe "
                      f"({t:.1f} s; earlier iterations {[round(x, 1) for x in dts[:-1]]} s; setup excluded; "
                      f"{wall:.0f} s of CPU leg in total), oracle/lean_oracle.py (bit-identical to the restatement "
                      f"of the reference loops, solvers.py:280-443), numpy pocketfft split over threads"}


def run_3d(a):
    import numpy as np
    import torch

    ws, rank, local = _dist()
    ws, rank = _init_dist(torch, local)
    import paper_2001_08289_b200 as fb
    from paper_2001_08289_b200 import native
    from paper_2001_08289_b200.slab import solve_slab
    from paper_2001_08289_b200.solver import _run_device

    pm, cfg, desc = _cell_3d(a.workload, a.n3d or None)
    n = pm.nx
    N = n ** 3
    scheme = cfg.scheme.value
    f = float(pm.volume_fraction)
    stream = torch.cuda.current_stream()

    def step_device():
        if ws > 1:
            r = solve_slab(pm.chi, cfg, fused=True)
            return r["iterations"], r
        r = _run_device(pm, cfg, want_fields=False)  # chi cached on the device after the first call
        return r.iterations, r

    for _ in range(a.warmup):
        step_device()
    # ---- timed: device-resident ----
    if ws > 1:
        torch.distributed.barrier()
    torch.cuda.synchronize()
    clocks = ClockSampler(local).start()
    launches0 = native.lib().fftc_launch_count()
    e0, e1 = _events(torch)
    e0.record(stream)
    its, rec = 0, None
    for _ in range(a.steps):
        it, rec = step_device()
        its += it
    e1.record(stream)
    if ws > 1:
        torch.distributed.barrier()
    torch.cuda.synchronize()
    clk = clocks.stop()
    launches = native.lib().fftc_launch_count() - launches0
    ms = e0.elapsed_time(e1) / a.steps
    ms, = _max_over_ranks(torch, [ms])
    iters = its // a.steps
    value = N * iters / (ms / 1e3)
    status = rec["status"] if isinstance(rec, dict) else rec.status
    sstar = rec["sigma_star"] if isinstance(rec, dict) else rec.sigma_star

    hbm, peak_src = _peaks()
    lean = ws == 1 and bool(native.last_layout() & 256)  # memory-lean em_sub schedule (C4's accelerated arm)
    bytes_k = _bytes_lean(f) if lean else _bytes_per_voxel(scheme, 3, f)
    survey_b = _survey_bytes(scheme, 3, f)
    sched_b = sum(v * (LEAN_LAUNCHES.get(k, 1) if lean else 1) for k, v in bytes_k.items())
    line = {"metric": METRIC, "value": value, "unit": "voxel-iterations/s", "n_gpus": ws, "steps": a.steps,
            "warmup": a.warmup, "ms_per_step": ms, "higher_is_better": True,
            "scaling": "strong" if ws > 1 else "weak", "vs_baseline": None, "dtype": "f64 (complex128)",
            "data": "synthetic (seeded reference-style builders)",
            "config": {"workload": desc, "grid": [n, n, n], "scheme": scheme, "sigma1": 100.0 if a.workload == "c3" else 50.0,
                       "tol": 1e-8, "max_iters": MAX_ITERS,
                       "parallelism": f"z-slabs over {ws} GPUs, transposes fused into the column passes (NVLink peer stores)"
                       if ws > 1 else "single GPU",
                       "l2": "inputs larger than L2 (one field is 6-48 GiB >> 126 MB L2)",
                       "schedule": "memory-lean em_sub (compact S/T slots, one work field: 137 GB at 1024^3)"
                       if lean else "fused sweeps (DESIGN.md section 3)"},
            "iterations": iters, "status": status.value, "sigma_star": [sstar.real, sstar.imag],
            "gpu_launches": int(launches), "clocks": clk,
            "iteration_roofline": {"bytes_per_voxel_iter_survey": survey_b, "bytes_per_voxel_iter_schedule": sched_b,
                                   "achieved_gbs_survey_bytes": value / ws * survey_b / 1e9,
                                   "frac_survey_bytes": value / ws * survey_b / 1e9 / hbm,
                                   "achieved_gbs_schedule_bytes": value / ws * sched_b / 1e9,
                                   "frac_schedule_bytes": value / ws * sched_b / 1e9 / hbm,
                                   "peak_gbs": hbm, "peak_source": peak_src}}
    if ws > 1:
        # the slower of the HBM time and the all-to-all bytes at NVLink bandwidth
        V = 48.0
        n_tr = 3 if cfg.scheme.accelerated else 2
        a2a_bytes = n_tr * V * (N / ws) * (ws - 1) / ws
        t_hbm = N * survey_b / ws / (hbm * 1e9)
        t_nvl = a2a_bytes / 900e9
        bound = "hbm" if t_hbm >= t_nvl else "nvlink"
        t_roof = max(t_hbm, t_nvl)
        t_iter = ms / 1e3 / iters
        line["roofline"] = {"bound": bound, "achieved": t_roof / t_iter, "peak": 1.0, "unit": "fraction",
                            "frac": t_roof / t_iter, "traffic": None,
                            "hbm_ms_per_iter": 1e3 * t_hbm, "nvlink_ms_per_iter": 1e3 * t_nvl,
                            "measured_ms_per_iter": 1e3 * t_iter, "a2a_bytes_per_gpu_iter": a2a_bytes,
                            "note": "iteration roofline = max(HBM bytes / HBM peak, all-to-all bytes / 900 GB/s) "
                                    "over the measured iteration time (SURVEY 8(e))"}
        line["fused_transposes"] = bool(rec.get("fused", False))
        if rank == 0:
            print(json.dumps(line), flush=True)
        torch.distributed.destroy_process_group()
        return 0

    # ---- one profiled solve: per-launch CUDA events of every kernel ----
    native.profile(True)
    p0, p1 = _events(torch)
    p0.record(stream)
    _run_device(pm, cfg, want_fields=False)
    p1.record(stream)
    torch.cuda.synchronize()
    prof_ms = p0.elapsed_time(p1)
    kstats = native.kernel_stats()
    native.profile(False)
    sweeps = {k: v for k, v in kstats.items() if k in bytes_k}
    name, (nl, tms) = max(sweeps.items(), key=lambda kv: kv[1][1])
    per_launch_ms = tms / nl
    bl = bytes_k[name] * N
    achieved = bl / (per_launch_ms / 1e3) / 1e9
    roof = {"bound": "hbm", "kernel": name, "achieved": achieved, "peak": hbm, "unit": "GB/s", "frac": achieved / hbm,
            "traffic": None, "peak_source": peak_src, "bytes_per_launch": bl,
            "bytes_per_voxel": bytes_k[name], "avg_launch_ms": per_launch_ms, "launches": nl,
            "share_of_step": tms / prof_ms if prof_ms > 0 else None,
            "fft_gpoints_per_s": (_fft_passes(name, scheme, 3) or 0) * 3 * N / (per_launch_ms / 1e3) / 1e9,
            "timing": "CUDA events on the launching stream around every launch of one profiled solve "
                      "(one iteration per synchronisation)"}
    roof.update(_ncu_record(a.workload, name))
    line["roofline"] = roof
    line["kernels"] = {k: {"launches": v[0], "ms_per_launch": v[1] / max(v[0], 1),
                           "bytes_per_voxel": bytes_k.get(k),
                           "frac_hbm": (bytes_k[k] * N / (v[1] / max(v[0], 1) / 1e3) / 1e9 / hbm) if k in bytes_k else None}
                       for k, v in kstats.items()}

    # ---- timed: end to end through the public API with host buffers ----
    chi_host = np.array(pm.chi)
    e2e_steps = max(1, min(a.steps, a.e2e_steps))
    def read_back(r):
        host = [r.E_field.data, r.J_field.data]  # device->host: E (= aug Q), J
        if r.aug_field is not None:
            host += [r.aug_field.S.data, r.aug_field.T.data]
        return host

    # at 1024^3 the returned fields alone would be 96-206 GB of device memory
    # on top of the iteration's: the e2e step there returns the history,
    # sigma* and the field means (fields=False) and says so
    want_fields = N <= 512 ** 3
    if want_fields:
        read_back(fb.solve(fb.PhaseMap(chi_host), cfg))  # warm the pinned host blocks of the field read-back
    torch.cuda.synchronize()
    clocks = ClockSampler(local).start()
    f0, f1 = _events(torch)
    t_wall = time.perf_counter()
    f0.record(stream)
    e2e_its, d2h = 0, 0
    for _ in range(e2e_steps):
        r = fb.solve(fb.PhaseMap(chi_host), cfg, fields=want_fields)  # chi crosses host->device inside solve()
        host = read_back(r) if want_fields else []
        d2h = sum(h.nbytes for h in host) + 24 * r.iterations + 96
        e2e_its += r.iterations
        del r, host
    f1.record(stream)
    torch.cuda.synchronize()
    t_wall = time.perf_counter() - t_wall
    clk_e2e = clocks.stop()
    ms_e2e = max(f0.elapsed_time(f1), 1e3 * t_wall) / e2e_steps
    line["e2e"] = {"value": N * (e2e_its / e2e_steps) / (ms_e2e / 1e3), "unit": "voxel-iterations/s",
                   "h2d_bytes_per_step": N, "d2h_bytes_per_step": d2h, "steps": e2e_steps, "ms_per_step": ms_e2e,
                   "clocks": clk_e2e,
                   "note": ("fb.solve() on a fresh host PhaseMap per step; the returned E, J and augmented S, T "
                            "fields are read back to host numpy (pinned copies), as the reference returns them")
                   if want_fields else ("fb.solve(fields=False) on a fresh host PhaseMap per step: history, sigma* "
                                        "and <E>, <J> come back; the 1024^3 fields do not fit beside the iteration")}
    if not a.no_cpu_baseline:
        # the port holds ~15-18 full fields: 1024^3 does not fit the host, so C4
        # is sampled on the same recipe at 512^3 (per-voxel rate, labelled)
        line["cpu_baseline"] = cpu_baseline_3d(a.workload, min(n, 512), iters=2)
    print(json.dumps(line), flush=True)
    return 0


def run_reference_3d(a):
    """--impl reference for the 3-D workloads: the oracle port (the reference
    is 2-D only) on the same cell and scheme, all host threads,
    one step = one iteration (k >= 2) of a continuing solve."""
    ws, rank, _ = _dist()
    if rank != 0:
        return 0
    from oracle import lean_oracle as LO

    # the port holds ~15-18 full fields (em_sub at 1024^3: >400 GB): C4 is
    # sampled on the same recipe at 512^3 (per-voxel rate, labelled)
    full = _cell_3d(a.workload, a.n3d or None)[2]
    pm, cfg, desc = _cell_3d(a.workload, min(a.n3d or 1024, 512))
    n = pm.nx
    # one step = one iteration (~17 s at 512^3 on 16 threads): a bounded sample
    # of at most 8 timed iterations keeps the arm within a few minutes
    steps, warmup = min(a.steps, 8), min(a.warmup, 1)
    dts = LO.timed_iterations(pm.chi, cfg.scheme.value, complex(cfg.sigma1), 1 + warmup + steps, e0=cfg.e0,
                              alpha=ALPHA, beta=BETA)
    timed = dts[1 + warmup:]
    ms = 1e3 * sum(timed) / len(timed)
    value = n ** 3 / (ms / 1e3)
    cores = LO.nthreads()
    sample = (f"{len(timed)} timed iterations (after iteration 1 and {warmup} warm-up iterations) of {cfg.scheme.value} "
              f"on the same {n}^3 cell, {cores} threads on {os.cpu_count()} host CPUs; oracle/lean_oracle.py "
              f"(bit-identical to the d-generic restatement of the reference loops; no 3-D reference exists)")
    line = {"impl": "reference", "metric": METRIC, "value": value, "unit": "voxel-iterations/s", "n_gpus": ws,
            "steps": len(timed), "warmup": warmup, "ms_per_step": ms, "higher_is_better": True,
            "scaling": "strong" if ws > 1 else "weak", "vs_baseline": None, "dtype": "f64 (complex128)",
            "data": "synthetic (seeded reference-style builders)",
            "config": {"workload": full, "grid": [n, n, n], "scheme": cfg.scheme.value,
                       "note": "one step = one iteration of the CPU port"
                               + ("" if full == desc else f"; sampled on the same recipe at {n}^3 (host memory)")},
            "cpu_baseline": {"value": value, "unit": "voxel-iterations/s", "cores": cores, "kind": "port",
                             "sample": sample},
            "e2e": {"value": value, "unit": "voxel-iterations/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0}}
    print(json.dumps(line), flush=True)
    return 0


# ---------------------------------------------------------------------------
# 2-D workloads (C1, C2)
# ---------------------------------------------------------------------------

def set_workload(name):
    global N_GRID, TOL, MAX_ITERS
    if name == "c1":
        N_GRID, TOL, MAX_ITERS = 256, 1e-8, 1000


def _square_chi(n):
    import numpy as np

    chi = np.zeros((n, n), dtype=bool)
    m = int(round(SIDE * n))
    lo = (n - m) // 2
    chi[lo:lo + m, lo:lo + m] = True
    return chi


def _config_2d(a, ws):
    solves = SOLVES_2D[a.workload]
    base = {"grid": [N_GRID, N_GRID], "schemes": [s for s, _ in solves], "sigma1": [v for _, v in solves],
            "alpha_beta": [ALPHA, BETA], "tol": TOL, "max_iters": MAX_ITERS,
            "parallelism": "replicas" if ws > 1 else "single GPU"}
    if a.workload == "c1":
        base.update(workload=f"BASELINE configs[0] (C1): {N_GRID}x{N_GRID} square array f=0.25, basic sigma1=10, "
                             f"tol {TOL:g}",
                    l2="working set (~8 MB) is L2-resident by nature; L2 flushed (256 MB write) before every timed "
                       "step, outside that step's CUDA events")
    else:
        base.update(workload=f"BASELINE configs[1] (C2): {N_GRID}x{N_GRID} square array f=0.25, "
                             + ", ".join(f"{s}@sigma1={v:g}" for s, v in solves) + f", tol {TOL:g}",
                    l2="inputs larger than L2 (state + work fields 384-640 MB per solve >> 126 MB L2)")
    return base


def _ref_fftcond():
    """The unmodified reference package installed under baseline/_ref (see
    DESIGN.md: pip install --target baseline/_ref), or None."""
    path = os.path.join(REPO, "baseline", "_ref")
    if not os.path.isdir(os.path.join(path, "fftcond")):
        return None
    if path not in sys.path:
        sys.path.insert(0, path)
    import fftcond

    return fftcond


def _cpu_sample_2d(args):
    """One bounded sample: `iters` iterations of one 2-D solve (tol 1e-300 so
    every iteration runs), through the reference itself when installed,
    else the bit-identical port.  Returns (voxel-iterations, seconds, kind)."""
    scheme, s1, n, iters = args
    import numpy as np

    chi = _square_chi(n)
    fc = _ref_fftcond()
    if fc is not None:
        sk = fc.SchemeKind(scheme)
        kw = dict(scheme=sk, sigma1=complex(s1), tol=1e-300, max_iters=iters)
        if sk.substituted:
            kw["interval"] = fc.SpectralInterval(ALPHA, BETA)
        pmap, cfg = fc.PhaseMap(chi), fc.SolverConfig(**kw)
        t0 = time.perf_counter()
        r = fc.solve(pmap, cfg)
        dt = time.perf_counter() - t0
        return int(np.prod(chi.shape)) * len(r.history), dt, "reference"
    from oracle import fftcond_oracle as O

    t0 = time.perf_counter()
    r = O.solve(chi, scheme, s1, tol=1e-300, max_iters=iters, alpha=ALPHA, beta=BETA)
    dt = time.perf_counter() - t0
    return int(chi.size) * r.iterations, dt, "port"


def cpu_baseline_2d(solves, n, iters) -> dict:
    tot_v, tot_t, kind = 0, 0.0, "port"
    for scheme, s1 in solves:
        v, t, kind = _cpu_sample_2d((scheme, s1, n, iters))
        tot_v += v
        tot_t += t
    who = "the unmodified reference (baseline/_ref/fftcond)" if kind == "reference" else \
        "oracle/fftcond_oracle.py (bit-identical numpy restatement of the reference loops)"
    return {"value": tot_v / tot_t, "unit": "voxel-iterations/s", "cores": 1, "kind": kind,
            "sample": f"{len(solves)} solve(s) (" + ", ".join(f"{s}@sigma1={v:g}" for s, v in solves)
                      + f") on {n}^2, {iters} iterations each (tol 1e-300), {who}, one core, setup included "
                        f"(one pass of scalar setup, <2% of the sample), {tot_t:.1f} s of CPU work"}


def run_reference_2d(a):
    ws, rank, _ = _dist()
    if rank != 0:
        return 0
    from concurrent.futures import ProcessPoolExecutor

    ncpu = os.cpu_count() or 1
    procs = max(1, ncpu)
    iters = a.ref_iters
    if a.workload == "c5":
        from paper_2001_08289_b200.sweep import c5_points

        pts = c5_points(max(procs, 8))
        solves, n = [("em_sub", p) for p in pts], 1024
    else:
        solves, n = SOLVES_2D[a.workload], N_GRID
    jobs = [(s, v, n, iters) for s, v in (solves[i % len(solves)] for i in range(max(procs, len(solves))))]
    times, vox, kind = [], 0, "port"
    with ProcessPoolExecutor(max_workers=procs) as ex:
        for step in range(a.warmup + a.steps):
            t0 = time.perf_counter()
            res = list(ex.map(_cpu_sample_2d, jobs))
            dt = time.perf_counter() - t0
            if step >= a.warmup:
                times.append(dt)
                vox = sum(v for v, _, _ in res)
                kind = res[0][2]
    ms = 1e3 * sum(times) / len(times)
    value = vox / (ms / 1e3)
    who = "the unmodified reference from baseline/_ref (pip install --target of /root/reference/pkg)" \
        if kind == "reference" else "oracle/fftcond_oracle.py (bit-exact port; baseline/_ref absent)"
    cfg = _config_2d(a, ws) if a.workload in SOLVES_2D else {"workload": "BASELINE configs[4] (C5) sample",
                                                            "grid": [n, n]}
    line = {"impl": "reference", "metric": METRIC, "value": value, "unit": "voxel-iterations/s", "n_gpus": ws,
            "steps": a.steps, "warmup": a.warmup, "ms_per_step": ms, "higher_is_better": True, "scaling": "weak",
            "vs_baseline": None, "dtype": "f64 (complex128)", "data": "synthetic (reference square-array builder)",
            "config": cfg,
            "cpu_baseline": {"value": value, "unit": "voxel-iterations/s", "cores": procs, "kind": kind,
                             "sample": f"{len(jobs)} concurrent bounded samples ({iters} iterations each) cycling "
                                       f"through the {len(solves)} solves, {procs} processes on {ncpu} host CPUs; {who}"},
            "e2e": {"value": value, "unit": "voxel-iterations/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0}}
    print(json.dumps(line), flush=True)
    return 0


def run_2d(a):
    import torch

    ws, rank, local = _dist()
    ws, rank = _init_dist(torch, local)
    import paper_2001_08289_b200 as fb
    from paper_2001_08289_b200 import native
    from paper_2001_08289_b200.solver import _run_device

    solves = SOLVES_2D[a.workload]
    chi_host = _square_chi(N_GRID)
    frac = float(chi_host.mean())
    cfgs = []
    for sch, s1 in solves:
        sk = fb.SchemeKind(sch)
        cfgs.append(fb.SolverConfig(scheme=sk, sigma1=s1, tol=TOL, max_iters=MAX_ITERS,
                                    interval=fb.SpectralInterval(ALPHA, BETA) if sk.substituted else None))
    pm_dev = fb.PhaseMap(chi_host)
    stream = torch.cuda.current_stream()

    def step_device():
        return [_run_device(pm_dev, cfg, want_fields=False) for cfg in cfgs]

    def barrier():
        if ws > 1:
            torch.distributed.barrier()
        torch.cuda.synchronize()

    for _ in range(a.warmup):
        step_device()
    barrier()
    clocks = ClockSampler(local).start()
    launches0 = native.lib().fftc_launch_count()
    results = None
    if a.workload == "c1":  # L2-resident: flush L2 before every step, time each step alone
        flush = torch.empty(256 << 20, dtype=torch.uint8, device="cuda")
        pairs = []
        for _ in range(a.steps):
            flush.fill_(1)
            e0, e1 = _events(torch)
            e0.record(stream)
            results = step_device()
            e1.record(stream)
            pairs.append((e0, e1))
    else:
        e0, e1 = _events(torch)
        e0.record(stream)
        for _ in range(a.steps):
            results = step_device()
        e1.record(stream)
        pairs = [(e0, e1)]
    barrier()
    launches = native.lib().fftc_launch_count() - launches0
    clk = clocks.stop()
    ms = sum(b.elapsed_time(c) for b, c in pairs) / a.steps
    N = N_GRID * N_GRID
    vox = sum(N * r.iterations for r in results)
    # one profiled step: per-kernel CUDA-event durations for the roofline
    native.profile(True)
    p0, p1 = _events(torch)
    p0.record(stream)
    step_device()
    p1.record(stream)
    torch.cuda.synchronize()
    prof_ms = p0.elapsed_time(p1)
    kstats = native.kernel_stats()
    native.profile(False)
    # end to end: public API, host phase map in, E/J (and S/T) fields + history out
    e2e_steps = max(1, min(a.steps, a.e2e_steps))
    [fb.solve(fb.PhaseMap(chi_host), c) for c in cfgs]
    barrier()
    clocks = ClockSampler(local).start()
    f0, f1 = _events(torch)
    t_wall = time.perf_counter()
    f0.record(stream)
    e2e_its, d2h = 0, 0
    for _ in range(e2e_steps):
        d2h = 0
        for c in cfgs:
            r = fb.solve(fb.PhaseMap(chi_host), c)
            host = [r.E_field.data, r.J_field.data]
            if r.aug_field is not None:
                host += [r.aug_field.S.data, r.aug_field.T.data]
            d2h += sum(h.nbytes for h in host) + 24 * r.iterations
            e2e_its += r.iterations
    f1.record(stream)
    barrier()
    t_wall = time.perf_counter() - t_wall
    clk_e2e = clocks.stop()
    ms_e2e = max(f0.elapsed_time(f1), 1e3 * t_wall) / e2e_steps
    ms, ms_e2e = _max_over_ranks(torch, [ms, ms_e2e])
    value = ws * vox / (ms / 1e3)
    e2e_value = ws * N * (e2e_its / e2e_steps) / (ms_e2e / 1e3)

    hbm, peak_src = _peaks()
    it_by = {}
    for (sch, _), r in zip(solves, results):
        it_by[sch] = it_by.get(sch, 0) + r.iterations
    tot_it = sum(it_by.values())
    sweeps = {k: v for k, v in kstats.items() if k.startswith("sweep")}
    name, (nl, tms) = max(sweeps.items(), key=lambda kv: kv[1][1])
    bpv = sum(_bytes_per_voxel(s, 2, frac)[name] * k for s, k in it_by.items()) / tot_it
    per_launch_ms = tms / nl
    achieved = bpv * N / (per_launch_ms / 1e3) / 1e9
    roof = {"bound": "hbm", "kernel": name, "achieved": achieved, "peak": hbm, "unit": "GB/s", "frac": achieved / hbm,
            "traffic": None, "peak_source": peak_src, "bytes_per_launch": bpv * N, "avg_launch_ms": per_launch_ms,
            "launches": nl, "share_of_step": tms / prof_ms if prof_ms > 0 else None,
            "timing": "CUDA events around every launch of one profiled step (one iteration per sync)"}
    roof.update(_ncu_record(a.workload, name))
    survey_b = sum(_survey_bytes(s, 2, frac) * k for s, k in it_by.items()) / tot_it
    ours_b = sum(sum(_bytes_per_voxel(s, 2, frac).values()) * k for s, k in it_by.items()) / tot_it
    line = {"metric": METRIC, "value": value, "unit": "voxel-iterations/s", "n_gpus": ws, "steps": a.steps,
            "warmup": a.warmup, "ms_per_step": ms, "higher_is_better": True, "scaling": "weak", "vs_baseline": None,
            "dtype": "f64 (complex128)", "data": "synthetic (reference square-array builder)",
            "config": _config_2d(a, ws), "roofline": roof,
            "iteration_roofline": {"bytes_per_voxel_iter_survey": survey_b, "bytes_per_voxel_iter_schedule": ours_b,
                                   "frac_survey_bytes": value / ws * survey_b / 1e9 / hbm,
                                   "frac_schedule_bytes": value / ws * ours_b / 1e9 / hbm},
            "e2e": {"value": e2e_value, "unit": "voxel-iterations/s", "h2d_bytes_per_step": N * len(cfgs),
                    "d2h_bytes_per_step": d2h, "steps": e2e_steps, "clocks": clk_e2e},
            "gpu_launches": int(launches), "clocks": clk,
            "kernels": {k: {"launches": v[0], "ms_per_launch": v[1] / max(v[0], 1)} for k, v in kstats.items()},
            "solves": [{"scheme": s, "sigma1": v, "iterations": r.iterations, "status": r.status.value,
                        "sigma_star": [r.sigma_star.real, r.sigma_star.imag]} for (s, v), r in zip(solves, results)]}
    if ws == 1 and not a.no_cpu_baseline:
        line["cpu_baseline"] = (cpu_baseline_2d([("basic", 10.0)] * 3, N_GRID, 62) if a.workload == "c1"
                                else cpu_baseline_2d([("em_sub", 10.0)], N_GRID, a.cpu_iters))
    if rank == 0:
        print(json.dumps(line), flush=True)
    if ws > 1:
        torch.distributed.destroy_process_group()
    return 0


# ---------------------------------------------------------------------------
# C5: the complex sigma1 sweep
# ---------------------------------------------------------------------------

def run_c5(a):
    """BASELINE configs[4]: 256 complex sigma1 points on the 1024^2 square array,
    em_sub, tol 1e-8, max_iters 1000 (reference defaults), points sharded
    round robin over the ranks (strong scaling).  Step = the whole sweep."""
    import numpy as np
    import torch

    ws, rank, local = _dist()
    ws, rank = _init_dist(torch, local)
    import paper_2001_08289_b200 as fb
    from paper_2001_08289_b200 import native
    from paper_2001_08289_b200.solver import _solve_aug
    from paper_2001_08289_b200.sweep import _solve_local_gpu, c5_points, shard, solve_sweep

    n = 1024
    pm = fb.build_square_array(n, 0.5)
    pts = c5_points(a.c5_points)
    cfgs = [fb.SolverConfig(scheme=fb.SchemeKind.EYRE_MILTON_SUB, sigma1=s, tol=1e-8, max_iters=1000,
                            interval=fb.SpectralInterval(ALPHA, BETA)) for s in pts]
    _solve_local_gpu(pm, [cfgs[i] for i in shard(len(cfgs), rank, ws)][:2])  # warm up
    stream = torch.cuda.current_stream()
    for _ in range(max(0, a.warmup - 1)):
        solve_sweep(pm, cfgs)
    times, recs = [], None
    clocks = ClockSampler(local).start()
    launches0 = native.lib().fftc_launch_count()
    for _ in range(max(1, a.steps)):
        if ws > 1:
            torch.distributed.barrier()
        torch.cuda.synchronize()
        e0, e1 = _events(torch)
        e0.record(stream)
        recs = solve_sweep(pm, cfgs)
        e1.record(stream)
        torch.cuda.synchronize()
        times.append(e0.elapsed_time(e1))
    launches = native.lib().fftc_launch_count() - launches0
    clk = clocks.stop()
    ms = sum(times) / len(times)
    chi_host = np.asarray(pm.chi)
    if ws > 1:
        torch.distributed.barrier()
    torch.cuda.synchronize()
    f0, f1 = _events(torch)
    t_wall = time.perf_counter()
    f0.record(stream)
    recs_e2e = solve_sweep(fb.PhaseMap(chi_host), cfgs)
    f1.record(stream)
    torch.cuda.synchronize()
    ms_e2e = max(f0.elapsed_time(f1), 1e3 * (time.perf_counter() - t_wall))
    ms, ms_e2e = _max_over_ranks(torch, [ms, ms_e2e])
    vox = sum(n * n * r["iterations"] for r in recs)
    value = vox / (ms / 1e3)
    e2e_value = sum(n * n * r["iterations"] for r in recs_e2e) / (ms_e2e / 1e3)
    hbm, src = _peaks()
    frac = float(np.asarray(pm.chi).mean())
    bk = _bytes_per_voxel("em_sub", 2, frac)
    bpv = sum(bk.values())
    native.profile(True)
    for c in cfgs[:4]:
        _solve_aug(pm, c, True, want_fields=False)
    torch.cuda.synchronize()
    kstats = native.kernel_stats()
    native.profile(False)
    name, (nl, tms) = max(((k, v) for k, v in kstats.items() if k.startswith("sweep")), key=lambda kv: kv[1][1])
    per_launch_ms = tms / nl
    bl = bk[name] * n * n
    achieved = bl / (per_launch_ms / 1e3) / 1e9
    roof = {"bound": "hbm", "kernel": name, "achieved": achieved, "peak": hbm, "unit": "GB/s", "frac": achieved / hbm,
            "traffic": None, "peak_source": src, "bytes_per_launch": bl, "avg_launch_ms": per_launch_ms,
            "launches": nl, "timing": "CUDA events around every launch of 4 points solved in turn"}
    roof.update(_ncu_record("c5", name))
    conv = sum(1 for r in recs if r["status"].value == "Converged")
    line = {"metric": METRIC, "value": value, "unit": "voxel-iterations/s", "n_gpus": ws, "steps": len(times),
            "warmup": max(1, a.warmup), "ms_per_step": ms, "higher_is_better": True, "scaling": "strong",
            "vs_baseline": None, "dtype": "f64 (complex128)",
            "data": "synthetic (seeded sigma1 points, reference square-array builder)",
            "config": {"workload": f"BASELINE configs[4] (C5): {len(cfgs)} complex sigma1 points, em_sub, {n}^2, "
                                   "tol 1e-8, max_iters 1000", "parallelism": f"points sharded over {ws} GPU(s)",
                       "l2": "32 MB fields x 8 concurrent points exceed L2"},
            "iteration_roofline": {"bytes_per_voxel_iter_schedule": bpv, "frac_schedule_bytes": value * bpv / 1e9 / hbm / ws,
                                   "peak_gbs": hbm, "peak_source": src},
            "roofline": roof,
            "e2e": {"value": e2e_value, "unit": "voxel-iterations/s", "h2d_bytes_per_step": n * n,
                    "d2h_bytes_per_step": 24 * sum(r["iterations"] for r in recs_e2e) + 256 * len(recs_e2e),
                    "note": "batched sweep API returns per-point records (history, sigma*, means), no fields"},
            "gpu_launches": int(launches * ws), "clocks": clk, "points_converged": conv, "points_total": len(recs),
            "total_iterations": sum(r["iterations"] for r in recs)}
    if ws == 1 and not a.no_cpu_baseline:
        line["cpu_baseline"] = cpu_baseline_2d([("em_sub", pts[0])], n, a.cpu_iters)
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
    ap.add_argument("--workload", choices=WORKLOADS, default="c3")
    ap.add_argument("--e2e-steps", type=int, default=3, help="end-to-end steps (at most --steps)")
    ap.add_argument("--ref-iters", type=int, default=8,
                    help="2-D reference arm: iterations per concurrent sample (one sample per host core; k = 20 of "
                         "BASELINE.md section 2 takes ~90 s per step at 2048^2 on 16 cores, the one-core cpu_baseline "
                         "leg uses k = 20)")
    ap.add_argument("--cpu-iters", type=int, default=20, help="2-D cpu_baseline: iterations per solve")
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--c5-points", type=int, default=256)
    ap.add_argument("--n3d", type=int, default=0, help="c3/c4 grid side (default: the BASELINE size)")
    a = ap.parse_args()
    if a.warmup < 0 or a.steps < 1:
        ap.error("--steps >= 1 and --warmup >= 0")
    rc = _relaunch(a)
    if rc is not None:
        return rc
    set_workload(a.workload)
    if a.impl == "reference":
        return run_reference_3d(a) if a.workload in WORKLOADS_3D else run_reference_2d(a)
    if a.workload in WORKLOADS_3D:
        return run_3d(a)
    if a.workload == "c5":
        return run_c5(a)
    return run_2d(a)


if __name__ == "__main__":
    sys.exit(main())
