"""z-slab decomposed 3-D solve over the ranks of a process group (BASELINE
config 4: 1024^3 random medium, "slab-decomposed across 1/2/4/8 B200 with
NCCL all-to-all FFT transposes").

Rank r owns z-planes [r*nz/G, (r+1)*nz/G) of every field.  Per iteration
(reference loop solvers.py:300-321 / :395-432):

  ROWS_FWD   local: prologue, x-FFT, y-FFT            -> partial <j>, sum|Js|^2
  transpose  all-to-all z-slabs -> y-slabs (A, and B for EM-type schemes)
  MID        local: z-FFT, Gamma projection, Parseval, z-iFFT -> partial residual
  transpose  all-to-all y-slabs -> z-slabs (A)
  all-reduce {<j>, sum|Js|^2, residual}; monitor (identical on every rank)
  ROWS_INV   local: y-iFFT, x-iFFT, state update       -> partial <raw iterate>
  all-reduce -> delta (mean-field pin) installed on every rank

The collectives are torch.distributed all_to_all_single / all_reduce (NCCL
over NVLink on GPUs, gloo for the CPU test).  Kernels are the same fused
sweeps as the single-GPU path (fftc_slab_* in include/fftcond_b200.h).
The per-rank work is a `backend` object so the decomposition logic can be
tested on CPU with a numpy backend (tests/slab_numpy.py).
"""

from __future__ import annotations

import ctypes as C

import numpy as np

from . import native
from .exceptions import BackendError
from .solver import SolverConfig, TerminationStatus, _params

PH_INIT, PH_ROWS_FWD, PH_MID, PH_ROWS_INV = 0, 1, 2, 3


def _dist(group):
    import torch.distributed as dist

    if dist.is_available() and dist.is_initialized():
        return dist, dist.get_rank(group), dist.get_world_size(group)
    return None, 0, 1


def slab_bounds(n: int, rank: int, world: int) -> tuple[int, int]:
    if n % world:
        raise ValueError(f"axis of length {n} does not split over {world} ranks")
    m = n // world
    return rank * m, m


class _DeviceArray:
    """A library (CUDA IPC-capable) allocation seen by torch through
    __cuda_array_interface__ (zero copy)."""

    def __init__(self, ptr: int, shape):
        self.__cuda_array_interface__ = {"shape": tuple(shape), "typestr": "<c16", "data": (ptr, False),
                                         "version": 3, "strides": None}


class GpuSlab:
    """Per-rank device state behind fftc_slab_* (one rank per GPU).

    shared=True allocates the slab work buffers through fftc_ipc_alloc, so
    ranks in other processes can map them (fused transposes)."""

    def __init__(self, chi_local: np.ndarray, n_global, z0, nzl, y0, nyl, cfg: SolverConfig, shared: bool = False):
        import torch

        nz, ny, nx = n_global
        self.torch = torch
        self.L = native.lib()
        self.em_type = cfg.scheme.accelerated
        self._owned, self._opened = [], []
        self.chi = torch.from_numpy(np.ascontiguousarray(chi_local).astype(np.uint8)).cuda()
        shape_z, shape_y = (3, nzl, ny, nx), (3, nyl, nz, nx)
        alloc = self._alloc_shared if shared else (
            lambda shape: torch.empty(shape, dtype=torch.complex128, device="cuda"))
        self.Az = alloc(shape_z)
        self.Ay = alloc(shape_y)
        self.Bz = alloc(shape_z) if self.em_type else self.Az
        self.By = alloc(shape_y) if self.em_type else self.Ay
        d = native.SlabDesc()
        d.d = 3
        d.n[0], d.n[1], d.n[2] = nx, ny, nz
        d.z0, d.nzl, d.y0, d.nyl = z0, nzl, y0, nyl
        d.chi = self.chi.data_ptr()
        self.params = _params(cfg, 3)
        self.h = C.c_void_p()
        rc = self.L.fftc_slab_create(C.byref(d), C.byref(self.params), self.Az.data_ptr(), self.Bz.data_ptr(),
                                     self.Ay.data_ptr(), self.By.data_ptr(), C.byref(self.h), self._stream())
        if rc:
            raise BackendError(f"fftc_slab_create failed ({rc}): {native.last_error()}")

    def _stream(self):
        return self.torch.cuda.current_stream().cuda_stream

    def _call(self, fn, *args):
        rc = fn(self.h, *args, self._stream())
        if rc:
            raise BackendError(f"{fn.__name__} failed ({rc}): {native.last_error()}")

    def phase(self, ph: int) -> np.ndarray:
        out = np.zeros(8)
        self._call(self.L.fftc_slab_phase, ph, out.ctypes.data)
        return out

    def set_delta(self, delta6: np.ndarray):
        d = np.ascontiguousarray(delta6, dtype=np.float64)
        self._call(self.L.fftc_slab_set_delta, d.ctypes.data)

    def monitor(self, totals8: np.ndarray) -> np.ndarray:
        t = np.ascontiguousarray(totals8, dtype=np.float64)
        rec = np.zeros(7)
        self._call(self.L.fftc_slab_monitor, t.ctypes.data, rec.ctypes.data)
        return rec

    def set_peers(self, world: int, ay, by, az) -> bool:
        """Fused transposes: device pointers of every rank's A_y, B_y, A_z
        (rank order, peer-accessible).  False when the grid cannot use them."""
        arr = C.c_void_p * world
        rc = self.L.fftc_slab_set_peers(self.h, world, arr(*ay), arr(*by) if self.em_type else None, arr(*az),
                                        self._stream())
        if rc == 3:
            return False
        if rc:
            raise BackendError(f"fftc_slab_set_peers failed ({rc}): {native.last_error()}")
        return True

    def local_pointers(self):
        return self.Ay.data_ptr(), self.By.data_ptr(), self.Az.data_ptr()

    def _alloc_shared(self, shape):
        ptr = C.c_void_p()
        nbytes = int(np.prod(shape)) * 16
        rc = self.L.fftc_ipc_alloc(nbytes, C.byref(ptr))
        if rc:
            raise BackendError(f"fftc_ipc_alloc failed ({rc}): {native.last_error()}")
        self._owned.append(ptr.value)
        return self.torch.as_tensor(_DeviceArray(ptr.value, shape), device="cuda")

    def ipc_handles(self):
        """64-byte CUDA IPC handles of (A_y, B_y, A_z), or None without shared buffers."""
        if not self._owned:
            return None
        out = []
        for t in (self.Ay, self.By, self.Az):
            h = C.create_string_buffer(64)
            rc = self.L.fftc_ipc_handle(t.data_ptr(), h)
            if rc:
                raise BackendError(f"fftc_ipc_handle failed ({rc}): {native.last_error()}")
            out.append(h.raw)
        return out

    def open_peer(self, handles):
        """Map another process's (A_y, B_y, A_z); returns their device pointers."""
        ptrs, seen = [], {}
        for h in handles:
            if h not in seen:  # B_y is A_y for basic-type schemes
                p = C.c_void_p()
                rc = self.L.fftc_ipc_open(h, C.byref(p))
                if rc:
                    raise BackendError(f"fftc_ipc_open failed ({rc}): {native.last_error()}")
                self._opened.append(p.value)
                seen[h] = p.value
            ptrs.append(seen[h])
        return tuple(ptrs)

    def finalize(self) -> np.ndarray:
        m = np.zeros(12)
        self._call(self.L.fftc_slab_finalize, None, None, None, m.ctypes.data)
        return m

    def close(self):
        if self.h:
            self.L.fftc_slab_destroy(self.h)
            self.h = C.c_void_p()
        self.torch.cuda.synchronize()
        for p in self._opened:
            self.L.fftc_ipc_close(p)
        self._opened = []
        self.Az = self.Ay = self.Bz = self.By = None
        for p in self._owned:
            self.L.fftc_ipc_free(p)
        self._owned = []


def _transpose_z_to_y(Az, Ay, world, group, dist):
    """(c, z_l, y, x) z-slabs -> (c, y_l, z, x) y-slabs through one all-to-all."""
    import torch

    d, nzl, ny, nx = Az.shape
    nyl = ny // world
    send = Az.view(d, nzl, world, nyl, nx).permute(2, 0, 1, 3, 4).contiguous()
    if world == 1:
        recv = send
    else:
        recv = torch.empty_like(send)
        dist.all_to_all_single(torch.view_as_real(recv), torch.view_as_real(send), group=group)
    # recv[q] = rank q's z-planes of my y-planes: (q, c, z_l, y_l, x)
    Ay.view(d, nyl, world, nzl, nx).copy_(recv.permute(1, 3, 0, 2, 4))


def _transpose_y_to_z(Ay, Az, world, group, dist):
    import torch

    d, nyl, nz, nx = Ay.shape
    nzl = nz // world
    send = Ay.view(d, nyl, world, nzl, nx).permute(2, 0, 3, 1, 4).contiguous()  # (q, c, z_l(q), y_l, x)
    if world == 1:
        recv = send
    else:
        recv = torch.empty_like(send)
        dist.all_to_all_single(torch.view_as_real(recv), torch.view_as_real(send), group=group)
    # recv[q] = rank q's y-planes of my z-planes: (q, c, z_l, y_l, x)
    Az.view(d, nzl, world, nyl, nx).copy_(recv.permute(1, 2, 0, 3, 4))


def _allreduce(vec: np.ndarray, dist, group, device) -> np.ndarray:
    if dist is None:
        return vec
    import torch

    if hasattr(dist, "get_backend") and dist.get_backend(group) == "gloo":
        device = "cpu"  # gloo reduces host tensors
    t = torch.from_numpy(np.ascontiguousarray(vec, dtype=np.float64)).to(device)
    dist.all_reduce(t, group=group)
    return t.cpu().numpy()


_STATUS = {0: TerminationStatus.CONVERGED, 1: TerminationStatus.MAX_ITERS, 2: TerminationStatus.DIVERGED}


def _gather_pointers(be, dist, group, comm, world, rank):
    """Every rank's (A_y, B_y, A_z) device pointers, peer-accessible, or None.

    Threads of one process (test communicators) gather the pointers directly.
    Processes exchange CUDA IPC handles of their library-allocated slab
    buffers and map the peers' (NVLink peer mappings between GPUs)."""
    if comm is not None and hasattr(comm, "all_gather_object"):
        return comm.all_gather_object(be.local_pointers())
    if dist is None or not hasattr(be, "ipc_handles"):
        return None
    allh = [None] * world
    dist.all_gather_object(allh, be.ipc_handles(), group=group)
    if any(h is None for h in allh):
        return None
    return [be.local_pointers() if q == rank else be.open_peer(h) for q, h in enumerate(allh)]


def _all_true(flag: bool, dist, group, device, comm) -> bool:
    if dist is None:
        return flag
    v = _allreduce(np.array([0.0 if flag else 1.0]), dist, group, device)
    return float(v[0]) == 0.0


def _barrier(dist, group, comm):
    if comm is not None and hasattr(comm, "barrier"):
        comm.barrier()
    elif dist is not None:
        dist.barrier(group=group)


def solve_slab(chi_global: np.ndarray, cfg: SolverConfig, *, group=None, backend_factory=None, comm=None,
               fused: bool = True) -> dict:
    """Slab-decomposed solve of a 3-D cell; every rank returns the same record dict.

    `comm` (tests): an object with `rank`, `world`, `all_to_all_single(out,
    inp, group=None)`, `all_reduce(t, group=None)` (and optionally
    `all_gather_object`, `barrier`) standing in for torch.distributed.
    `fused`: use the transposes fused into the column passes (peer stores)
    when every rank can; otherwise the all-to-all transposes."""
    if comm is not None:
        dist, rank, world = comm, comm.rank, comm.world
    else:
        dist, rank, world = _dist(group)
    chi_global = np.asarray(chi_global, dtype=bool)
    if chi_global.ndim != 3:
        raise ValueError("slab decomposition is for 3-D cells")
    nz, ny, nx = chi_global.shape
    z0, nzl = slab_bounds(nz, rank, world)
    y0, nyl = slab_bounds(ny, rank, world)
    factory = backend_factory or GpuSlab
    if factory is GpuSlab:  # processes share their slab buffers for the fused transposes
        be = GpuSlab(chi_global[z0:z0 + nzl], (nz, ny, nx), z0, nzl, y0, nyl, cfg,
                     shared=fused and world > 1 and comm is None)
    else:
        be = factory(chi_global[z0:z0 + nzl], (nz, ny, nx), z0, nzl, y0, nyl, cfg)
    device = "cuda" if factory is GpuSlab else "cpu"
    if world == 1 and comm is None:
        dist = None
    e0 = cfg.e0_vector(3)
    e0v = np.array([[z.real, z.imag] for z in e0]).ravel()
    try:
        def global_delta(parts):
            tot = _allreduce(parts[:6], dist, group, device)
            return tot - (world - 1) * e0v

        use_fused = False
        if fused and (world > 1 or comm is not None) and hasattr(be, "set_peers"):
            ptrs = _gather_pointers(be, dist, group, comm, world, rank)
            ok = ptrs is not None and be.set_peers(world, [p[0] for p in ptrs], [p[1] for p in ptrs],
                                                    [p[2] for p in ptrs])
            use_fused = _all_true(ok, dist, group, device, comm)
            some_fused = not _all_true(not ok, dist, group, device, comm)
            if some_fused and not use_fused:
                # set_peers cannot be undone on the ranks where it succeeded: every
                # rank raises (the decision is collective), none waits in a collective
                raise BackendError("ranks disagree on fused transposes")
        be.set_delta(global_delta(be.phase(PH_INIT)))
        history, rec = [], None
        for k in range(1, cfg.max_iters + 1):
            fwd = be.phase(PH_ROWS_FWD)
            if use_fused:
                _barrier(dist, group, comm)  # every y-slab filled by the peers' y passes
            else:
                _transpose_z_to_y(be.Az, be.Ay, world, group, dist)
                if be.em_type:
                    _transpose_z_to_y(be.Bz, be.By, world, group, dist)
            mid = be.phase(PH_MID)
            if not use_fused:
                _transpose_y_to_z(be.Ay, be.Az, world, group, dist)
            tot = _allreduce(np.concatenate([fwd[:7], mid[:1]]), dist, group, device)
            rec = be.monitor(tot)
            if int(rec[3]) > len(history):
                history.append((complex(rec[4], rec[5]), float(rec[6])))
            if rec[0]:
                break
            be.set_delta(global_delta(be.phase(PH_ROWS_INV)))
        means = _allreduce(be.finalize(), dist, group, device)
        if use_fused:
            _barrier(dist, group, comm)  # no peer still stores into this rank's buffers when they are freed
        sstar = history[-1][0] if history else complex(rec[4], rec[5])
        return dict(status=_STATUS[int(rec[1])], degenerate_flux=bool(rec[2]), iterations=len(history),
                    sigma_star=sstar, history=history, fused=use_fused,
                    mean_E=np.array([complex(means[2 * c], means[2 * c + 1]) for c in range(3)]),
                    mean_J=np.array([complex(means[6 + 2 * c], means[6 + 2 * c + 1]) for c in range(3)]),
                    world=world)
    finally:
        close = getattr(be, "close", None)
        if close:
            close()
