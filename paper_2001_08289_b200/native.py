"""ctypes binding of the C ABI declared in ``include/fftcond_b200.h``.

The product path has no CPU fallback: if ``libfftcond_b200.so`` is missing
or does not export the declared symbols, :func:`lib` raises.
"""

from __future__ import annotations

import ctypes as C
import os
import threading

HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.environ.get("FFTC_LIB") or os.path.join(HERE, "libfftcond_b200.so")  # FFTC_LIB: A/B builds

# every symbol declared in include/fftcond_b200.h
FFTC_AUG_CHI, FFTC_AUG_LOCAL_A, FFTC_AUG_INV_SHIFTED = 0, 1, 2
FFTC_RED_SUM, FFTC_RED_DOT, FFTC_RED_NORM2, FFTC_RED_OFF_SUPPORT = 0, 1, 2, 3
FFTC_MASK_NONE, FFTC_MASK_CHI = 0, 1

EXPORTS = (
    "fftc_solve",
    "fftc_solve_host",
    "fftc_supported_length",
    "fftc_fused_length",
    "fftc_last_error",
    "fftc_version",
    "fftc_launch_count",
    "fftc_last_layout",
    "fftc_fft",
    "fftc_gamma1",
    "fftc_aug_apply",
    "fftc_apply_sigma",
    "fftc_reduce",
    "fftc_slab_set_peers",
    "fftc_ipc_alloc",
    "fftc_ipc_free",
    "fftc_ipc_handle",
    "fftc_ipc_open",
    "fftc_ipc_close",
    "fftc_profile",
    "fftc_kernel_stats",
    "fftc_solve_batch",
    "fftc_slab_create",
    "fftc_slab_phase",
    "fftc_slab_set_delta",
    "fftc_slab_monitor",
    "fftc_slab_finalize",
    "fftc_slab_destroy",
)

FFTC_CONVERGED, FFTC_MAX_ITERS, FFTC_DIVERGED = 0, 1, 2


class Problem(C.Structure):
    _fields_ = [("d", C.c_int32), ("reserved", C.c_int32), ("n", C.c_int64 * 3),
                ("chi", C.c_void_p)]


class Params(C.Structure):
    _fields_ = [("scheme", C.c_int32), ("reserved", C.c_int32),
                ("sigma1", C.c_double * 2), ("sigma0", C.c_double * 2), ("t", C.c_double * 2),
                ("p1", C.c_double * 2), ("p2", C.c_double * 2), ("p3", C.c_double * 2),
                ("e0", (C.c_double * 2) * 3), ("tol", C.c_double), ("max_iters", C.c_int64),
                ("gamma1_scale", C.c_double)]


class Result(C.Structure):
    _fields_ = [("status", C.c_int32), ("degenerate_flux", C.c_int32), ("iterations", C.c_int64),
                ("sigma_star", C.c_double * 2), ("mean_E", (C.c_double * 2) * 3),
                ("mean_J", (C.c_double * 2) * 3), ("kernel_launches", C.c_int64),
                ("device_ms", C.c_double)]


class SlabDesc(C.Structure):
    _fields_ = [("d", C.c_int32), ("reserved", C.c_int32), ("n", C.c_int64 * 3), ("z0", C.c_int64),
                ("nzl", C.c_int64), ("y0", C.c_int64), ("nyl", C.c_int64), ("chi", C.c_void_p)]


class KStat(C.Structure):
    _fields_ = [("name", C.c_char * 32), ("launches", C.c_int64), ("total_ms", C.c_double)]


_lock = threading.Lock()
_lib = None


def lib():
    """Load the CUDA library once; raise loudly if it is absent."""
    global _lib
    with _lock:
        if _lib is not None:
            return _lib
        if not os.path.exists(LIB_PATH):
            raise ImportError(
                f"{LIB_PATH} not found: build it with `python -m paper_2001_08289_b200.build_ext` "
                "(there is no CPU fallback)")
        L = C.CDLL(LIB_PATH)
        for name in EXPORTS:
            getattr(L, name)  # AttributeError if missing
        vp, i64 = C.c_void_p, C.c_int64
        L.fftc_solve.argtypes = [C.POINTER(Problem), C.POINTER(Params), vp, i64, vp, vp, vp,
                                 C.POINTER(Result), vp]
        L.fftc_solve.restype = C.c_int
        L.fftc_solve_host.argtypes = [C.POINTER(Problem), C.POINTER(Params), vp, i64, vp, vp, vp,
                                      C.POINTER(Result)]
        L.fftc_solve_host.restype = C.c_int
        L.fftc_solve_batch.argtypes = [C.POINTER(Problem), C.POINTER(Params), C.c_int32, vp, i64,
                                       C.POINTER(Result), vp]
        L.fftc_solve_batch.restype = C.c_int
        L.fftc_slab_create.argtypes = [C.POINTER(SlabDesc), C.POINTER(Params), vp, vp, vp, vp,
                                       C.POINTER(C.c_void_p), vp]
        L.fftc_slab_create.restype = C.c_int
        L.fftc_slab_phase.argtypes = [vp, C.c_int32, vp, vp]
        L.fftc_slab_phase.restype = C.c_int
        L.fftc_slab_set_delta.argtypes = [vp, vp, vp]
        L.fftc_slab_set_delta.restype = C.c_int
        L.fftc_slab_monitor.argtypes = [vp, vp, vp, vp]
        L.fftc_slab_monitor.restype = C.c_int
        L.fftc_slab_finalize.argtypes = [vp, vp, vp, vp, vp, vp]
        L.fftc_slab_finalize.restype = C.c_int
        L.fftc_slab_set_peers.argtypes = [vp, C.c_int32, vp, vp, vp, vp]
        L.fftc_slab_set_peers.restype = C.c_int
        L.fftc_ipc_alloc.argtypes = [i64, C.POINTER(C.c_void_p)]
        L.fftc_ipc_alloc.restype = C.c_int
        L.fftc_ipc_free.argtypes = [vp]
        L.fftc_ipc_free.restype = C.c_int
        L.fftc_ipc_handle.argtypes = [vp, vp]
        L.fftc_ipc_handle.restype = C.c_int
        L.fftc_ipc_open.argtypes = [vp, C.POINTER(C.c_void_p)]
        L.fftc_ipc_open.restype = C.c_int
        L.fftc_ipc_close.argtypes = [vp]
        L.fftc_ipc_close.restype = C.c_int
        L.fftc_slab_destroy.argtypes = [vp]
        L.fftc_slab_destroy.restype = None
        L.fftc_fft.argtypes = [C.POINTER(Problem), vp, C.c_int32, C.c_int32, vp]
        L.fftc_fft.restype = C.c_int
        L.fftc_gamma1.argtypes = [C.POINTER(Problem), vp, vp, C.c_double, vp]
        L.fftc_gamma1.restype = C.c_int
        L.fftc_aug_apply.argtypes = [C.POINTER(Problem), C.c_int32, vp, vp, vp, vp, vp, vp, vp, vp]
        L.fftc_aug_apply.restype = C.c_int
        L.fftc_apply_sigma.argtypes = [C.POINTER(Problem), vp, vp, vp, vp]
        L.fftc_apply_sigma.restype = C.c_int
        L.fftc_reduce.argtypes = [C.POINTER(Problem), C.c_int32, C.c_int32, vp, vp, vp, vp]
        L.fftc_reduce.restype = C.c_int
        L.fftc_profile.argtypes = [C.c_int32]
        L.fftc_profile.restype = None
        L.fftc_kernel_stats.argtypes = [C.POINTER(KStat), C.c_int32]
        L.fftc_kernel_stats.restype = C.c_int
        L.fftc_supported_length.argtypes = [i64]
        L.fftc_supported_length.restype = C.c_int
        L.fftc_fused_length.argtypes = [i64]
        L.fftc_fused_length.restype = C.c_int
        L.fftc_last_error.argtypes = []
        L.fftc_last_error.restype = C.c_char_p
        L.fftc_version.restype = C.c_int
        L.fftc_launch_count.restype = C.c_int64
        L.fftc_last_layout.restype = C.c_int32
        _lib = L
        return L


def profile(enable: bool):
    lib().fftc_profile(1 if enable else 0)


def kernel_stats() -> dict:
    """{kind: (launches, total device ms)} since the last profile(True)."""
    buf = (KStat * 16)()
    n = lib().fftc_kernel_stats(buf, 16)
    return {buf[i].name.decode(): (int(buf[i].launches), float(buf[i].total_ms)) for i in range(n)}


def last_layout() -> int:
    """z-block shift of this thread's last solve's work fields (0 = reference layout)."""
    return int(lib().fftc_last_layout())


def last_error() -> str:
    return lib().fftc_last_error().decode(errors="replace")


def cpair(z) -> tuple:
    z = complex(z)
    return (z.real, z.imag)
