"""ctypes binding of libkmf_b200.so (the C ABI declared in include/kmf_b200.h).

The shared library is built in-tree (``make -C paper_2108_07031_b200/csrc`` or
``__graft_entry__.build()``).  There is no fallback: if the library is
missing, or no CUDA device is visible, every device operation raises.
"""

from __future__ import annotations

import ctypes as C
import os
from pathlib import Path

import numpy as np

LIB_PATH = Path(__file__).resolve().parent / "libkmf_b200.so"

KMF_OK, KMF_EPOSITIVITY, KMF_EINVAL, KMF_ECUDA, KMF_ENCCL, KMF_EPEER = 0, 1, 2, 3, 4, 5
KMF_PEER_HANDLE_BYTES = 128
BENCH_KERNELS = 3  # KMF_BENCH_KERNELS: interior flux, first order, sweeps
DIAG_LAST_RUN = 2  # kmf_diag_* `which`: the final gradients of the last run

(CTX_NONE, CTX_INITIAL, CTX_FLUX_XP, CTX_FLUX_XM, CTX_FLUX_YP, CTX_FLUX_YM,
 CTX_WALL_TANGENT, CTX_WALL_NORMAL, CTX_OUTER_TANGENT, CTX_OUTER_NORMAL,
 CTX_C2P_DENSITY, CTX_C2P_PRESSURE, CTX_Q2P, CTX_P2Q) = range(14)

_dp = C.POINTER(C.c_double)
_i64p = C.POINTER(C.c_int64)
_u8p = C.POINTER(C.c_uint8)


class Stencil(C.Structure):
    _fields_ = [
        ("n_owners", C.c_int64), ("n_edges", C.c_int64),
        ("ptr", _i64p), ("idx", _i64p),
        ("dx", _dp), ("dy", _dp),
        ("sxx", _dp), ("sxy", _dp), ("syy", _dp), ("det", _dp),
    ]


class Frame(C.Structure):
    _fields_ = [
        ("b", C.c_int64), ("points", _i64p),
        ("tx", _dp), ("ty", _dp), ("nx", _dp), ("ny", _dp),
        ("tplus", Stencil), ("tminus", Stencil), ("normal", Stencil),
    ]


class Geometry(C.Structure):
    _fields_ = [
        ("n", C.c_int64), ("x", _dp), ("y", _dp), ("flag", _i64p), ("d_min", _dp),
        ("full", Stencil),
        ("split_sxx", _dp * 4), ("split_sxy", _dp * 4), ("split_syy", _dp * 4),
        ("det_safe", _dp * 4),
        ("has_wall", C.c_int), ("has_outer", C.c_int),
        ("wall", Frame), ("outer", Frame),
        ("perm", _i64p),
    ]


class Params(C.Structure):
    _fields_ = [
        ("gamma", C.c_double), ("cfl", C.c_double), ("fs", C.c_double * 4),
        ("n_inner", C.c_int), ("mode", C.c_int), ("convergence_tol", C.c_double),
        ("instrument", C.c_int), ("timing_skip", C.c_int),
    ]


class ErrorInfo(C.Structure):
    _fields_ = [
        ("code", C.c_int), ("iteration", C.c_int), ("stage", C.c_int), ("context", C.c_int),
        ("count", C.c_int64), ("n_indices", C.c_int64), ("message", C.c_char * 256),
    ]


_lib = None


def lib():
    """Load the CUDA library (once).  Raises if it is missing."""
    global _lib
    if _lib is not None:
        return _lib
    if not LIB_PATH.exists():
        raise RuntimeError(
            f"{LIB_PATH} is missing: build it with `make -C paper_2108_07031_b200/csrc` "
            "or `python -c 'import __graft_entry__; __graft_entry__.build()'` "
            "(there is no CPU fallback)"
        )
    L = C.CDLL(str(LIB_PATH))
    vp = C.c_void_p
    sig = {
        "kmf_abi_version": (C.c_int, []),
        "kmf_device_count": (C.c_int, []),
        "kmf_strerror": (C.c_char_p, []),
        "kmf_create": (C.c_int, [C.POINTER(vp), C.POINTER(Geometry), C.c_int]),
        "kmf_destroy": (None, [vp]),
        "kmf_set_state": (C.c_int, [vp, _dp]),
        "kmf_run": (C.c_int, [vp, C.POINTER(Params), C.c_int, _dp, C.POINTER(C.c_int), C.POINTER(C.c_int)]),
        "kmf_prepare": (C.c_int, [vp, C.POINTER(Params)]),
        "kmf_run_cases": (C.c_int, [vp, C.POINTER(Params), C.c_int, C.c_int, C.POINTER(C.c_void_p),
                                    C.POINTER(C.c_void_p), C.POINTER(C.c_void_p), _dp, C.POINTER(C.c_int),
                                    C.POINTER(C.c_int), C.POINTER(C.c_int)]),
        "kmf_get_state": (C.c_int, [vp, _dp, _dp]),
        "kmf_stage_seconds": (C.c_int, [vp, _dp]),
        "kmf_last_error": (C.c_int, [vp, C.POINTER(ErrorInfo)]),
        "kmf_last_indices": (C.c_int, [vp, _i64p, C.c_int64]),
        "kmf_diag_flux": (C.c_int, [vp, C.c_int, _u8p]),
        "kmf_diag_frame": (C.c_int, [vp, C.c_int, C.c_int, _u8p]),
        "kmf_diag_stage_state": (C.c_int, [vp, C.c_int, _dp]),
        "kmf_op_timestep": (C.c_int, [vp, _dp, C.c_double, C.c_double, _dp]),
        "kmf_op_first_order": (C.c_int, [vp, _dp, _dp, _dp]),
        "kmf_op_q_derivatives": (C.c_int, [vp, _dp, C.c_int, _dp, _dp, _dp, _dp, _dp]),
        "kmf_op_flux_residual": (C.c_int, [vp, _dp, _dp, _dp, C.c_int, C.c_double, _dp]),
        "kmf_op_boundary": (C.c_int, [vp, _dp, _dp, _dp, _dp, C.c_double, _dp]),
        "kmf_op_primitives_to_q": (C.c_int, [C.c_int64, _dp, C.c_double, _dp, _u8p]),
        "kmf_op_q_to_primitives": (C.c_int, [C.c_int64, _dp, C.c_double, _dp, _u8p]),
        "kmf_op_primitives_to_conserved": (C.c_int, [C.c_int64, _dp, C.c_double, _dp, _u8p]),
        "kmf_op_conserved_to_primitives": (C.c_int, [C.c_int64, _dp, C.c_double, _dp, _u8p]),
        "kmf_op_split_flux": (C.c_int, [C.c_int64, _dp, C.c_int, C.c_int, C.c_double, _dp]),
        "kmf_op_full_flux": (C.c_int, [C.c_int64, _dp, C.c_int, C.c_double, _dp]),
        "kmf_op_state_update": (C.c_int, [C.c_int64, _dp, _dp, C.c_int, _dp, _dp, _dp]),
        "kmf_op_residue": (C.c_int, [C.c_int64, _dp, _dp, _dp]),
        "kmf_bench_steps": (C.c_int, [vp, C.POINTER(Params), C.c_int, C.c_int64, _dp, _dp, C.POINTER(C.c_int)]),
        "kmf_fp64_peak": (C.c_int, [_dp]),
        "kmf_fastmath_probe": (C.c_int, [C.c_int64, _dp, C.c_int, _dp]),
        "kmf_probe_edge_state": (C.c_int, [C.c_int64, _dp, C.c_double, _dp, _dp]),
        "kmf_set_partition": (C.c_int, [vp, C.c_int64, C.c_int64, C.c_int, C.c_int, C.c_int, _i64p, _i64p, C.c_int,
                                        C.POINTER(C.c_int), _i64p, _i64p, _i64p, _i64p]),
        "kmf_nccl_get_unique_id": (C.c_int, [C.c_void_p]),
        "kmf_nccl_init": (C.c_int, [vp, C.c_void_p, C.c_int, C.c_int]),
        "kmf_run_group": (C.c_int, [C.POINTER(vp), C.c_int, C.POINTER(Params), C.c_int, _dp, C.POINTER(C.c_int),
                                    C.POINTER(C.c_int)]),
        "kmf_peer_handle": (C.c_int, [vp, C.c_void_p]),
        "kmf_peer_open": (C.c_int, [vp, C.c_void_p, _i64p, _i64p]),
        "kmf_peer_link": (C.c_int, [C.POINTER(vp), C.c_int]),
        "kmf_peer_counters": (C.c_int, [vp, C.POINTER(C.c_uint64)]),
        "kmf_run_linked": (C.c_int, [C.POINTER(vp), C.c_int, C.POINTER(Params), C.c_int, _dp, C.POINTER(C.c_int),
                                     C.POINTER(C.c_int)]),
        "kmf_host_alloc": (C.c_void_p, [C.c_int64]),
        "kmf_host_free": (None, [C.c_void_p]),
    }
    for name, (res, args) in sig.items():
        fn = getattr(L, name)
        fn.restype = res
        fn.argtypes = args
    _lib = L
    return L


EXPORTED = (
    "kmf_abi_version", "kmf_device_count", "kmf_strerror", "kmf_create", "kmf_destroy",
    "kmf_set_state", "kmf_run", "kmf_prepare", "kmf_get_state", "kmf_stage_seconds", "kmf_last_error",
    "kmf_last_indices", "kmf_diag_flux", "kmf_diag_frame", "kmf_diag_stage_state",
    "kmf_op_timestep", "kmf_op_first_order", "kmf_op_q_derivatives", "kmf_op_flux_residual",
    "kmf_op_boundary", "kmf_op_primitives_to_q", "kmf_op_q_to_primitives",
    "kmf_op_primitives_to_conserved", "kmf_op_conserved_to_primitives", "kmf_op_split_flux",
    "kmf_op_full_flux", "kmf_op_state_update", "kmf_op_residue", "kmf_bench_steps", "kmf_fp64_peak", "kmf_fastmath_probe",
    "kmf_probe_edge_state",
    "kmf_host_alloc", "kmf_host_free", "kmf_set_partition", "kmf_nccl_get_unique_id", "kmf_nccl_init",
    "kmf_run_group", "kmf_run_cases", "kmf_peer_handle", "kmf_peer_open", "kmf_peer_link", "kmf_run_linked",
    "kmf_peer_counters",
)


def pinned(shape, dtype=np.float64):
    """numpy view of pinned (page-locked) host memory; freed with the array."""
    count = int(np.prod(shape))
    nbytes = count * np.dtype(dtype).itemsize
    L = lib()
    ptr = L.kmf_host_alloc(nbytes)
    if not ptr:
        raise DeviceError("kmf_host_alloc failed")
    buf = (C.c_char * nbytes).from_address(ptr)
    arr = np.frombuffer(buf, dtype=dtype, count=count).reshape(shape)
    import weakref

    weakref.finalize(buf, L.kmf_host_free, ptr)  # arr.base keeps buf alive
    return arr


class DeviceError(RuntimeError):
    """A CUDA / ABI failure (not a physics error)."""


def check(rc: int, what: str):
    if rc == KMF_OK:
        return
    msg = lib().kmf_strerror().decode(errors="replace")
    if rc == KMF_EINVAL:
        raise ValueError(msg or f"{what}: invalid argument")
    raise DeviceError(f"{what} failed (code {rc}): {msg}")


def require_device():
    n = lib().kmf_device_count()
    if n <= 0:
        raise DeviceError("no CUDA device visible: the B200 path has no CPU fallback")
    return n


def dptr(a: np.ndarray):
    return a.ctypes.data_as(_dp)


def i64ptr(a: np.ndarray):
    return a.ctypes.data_as(_i64p)


def u8ptr(a: np.ndarray):
    return a.ctypes.data_as(_u8p)


def f64(a) -> np.ndarray:
    return np.ascontiguousarray(np.asarray(a, dtype=np.float64))


def i64(a) -> np.ndarray:
    return np.ascontiguousarray(np.asarray(a, dtype=np.int64))


def device_index() -> int:
    return int(os.environ.get("KMF_DEVICE", "0"))
