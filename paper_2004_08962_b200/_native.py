"""ctypes binding of libhicu_b200.so (include/hicu_b200.h).

There is no CPU fallback: importing the operators works on any machine, but
every call that computes goes through this library and raises
:class:`NativeError` when the library is missing or no CUDA device exists.
"""

from __future__ import annotations

import ctypes
import os
from ctypes import POINTER, c_char, c_double, c_int, c_int32, c_int64, c_size_t, c_uint32, c_void_p

from .errors import STATUS_TO_EXC, NativeError

LIB_PATH = os.path.join(os.path.dirname(os.path.abspath(__file__)), "libhicu_b200.so")
MAX_NDIM = 8

REC_OBJ, REC_NUM, REC_DEN, REC_ETA, REC_OBJ_AFTER, REC_GNORM2, REC_DEGENERATE, REC_TIME = range(8)
REC_SLOTS = 8
GEOM_COIL_SEPARABLE = 1
GEOM_FORCE_SIMT_GRAM = 2
GEOM_FORCE_SIMT_CONV = 4
GEOM_FORCE_DENSE_GRAM = 8
GEOM_FORCE_LAG_GRAM = 16
GEOM_FORCE_FFMA_LAG = 32
GRAM_PATHS = {0: "simt", 1: "tcgen05", 2: "lag"}
PROF_KINDS = ("gram", "nystrom", "householder", "conv_fwd", "scatter", "conv_els", "update")


class HicuGeom(ctypes.Structure):
    _fields_ = [
        ("ndim", c_int32),
        ("n", c_int32),
        ("dims", c_int64 * MAX_NDIM),
        ("roff", c_int64 * MAX_NDIM),
        ("rext", c_int64 * MAX_NDIM),
        ("circular", c_uint32),
        ("flags", c_int32),
        ("pos", c_void_p),
        ("koff", c_void_p),
        ("kext", c_int64 * MAX_NDIM),
    ]


class HicuStageArgs(ctypes.Structure):
    _fields_ = [
        ("geom", HicuGeom),
        ("r", c_int32), ("ell", c_int32), ("p", c_int32), ("gsteps", c_int32), ("iters", c_int32),
        ("dc_mode", c_int32),
        ("lam", c_double),
        ("householder_tol", c_double),
        ("N", c_int64),
        ("y", c_void_p), ("mask", c_void_p), ("x0", c_void_p), ("omega", c_void_p), ("pbig", c_void_p),
        ("inject_v", c_void_p),
        ("G", c_void_p), ("gram_ws", c_void_p), ("gram_ws_bytes", c_size_t),
        ("nys_ws", c_void_p), ("nys_ws_bytes", c_size_t),
        ("V", c_void_p), ("refl", c_void_p), ("tau", c_void_p), ("flags", c_void_p), ("status", c_void_p),
        ("B", c_void_p), ("qt32", c_void_p), ("u", c_void_p), ("g", c_void_p),
        ("obj_parts", c_void_p), ("dc_parts", c_void_p), ("els_parts", c_void_p),
        ("rec", c_void_p),
        ("ref", c_void_p), ("ser_parts", c_void_p), ("ser_stride", c_int32),
        ("prof", c_void_p),
    ]


class HicuP2P(ctypes.Structure):
    _fields_ = [("peer", c_int32), ("kind", c_int32), ("buf", c_void_p), ("bytes", c_int64)]


P2P_SEND, P2P_RECV = 0, 1

_GP = POINTER(HicuGeom)
_SIGS = {
    "hicu_abi_version": (c_int, []),
    "hicu_last_error": (ctypes.c_char_p, []),
    "hicu_status_string": (ctypes.c_char_p, [c_int]),
    "hicu_device_sm_count": (c_int, [POINTER(c_int)]),
    "hicu_conv_nparts": (c_int, [_GP]),
    "hicu_scatter_nparts": (c_int, [_GP]),
    "hicu_conv_fwd": (c_int, [_GP, c_void_p, c_void_p, c_int, c_void_p, c_void_p, c_void_p]),
    "hicu_conv_els": (c_int, [_GP, c_void_p, c_void_p, c_int, c_void_p, c_void_p, c_void_p]),
    "hicu_conv_adj": (c_int, [_GP, c_void_p, c_void_p, c_int, c_void_p, c_void_p]),
    "hicu_scatter_dc": (c_int, [_GP, c_void_p, c_int, c_void_p, c_void_p, c_void_p, c_void_p, c_int, c_double,
                                c_void_p, c_void_p, c_void_p]),
    "hicu_step_update": (c_int, [c_int64, c_void_p, c_void_p, c_void_p, c_int, c_void_p, c_int, c_void_p, c_int,
                                 c_int, c_double, c_void_p, c_void_p]),
    "hicu_ser_nparts": (c_int, [c_int64]),
    "hicu_step_reduce": (c_int, [c_void_p, c_int, c_void_p, c_int, c_void_p, c_int, c_void_p, c_void_p]),
    "hicu_step_apply": (c_int, [c_int64, c_void_p, c_void_p, c_void_p, c_int, c_double, c_void_p, c_void_p]),
    "hicu_dc_nparts": (c_int, [c_int64]),
    "hicu_dc_apply": (c_int, [c_int64, c_void_p, c_void_p, c_void_p, c_void_p, c_int, c_double, c_void_p, c_void_p]),
    "hicu_ser_parts": (c_int, [c_int64, c_void_p, c_void_p, c_void_p, POINTER(c_int), c_void_p]),
    "hicu_soft_terms": (c_int, [c_int64, c_void_p, c_void_p, c_void_p, c_void_p, c_void_p, POINTER(c_int),
                                c_void_p]),
    "hicu_gram_workspace": (c_size_t, [_GP]),
    "hicu_gram_uses_tensor_cores": (c_int, [_GP]),
    "hicu_gram_lag_uses_tensor_cores": (c_int, [_GP]),
    "hicu_gram_path": (c_int, [_GP]),
    "hicu_eigh_top_workspace": (c_size_t, [c_int, c_int]),
    "hicu_eigh_top": (c_int, [c_int, c_int, c_void_p, c_void_p, c_void_p, c_void_p, c_size_t, c_void_p]),
    "hicu_comm_available": (c_int, []),
    "hicu_comm_unique_id": (c_int, [c_void_p]),
    "hicu_comm_init": (c_int, [c_int, c_int, c_void_p, POINTER(c_void_p)]),
    "hicu_comm_destroy": (c_int, [c_void_p]),
    "hicu_allreduce": (c_int, [c_void_p, c_void_p, c_int64, c_void_p]),
    "hicu_halo_exchange": (c_int, [c_void_p, c_int, c_void_p, c_void_p]),
    "hicu_gram_flops": (c_double, [_GP]),
    "hicu_conv_uses_tensor_cores": (c_int, [_GP, c_int]),
    "hicu_gram": (c_int, [_GP, c_void_p, c_void_p, c_void_p, c_size_t, c_void_p]),
    "hicu_zgemm": (c_int, [c_char, c_char, c_int, c_int, c_int, c_void_p, c_int, c_void_p, c_int, c_void_p, c_int,
                           c_void_p]),
    "hicu_nystrom_workspace": (c_size_t, [c_int, c_int]),
    "hicu_nystrom": (c_int, [c_int, c_int, c_int, c_void_p, c_void_p, c_void_p, c_void_p, c_size_t, c_void_p,
                             c_void_p]),
    "hicu_complement_jl": (c_int, [c_int, c_int, c_int, c_int, c_void_p, c_void_p, c_void_p, c_void_p, c_void_p,
                                   c_void_p, c_void_p, c_double, c_void_p, c_void_p]),
    "hicu_householder": (c_int, [c_int, c_int, c_void_p, c_double, c_void_p, c_void_p, c_void_p, c_void_p,
                                 c_void_p]),
    "hicu_apply_reflectors": (c_int, [c_int, c_int, c_void_p, c_void_p, c_void_p, c_int, c_void_p, c_void_p,
                                      c_void_p, c_int, c_void_p]),
    "hicu_nullspace_jl_supported": (c_int, [c_int, c_int]),
    "hicu_nullspace_jl_workspace": (c_size_t, [c_int, c_int]),
    "hicu_nullspace_jl_ws": (c_int, [c_int, c_int, c_void_p, c_int, c_void_p, c_void_p, c_void_p, c_int, c_void_p,
                                     c_void_p, c_size_t, c_void_p]),
    "hicu_nullspace_jl": (c_int, [c_int, c_int, c_void_p, c_int, c_void_p, c_void_p, c_void_p, c_int, c_void_p,
                                  c_void_p]),
    "hicu_run_stage": (c_int, [POINTER(HicuStageArgs), c_void_p]),
    "hicu_timestamp": (c_int, [c_void_p, c_void_p]),
    "hicu_prof_create": (c_int, [c_int, POINTER(c_void_p)]),
    "hicu_prof_destroy": (c_int, [c_void_p]),
    "hicu_prof_reset": (c_int, [c_void_p]),
    "hicu_prof_summary": (c_int, [c_void_p, POINTER(c_double), POINTER(c_int)]),
    "hicu_launch_count": (ctypes.c_longlong, []),
    "hicu_coil_workspace": (c_size_t, [c_int64, c_int]),
    "hicu_coil_cov": (c_int, [c_int64, c_int, c_void_p, c_void_p, c_void_p, c_void_p, c_size_t, c_void_p]),
    "hicu_coil_basis_workspace": (c_size_t, [c_int]),
    "hicu_coil_basis": (c_int, [c_int, c_int, c_void_p, c_void_p, c_void_p, c_void_p, c_size_t, c_void_p]),
    "hicu_coil_apply": (c_int, [c_int64, c_int, c_int, c_void_p, c_void_p, c_void_p, c_void_p, c_void_p,
                                c_void_p]),
}

EXPORTED = tuple(_SIGS)

_lib = None


def load(path: str = LIB_PATH):
    """Load the shared library (without touching the GPU)."""
    global _lib
    if _lib is not None:
        return _lib
    if not os.path.exists(path):
        raise NativeError(
            f"CUDA extension not built: {path} is missing (run __graft_entry__.build() or "
            "python paper_2004_08962_b200/_build.py)"
        )
    try:
        lib = ctypes.CDLL(path)
    except OSError as e:  # pragma: no cover - depends on the host
        raise NativeError(f"cannot load {path}: {e}") from e
    for name, (res, args) in _SIGS.items():
        fn = getattr(lib, name)
        fn.restype = res
        fn.argtypes = args
    _lib = lib
    return lib


def lib():
    return load()


def check(status: int, what: str = "") -> None:
    if status == 0:
        return
    L = lib()
    msg = L.hicu_last_error().decode(errors="replace")
    exc = STATUS_TO_EXC.get(status, NativeError)
    raise exc(f"{what}: {msg}" if what else msg)


def require_cuda():
    """Return the torch module after checking a CUDA device is present."""
    import torch

    if not torch.cuda.is_available():
        raise NativeError("no CUDA device: the HICU B200 path has no CPU fallback")
    load()
    return torch


def stream_handle(stream=None) -> int:
    import torch

    s = stream if stream is not None else torch.cuda.current_stream()
    return int(s.cuda_stream)


class Profiler:
    """Native CUDA-event profiler (hicu_prof_*): per kernel class totals."""

    def __init__(self, capacity: int = 1 << 16):
        self.h = c_void_p()
        check(lib().hicu_prof_create(capacity, ctypes.byref(self.h)), "prof_create")

    def reset(self):
        lib().hicu_prof_reset(self.h)

    def summary(self) -> dict:
        ms = (c_double * len(PROF_KINDS))()
        cnt = (c_int * len(PROF_KINDS))()
        check(lib().hicu_prof_summary(self.h, ms, cnt), "prof_summary")
        return {k: {"ms": ms[i], "launches": cnt[i]} for i, k in enumerate(PROF_KINDS)}

    def __del__(self):
        try:
            if self.h:
                lib().hicu_prof_destroy(self.h)
        except Exception:
            pass
