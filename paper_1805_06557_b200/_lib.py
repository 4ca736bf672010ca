"""ctypes binding of libswx.so (include/swx.h).

There is deliberately no CPU fallback: importing the compute API on a host
without the built library or without a CUDA device raises
``ConfigurationError`` (north star: "no CPU fallback").
"""

from __future__ import annotations

import ctypes
import os
import threading

from .errors import ConfigurationError, DataError, SolverError, SwerexiError

HERE = os.path.dirname(os.path.abspath(__file__))
# SWX_LIB: an alternative build of the same library (A/B measurements)
LIB_PATH = os.environ.get("SWX_LIB") or os.path.join(HERE, "libswx.so")

SWX_OK, SWX_ERR_CONFIG, SWX_ERR_SOLVER, SWX_ERR_DATA, SWX_ERR_CUDA = range(5)
SWX_GROUP_LG, SWX_GROUP_L = 0, 1
SWX_TEND_LC, SWX_TEND_N = 1, 2

# every symbol include/swx.h declares, with (restype, argtypes)
_P = ctypes.c_void_p
_I = ctypes.c_int
_D = ctypes.c_double
_S = ctypes.c_size_t
_IP = ctypes.POINTER(ctypes.c_int)


class C128(ctypes.Structure):
    _fields_ = [("re", ctypes.c_double), ("im", ctypes.c_double)]


SIGNATURES = {
    "swx_version": (_I, []),
    "swx_last_error": (ctypes.c_char_p, []),
    "swx_solver_create": (_I, [ctypes.POINTER(_P), _I, _I, _D, _D, _D, _D]),
    "swx_solver_destroy": (_I, [_P]),
    "swx_solver_warm": (_I, [_P, _P, _I, _IP, _IP, _P]),
    "swx_rexi_workspace_bytes": (_S, [_P, _I, _I, _I]),
    "swx_rexi_sum": (_I, [_P, _I, _P, _P, _I, _I, _I, _P, _P, _S, _P]),
    "swx_rexi_prepared_bytes": (_S, [_P, _I, _I, _I]),
    "swx_rexi_prepare": (_I, [_P, _I, _P, _I, _I, _P, _S, _P]),
    "swx_rexi_sum_prepared": (_I, [_P, _I, _P, _P, _P, _I, _I, _I, _P, _P, _S, _P]),
    "swx_rexi_sum_prepared_axpy": (_I, [_P, _I, _P, _P, _P, _I, _I, _I, _P, _D, _P, _P, _S, _P]),
    "swx_rexi_sum_prepared_ready": (_I, [_P, _I, _P, _P, _P, _I, _I, _I, _P, _D, _P, _P, _S, _P, _P]),
    "swx_apply": (_I, [_P, C128, _P, _P, _P]),
    "swx_tree_combine": (_I, [_I, _I, _I, _P, _I, _P, _P]),
    "swx_tree_combine_flat": (_I, [_S, _I, _P, _P, _P]),
    "swx_state_axpy": (_I, [_I, _I, _P, _D, _P, _P, _P]),
    "swx_sht_create": (_I, [ctypes.POINTER(_P), _I, _I, _I, _D, _D, _P, _P, _P]),
    "swx_sht_destroy": (_I, [_P]),
    "swx_sht_workspace_bytes": (_S, [_P]),
    "swx_sht_synthesis": (_I, [_P, _I, _P, _P, _P, _S, _P]),
    "swx_sht_analysis": (_I, [_P, _I, _P, _P, _P, _S, _P]),
    "swx_sht_uv": (_I, [_P, _P, _P, _P, _P, _P, _S, _P]),
    "swx_sht_vortdiv": (_I, [_P, _P, _P, _P, _P, _P, _S, _P]),
    "swx_sht_tendency": (_I, [_P, _I, _P, _P, _P, _S, _P]),
    "swx_sht_tendency_sub": (_I, [_P, _I, _P, _P, _P, _P, _S, _P]),
    "swx_sht_set_synth_event": (_I, [_P, _P]),
    "swx_sht_set_done_signal": (_I, [_P, _I, ctypes.POINTER(_P)]),
    "swx_sht_tendency_profile": (_I, [_P, _I, _P, _P, _P, _S, _P, _P]),
    "swx_fp64_fma_probe": (_I, [_P, _I, _I, _P]),
    "swx_l_partition_geometry": (_I, [_I, ctypes.POINTER(_I), ctypes.POINTER(_I)]),
    "swx_host_pack": (_I, [_I, _I, _P, _P]),
    "swx_host_unpack": (_I, [_I, _I, _P, _P]),
    "swx_trace": (_I, [_I, _P, _I]),
    "swx_trace_rexi": (_I, [_I, _P, _I]),
    "swx_shard_init": (_I, [_P, _I, _I, _I, _I]),
    "swx_sht_shard_counts": (_S, [_P, _P, _I, _I, _P, _P]),
    "swx_sht_tendency_shard": (_I, [_P, _I, _I, _P, _P, _P, _P, _P, _P, _P, _S, _P]),
    "swx_sht_shard_push": (_I, [_P, _P, _I, _I, _P, _P, _P]),
    "swx_sht_peer_map_create": (_I, [_P, _P, _P, ctypes.POINTER(_P)]),
    "swx_sht_peer_map_destroy": (_I, [_P]),
    "swx_sht_tendency_shard_peer": (_I, [_P, _I, _I, _P, _P, _P, _P, _P, _P, _S, _P]),
    "swx_solver_set_columns": (_I, [_P, _I, _I]),
    "swx_solver_cache_bytes": (_S, [_P]),
    "swx_sht_tendency_part": (_I, [_P, _I, _I, _I, _I, _P, _P, _P, _P, _S, _P]),
    "swx_sht_has_stages": (_I, [_P]),
    "swx_sht_transform_shard_counts": (_S, [_P, _P, _I, _I, _P, _P]),
    "swx_sht_synthesis_shard": (_I, [_P, _I, _I, _P, _P, _P, _P, _P, _P, _S, _P]),
    "swx_sht_analysis_shard": (_I, [_P, _I, _I, _P, _P, _P, _P, _P, _P, _S, _P]),
}

SWX_MAX_RANKS = 64


class Shard(ctypes.Structure):
    """swx_shard (include/swx.h): column and latitude-pair bounds of K ranks."""
    _fields_ = [("nranks", ctypes.c_int), ("rank", ctypes.c_int),
                ("m_bounds", ctypes.c_int * (SWX_MAX_RANKS + 1)),
                ("p_bounds", ctypes.c_int * (SWX_MAX_RANKS + 1))]

_lib = None
_lock = threading.Lock()


def load(path: str = LIB_PATH) -> ctypes.CDLL:
    """Load and type the library (no device needed)."""
    global _lib
    with _lock:
        if _lib is not None:
            return _lib
        if not os.path.exists(path):
            raise ConfigurationError(
                f"{path} is missing: build it with `python -m paper_1805_06557_b200.build` "
                "(there is no CPU fallback)")
        lib = ctypes.CDLL(path)
        for name, (res, args) in SIGNATURES.items():
            fn = getattr(lib, name)
            fn.restype = res
            fn.argtypes = args
        _lib = lib
        return lib


def lib() -> ctypes.CDLL:
    """The library, after checking a CUDA device is present."""
    import torch

    if not torch.cuda.is_available():
        raise ConfigurationError(
            "no CUDA device: the B200 REXI path has no CPU fallback")
    return load()


def check(rc: int, err_pole: int | None = None, err_index: int | None = None):
    if rc == SWX_OK:
        return
    msg = load().swx_last_error().decode(errors="replace")
    if rc == SWX_ERR_SOLVER:
        exc = SolverError(msg)
        exc.pole = err_pole
        exc.index = err_index
        raise exc
    if rc == SWX_ERR_CONFIG:
        raise ConfigurationError(msg)
    if rc == SWX_ERR_DATA:
        raise DataError(msg)
    raise SwerexiError(f"CUDA failure in libswx: {msg}")


def c128(z: complex) -> C128:
    z = complex(z)
    return C128(z.real, z.imag)
